"""Per-SM throughput of cp.async.bulk copies from an L2-resident window, by op size (tools/tma_probe.cu):
each op seems to cost a fixed ~0.3 us of the SM's TMA unit regardless of its size up to 32 KB."""
import ctypes as C
import os
import subprocess

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "libprobe.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                       "-Xcompiler", "-fPIC", "-o", so, os.path.join(HERE, "tma_probe.cu")])
lib = C.CDLL(so)
lib.probe_bulk_l2.argtypes = [C.c_void_p, C.c_long, C.c_int, C.c_int, C.c_int, C.c_long, C.c_int, C.c_void_p, C.c_void_p]
buf = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
sink = torch.zeros(1024, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
import sys
SHARED = [int(a) for a in sys.argv[1:]] or [1]
for shared in SHARED:
  print(f"-- shared window {shared} (1: every CTA reads the same 3 MB window; 0: a private window per CTA)")
  for ctas in (84, 148):
    for chunk, stages in ((4096, 32), (8192, 16), (16384, 12), (32768, 6), (49152, 4), (65536, 3), (98304, 2)):
        per = 32 << 20
        wrap = 3 << 20 if shared else 512 << 10
        f = lambda: lib.probe_bulk_l2(buf.data_ptr(), per, chunk, stages, ctas, wrap, shared, sink.data_ptr(), s)  # noqa
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); f(); e1.record(); e1.synchronize()
        ms = e0.elapsed_time(e1)
        tot = per * ctas
        ops = per // chunk
        print(f"ctas={ctas:3d} chunk={chunk >> 10:3d}KB stages={stages:2d} (in flight {chunk * stages >> 10} KB): "
              f"{tot / ms / 1e6:8.0f} GB/s total {tot / ms / 1e6 / ctas:6.1f} GB/s/SM  {ms * 1e6 / ops:6.1f} ns/op",
              flush=True)
