"""Per-SM streaming bandwidth calibration (bulk copies vs vector loads)."""
import ctypes as C
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "libprobe.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                           "-Xcompiler", "-fPIC", "-o", so, os.path.join(HERE, "tma_probe.cu")])
lib = C.CDLL(so)
lib.probe_bulk.argtypes = [C.c_void_p, C.c_long, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
lib.probe_ldg.argtypes = [C.c_void_p, C.c_long, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
buf = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
sink = torch.zeros(1024, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timeit(fn, total):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        flush.add_(1)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[2]
    return ms, total / ms / 1e6


s = torch.cuda.current_stream().cuda_stream
for ctas in (28, 74, 148):
    per = (1 << 30) // ctas // 65536 * 65536
    for chunk, stages in ((16384, 4), (16384, 8), (16384, 12), (32768, 6), (8192, 16), (4096, 32)):
        ms, gbs = timeit(lambda: lib.probe_bulk(buf.data_ptr(), per, chunk, stages, ctas, sink.data_ptr(), s), per * ctas)
        print(f"bulk ctas={ctas:3d} chunk={chunk:5d} stages={stages:2d} inflight={chunk*stages//1024:4d}KB: "
              f"{gbs:7.0f} GB/s total, {gbs/ctas:6.1f} GB/s/SM", flush=True)
    for thr in (256, 1024):
        ms, gbs = timeit(lambda: lib.probe_ldg(buf.data_ptr(), per, ctas, thr, sink.data_ptr(), s), per * ctas)
        print(f"ldg  ctas={ctas:3d} threads={thr}: {gbs:7.0f} GB/s total, {gbs/ctas:6.1f} GB/s/SM", flush=True)
