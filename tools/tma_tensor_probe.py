"""Per-SM throughput of cp.async.bulk (1-D) vs cp.async.bulk.tensor.2d copies from an L2-resident window, by
op size and number of issuing warps (tools/tma_probe.cu tensor_stream)."""
import ctypes as C
import os
import subprocess

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "libprobe.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                       "-Xcompiler", "-fPIC", "-o", so, os.path.join(HERE, "tma_probe.cu"), "-lcuda"])
lib = C.CDLL(so)
lib.probe_tensor.argtypes = [C.c_void_p, C.c_long, C.c_long, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                             C.c_void_p]
rows_total = (3 << 20) // 128          # 3 MB window (L2-resident), shared by all CTAs
buf = torch.empty(rows_total * 128, dtype=torch.uint8, device="cuda")
sink = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for ctas in (84, 148):
    for tensor in (0, 1):
        for issuers in (1, 2, 4):
            for box_rows, stages in ((32, 24), (64, 24), (128, 12), (256, 6)):
                if stages % issuers:
                    continue
                per = 32 << 20
                rows = per // 128
                f = lambda: lib.probe_tensor(buf.data_ptr(), rows_total, rows, box_rows, stages, issuers, tensor, ctas,  # noqa
                                             sink.data_ptr(), s)
                rc = f()
                assert rc == 0, rc
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record(); f(); e1.record(); e1.synchronize()
                ms = e0.elapsed_time(e1)
                ops = rows // box_rows
                print(f"ctas={ctas:3d} {'tensor' if tensor else 'bulk  '} issuers={issuers} op={box_rows * 128 >> 10:2d}KB "
                      f"in flight {box_rows * 128 * stages >> 10:3d} KB: {per * ctas / ms / 1e6:7.0f} GB/s total "
                      f"{per / ms / 1e6:6.1f} GB/s/SM {ms * 1e6 / ops:6.1f} ns/op", flush=True)
