import ctypes as C
import os
import subprocess
import torch
HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "libprobe.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                       "-Xcompiler", "-fPIC", "-o", so, os.path.join(HERE, "tma_probe.cu")])
lib = C.CDLL(so)
lib.probe_mma.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int]
out = torch.zeros(4, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
import sys
ctas = int(sys.argv[1]) if len(sys.argv) > 1 else 1
groups = int(sys.argv[2]) if len(sys.argv) > 2 else 28
for n in (16, 64, 128, 240, 256):
    for variant in (0, 1, 3):
        for _ in range(2):
            lib.probe_mma(n, groups, variant, out.data_ptr(), s, ctas)
        torch.cuda.synchronize()
        issue, total = out[0].item(), out[1].item()
        mmas = groups * 8
        ideal = 128 * n / 256
        print(f"N={n:3d} variant={variant}: issue {issue/mmas:7.1f} cyc/MMA, complete {total/mmas:7.1f} cyc/MMA "
              f"(ideal {ideal:.0f})", flush=True)
