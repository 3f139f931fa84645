"""tcgen05.mma issue / completion rate, cta_group::1 (M = 128) vs cta_group::2 (M = 256 over an SM pair), by N
(tools/tma_probe.cu mma_probe / mma2_probe; one CTA / one pair, operands = smem garbage, timing only)."""
import ctypes as C
import os
import subprocess

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "libprobe.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                       "-Xcompiler", "-fPIC", "-o", so, os.path.join(HERE, "tma_probe.cu"), "-lcuda"])
lib = C.CDLL(so)
out = torch.zeros(4, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
groups = 1000
for n in (64, 128, 192, 240, 256):
    assert lib.probe_mma(n, groups, 0, C.c_void_p(out.data_ptr()), C.c_void_p(s), 1) == 0
    torch.cuda.synchronize()
    o1 = out.cpu().tolist()
    assert lib.probe_mma2(n, groups, C.c_void_p(out.data_ptr()), C.c_void_p(s)) == 0
    torch.cuda.synchronize()
    o2 = out.cpu().tolist()
    print(f"N={n:3d}: cta_group::1 M=128 {o1[1] / (groups * 8):6.1f} cyc/MMA   cta_group::2 M=256 "
          f"{o2[1] / (groups * 8):6.1f} cyc/MMA (issue {o2[0] / (groups * 8):6.1f})", flush=True)
