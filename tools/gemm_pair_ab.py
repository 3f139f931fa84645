"""A/B of the GEMM schedules at the C3 projection shapes (c = 236 and 112 tokens): single-CTA
kernel (tuning key 10 = 0) vs the CTA-pair stream-K kernel (key 10 = 32).  Timing only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import gemm_bench as gb  # noqa: E402
from gemm_bench import N, lib  # noqa: E402

SHAPES = [("qkv", 10752, 3584, N.EPI_BF16), ("gate_up", 14336, 3584, N.EPI_SWIGLU),
          ("o", 3584, 3584, N.EPI_RESID), ("down", 3584, 7168, N.EPI_RESID), ("head", 152064, 3584, N.EPI_F32)]
for m in (236, 112):
    for name, n, k, kind in SHAPES:
        for mode in (0, 32):
            lib.vlc_set_tuning(10, mode)
            print(f"{name:8s} pair={mode:2d} ", end="")
            gb.run(n, k, m, 0, kind=kind, reps=10 if name == "head" else 20)
