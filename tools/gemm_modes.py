"""C3 GEMM shapes under each weight-tile mode (vlc_set_tuning key 7): 1 = 128-row, 2 = 256-row."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import gemm_bench as gb  # noqa: E402

N = gb.N
for m in (236, 112, 44):
    for mode in (1, 2):
        gb.lib.vlc_set_tuning(7, mode)
        print(f"-- mode {mode} m={m}", flush=True)
        for n, k, kind in ((10752, 3584, N.EPI_BF16), (3584, 3584, N.EPI_RESID), (14336, 3584, N.EPI_BF16),
                           (3584, 7168, N.EPI_RESID)):
            gb.run(n, k, m, 0, kind=kind)
    if m == 236:
        gb.run(152064, 3584, 236, 0, kind=N.EPI_F32)
gb.lib.vlc_set_tuning(7, 1)
