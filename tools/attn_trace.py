"""Per-iteration event trace of attention CTA 0 at the C3 shape (vlc_set_trace_buffer)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import attn_bench as ab  # noqa: E402  (runs its own timing first)

if len(sys.argv) > 1:
    ab.lib.vlc_set_tuning(15, int(sys.argv[1]))
    ab.ONE = int(sys.argv[1]) in (30, 31, 32, 33, 34, 35, 36, 37, 38, 39)
a, keep, n = ab.setup()
buf = torch.zeros(256, dtype=torch.int64, device="cuda")
ab.lib.vlc_set_trace_buffer(buf.data_ptr())
ab.N.check(ab.lib.vlc_attn_pp(a, torch.cuda.current_stream().cuda_stream), "pp")
torch.cuda.synchronize()
ab.lib.vlc_set_trace_buffer(None)
t = buf.cpu().numpy().astype(np.float64)
t0 = t[t > 0].min()
us = np.where(t > 0, (t - t0) / 1e3, np.nan)   # k-cycles of SM clock
print("(k-cycles)\niter | softmaxA: s_ready ld_done exp_done arrived | MMA: pA_ok A_issued pB_ok B_issued | load_go | "
      "softmaxB: s_ready ld_done exp_done arrived")
for j in range(16):
    sa = us[j * 4:j * 4 + 4]
    mm = us[64 + j * 4:64 + j * 4 + 4]
    sb = us[160 + j * 4:160 + j * 4 + 4]
    print(f"{j:3d} | " + " ".join(f"{v:6.2f}" for v in sa) + " | " + " ".join(f"{v:6.2f}" for v in mm) +
          f" | {us[128 + j]:6.2f} | " + " ".join(f"{v:6.2f}" for v in sb))
