"""Microbenchmark of vlc_attn_paged at the C3 layer shape (hd 128, 28 heads, 4128 keys, 236 queries):
all chunks from request rows vs all from store pages (in-smem re-rotation).  Timing only."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
from paper_2512_12977_b200 import _native as nat  # noqa: E402
if os.environ.get("VLC_LIB_VARIANT"):          # experiment builds (tools/build_variant.py)
    nat.LIB_PATH = os.environ["VLC_LIB_VARIANT"]
from test_kernels_gpu import _paged_case  # noqa: E402


def run(store_every, nq=236, reps=50):
    a, out, ref, keep = _paged_case(nat, 128, 28, 4128, nq, True, store_every, 7)
    lib = nat.load()
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(5):
        nat.check(lib.vlc_attn_paged(a, s), "attn")
    torch.cuda.synchronize()
    err = (out[keep["rowof"].long()].float() - ref).abs().max().item()
    flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        nat.check(lib.vlc_attn_paged(a, s), "attn")
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    print(f"store_every={store_every} nq={nq} items={a.n_items} slots={a.ws_slots}: p50 {ts[len(ts)//2]:.1f} us "
          f"min {ts[0]:.1f} us  err {err:.2e}", flush=True)


if __name__ == "__main__":
    for se in ([int(a) for a in sys.argv[1:]] or (0, 1)):
        run(se)
