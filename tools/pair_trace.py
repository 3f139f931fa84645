"""Per-unit stamps of the CTA-pair GEMM's data path (experiment build with -DVLC_PAIR_TRACE:
  python tools/build_variant.py exp/v/lib_PTRACE.so -DVLC_PAIR_TRACE
  VLC_LIB_VARIANT=exp/v/lib_PTRACE.so python tools/pair_trace.py)
Stamps per unit u (one 128-wide k-block of one tile) of a pair's range: s0 producer issued the unit's copies,
s1 leader saw its own stage land, s2 leader saw the peer's relay, s3 leader committed the unit's UMMAs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_12977_b200 import _native as N  # noqa: E402
if os.environ.get("VLC_LIB_VARIANT"):
    N.LIB_PATH = os.environ["VLC_LIB_VARIANT"]
lib = N.load()
ws = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
cnt = torch.zeros(1 << 16, dtype=torch.int32, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def trace(n, k, m, label):
    R = N.row_tile(m, n)
    W = N.pack(torch.randn(n, k, device="cuda").bfloat16(), 128)
    X = N.pack(torch.randn(m, k, device="cuda").bfloat16(), R, rows_cap=-(-m // R) * R)
    out = torch.zeros(m + 256, n, device="cuda", dtype=torch.float32)
    e = N.Epilogue()
    e.kind, e.n_valid, e.m_tokens, e.out, e.ldo = N.EPI_F32, n, m, out.data_ptr(), n
    dbg = torch.zeros(4096 + 148 * 64 * 4, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for it in range(3):
        flush.add_(1)
        lib.vlc_set_debug_buffer(dbg.data_ptr() if it == 2 else None)
        N.check(lib.vlc_gemm_bf16(W.data_ptr(), n, k, X.data_ptr(), -(-m // R) * R, m, e, 0, ws.data_ptr(),
                                  ws.numel() * 4, cnt.data_ptr(), s), "g")
        torch.cuda.synchronize()
    lib.vlc_set_debug_buffer(None)
    d = dbg[4096:].view(148, 64, 4).cpu().numpy().astype(np.float64)
    t0 = d[d > 0].min()
    d = np.where(d > 0, (d - t0) / 1e3, np.nan)
    lead = d[0::2]                       # leader CTAs: s0 own producer, s1 own land, s2 peer relay, s3 commit
    peer = d[1::2]                       # non-leader: s0 its producer, s1 its stage landed (relay time)
    U = slice(6, 40)
    land = lead[:, U, 1] - lead[:, U, 0]
    peer_land = peer[:, U, 1] - peer[:, U, 0]
    wait_peer = lead[:, U, 2] - lead[:, U, 1]
    cad = np.diff(lead[:, :, 3], axis=1)[:, U]
    reissue = lead[:, 9:43, 0] - lead[:, 6:40, 3]      # producer re-issue after the commit 3 units earlier
    med = lambda a: np.nanmedian(a)  # noqa: E731
    print(f"{label}: N={n} K={k} M={m}")
    print(f"   own stage issue -> landed (leader)      {med(land):6.2f} us   (peer CTA {med(peer_land):6.2f} us)")
    print(f"   leader: own landed -> peer relay seen   {med(wait_peer):6.2f} us")
    print(f"   commit cadence per unit                 {med(cad):6.2f} us")
    print(f"   issue of unit u+3 - commit of unit u    {med(reissue):6.2f} us")
    print(f"   first units: s0 {np.round(np.nanmedian(lead[:, :6, 0], axis=0), 2)}  s3 "
          f"{np.round(np.nanmedian(lead[:, :6, 3], axis=0), 2)}")


lib.vlc_set_tuning(10, -16)                  # CTA pair for the one-wave shape as well
trace(10752, 3584, 236, "QKV shape, pair stream-K")
lib.vlc_set_tuning(10, 160)
trace(152064, 3584, 236, "LM head, pair stream-K")
