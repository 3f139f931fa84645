"""Cluster-multicast activation loads in the one-tile-per-CTA GEMM (tuning key 16): timing + check."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_12977_b200 import _native as N  # noqa: E402
import gemm_bench as gb  # noqa: E402

lib = N.load()


def check(n, k, m, mc):
    lib.vlc_set_tuning(16, mc)
    R = N.row_tile(m)
    Wf = torch.randn(n, k, device="cuda").bfloat16()
    Xf = torch.randn(m, k, device="cuda").bfloat16()
    W, X = N.pack(Wf, 128), N.pack(Xf, R, rows_cap=-(-m // R) * R)
    out = torch.zeros(m + 256, n, device="cuda", dtype=torch.float32)
    e = N.Epilogue()
    e.kind, e.n_valid, e.m_tokens, e.out, e.ldo = N.EPI_F32, n, m, out.data_ptr(), n
    N.check(lib.vlc_gemm_bf16(W.data_ptr(), n, k, X.data_ptr(), -(-m // R) * R, m, e, 0, gb.ws.data_ptr(),
                              gb.ws.numel() * 4, gb.cnt.data_ptr(), torch.cuda.current_stream().cuda_stream), "g")
    torch.cuda.synchronize()
    ref = Xf.float() @ Wf.float().t()
    err = ((out[:m] - ref).abs().max() / ref.abs().max()).item()
    print(f"check N={n} K={k} M={m} mc={mc}: rel err {err:.2e}", flush=True)
    assert err < 1e-3


if __name__ == "__main__":
    for mc in (1, 8):
        for n, k, m in ((14336, 3584, 236), (1024, 512, 100)):
            check(n, k, m, mc)
    for mc in (1, 8, 1, 8):
        lib.vlc_set_tuning(16, mc)
        print(f"-- mc {mc}", flush=True)
        for n, k, m, kind in ((10752, 3584, 236, N.EPI_BF16), (14336, 3584, 236, N.EPI_BF16),
                              (14336, 3584, 236, N.EPI_SWIGLU), (10752, 3584, 112, N.EPI_BF16)):
            gb.run(n, k, m, 0, kind=kind)
    lib.vlc_set_tuning(16, 1)
