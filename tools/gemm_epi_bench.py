"""Epilogue cost of the C3 GEMMs: the same weights/activations timed with the plain BF16
epilogue and with the fused ones used in the chain (QKV_ROPE, SWIGLU), plus per-CTA phases."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_12977_b200 import _native as N  # noqa: E402
if os.environ.get("VLC_LIB_VARIANT"):          # experiment builds (tools/build_variant.py)
    N.LIB_PATH = os.environ["VLC_LIB_VARIANT"]

lib = N.load()
ws = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
cnt = torch.zeros(1 << 16, dtype=torch.int32, device="cuda")
kv, hd, m, n_keys = 3584, 128, 236, 4128


def timed(W, n, k, X, R, e, reps=20):
    def go(w):
        N.check(lib.vlc_gemm_bf16(w.data_ptr(), n, k, X.data_ptr(), -(-m // R) * R, m, e, 0, ws.data_ptr(),
                                  ws.numel() * 4, cnt.data_ptr(), torch.cuda.current_stream().cuda_stream), "g")
    go(W[0])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for r in range(reps):
            go(W[r % len(W)])
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    g.replay()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def phases(W, n, k, X, R, e):
    dbg = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    flush.add_(1)
    lib.vlc_set_debug_buffer(dbg.data_ptr())
    N.check(lib.vlc_gemm_bf16(W.data_ptr(), n, k, X.data_ptr(), -(-m // R) * R, m, e, 0, ws.data_ptr(),
                              ws.numel() * 4, cnt.data_ptr(), torch.cuda.current_stream().cuda_stream), "g")
    torch.cuda.synchronize()
    lib.vlc_set_debug_buffer(None)
    d = dbg.view(148, 8).cpu().numpy().astype("float64")
    alive = d[:, 0] > 0
    d = d[alive]
    t0 = d[:, 0].min()
    d = np.where(d > 0, (d - t0) / 1e3, np.nan)
    if n == 3 * kv and alive.sum() == n // 128:    # one tile per CTA: the section of CTA g is g * 128 // kv
        sec = (np.arange(len(d)) * 128) // kv
        for sidx, nm in enumerate("QKV"):
            sel = sec == sidx
            print(f"     section {nm}: acc_full med {np.nanmedian(d[sel, 3]):6.2f}  epilogue end med "
                  f"{np.nanmedian(d[sel, 4]):6.2f} max {np.nanmax(d[sel, 4]):6.2f}")
    for i, nm in enumerate(["start", "prod_go", "prod_done", "acc_full", "partials_done", "fixup_go", "epi_end",
                            "exit"]):
        col = d[:, i]
        col = col[~np.isnan(col)]
        if len(col):
            print(f"     {nm:14s} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f}")


def main():
    k = 3584
    R = N.row_tile(m)
    X = N.pack(torch.randn(m, k, device="cuda").bfloat16(), R, rows_cap=-(-m // R) * R)
    # QKV
    n = 3 * kv
    if os.environ.get("GU_ONLY"):
        return gu(m, k, R, X)
    Ws = [N.pack(torch.randn(n, k, device="cuda").bfloat16(), 128) for _ in range(4)]
    q = torch.zeros(m + 256, kv, device="cuda", dtype=torch.bfloat16)
    kc = torch.zeros(n_keys + 64, kv, device="cuda", dtype=torch.bfloat16)
    vc = torch.zeros_like(kc)
    kpre = torch.zeros(256, kv, device="cuda", dtype=torch.bfloat16)
    pos = torch.from_numpy(np.sort(np.random.default_rng(0).permutation(n_keys)[:m]).astype(np.int32)).cuda()
    qmap = torch.randperm(m, device="cuda").int()
    half = hd // 2
    inv = (10000.0 ** (-np.arange(half, dtype=np.float32) * (2.0 / hd))).astype(np.float32)
    ang = np.arange(n_keys + 64, dtype=np.float32)[:, None] * inv
    cos = torch.from_numpy(np.cos(ang)).cuda()
    sin = torch.from_numpy(np.sin(ang)).cuda()
    c_, s_ = np.cos(ang), np.sin(ang)
    cs = torch.from_numpy(np.ascontiguousarray(np.stack([c_.reshape(len(ang), half // 2, 2),
                                                         s_.reshape(len(ang), half // 2, 2)], axis=2)
                                              .reshape(len(ang), hd))).cuda()
    out = torch.zeros(m + 256, n, device="cuda", dtype=torch.bfloat16)
    plain = N.Epilogue()
    plain.kind, plain.n_valid, plain.m_tokens, plain.out, plain.ldo = N.EPI_BF16, n, m, out.data_ptr(), n
    rope = N.Epilogue()
    for kk, v in dict(kind=N.EPI_QKV_ROPE, n_valid=n, m_tokens=m, out=q.data_ptr(), ldo=kv, out2=kc.data_ptr(), ld2=kv,
                      out3=vc.data_ptr(), ld3=kv, out4=kpre.data_ptr(), ld4=kv, map1=qmap.data_ptr(),
                      map2=pos.data_ptr(), pos=pos.data_ptr(), cos_tab=cos.data_ptr(), sin_tab=sin.data_ptr(),
                      tab_ld=half, hd=hd, seg=kv, cs_tab=cs.data_ptr() if os.environ.get("CS", "1") == "1" else None).items():
        setattr(rope, kk, v)
    if os.environ.get("ROPE_ONLY"):
        rope_nk = N.Epilogue()
        for f, _ in rope._fields_:
            setattr(rope_nk, f, getattr(rope, f))
        rope_nk.out4 = None
        rope_id = N.Epilogue()     # identity Q/K destination maps (map1 = None: q row = token)
        for f, _ in rope._fields_:
            setattr(rope_id, f, getattr(rope, f))
        rope_id.map1 = None
        for name, e in (("qkv bf16", plain), ("qkv rope", rope), ("qkv rope no kpre", rope_nk),
                        ("qkv rope q identity", rope_id)):
            print(f"{name}: {timed(Ws, n, k, X, R, e):.2f} us", flush=True)
            phases(Ws[0], n, k, X, R, e)
        return
    for name, e in (("qkv bf16", plain), ("qkv rope", rope)):
        for um in (64, 1000):
            lib.vlc_set_tuning(9, um)
            print(f"{name} unsplit_min={um}: {timed(Ws, n, k, X, R, e):.2f} us", flush=True)
            phases(Ws[0], n, k, X, R, e)
        lib.vlc_set_tuning(9, 64)
    gu(m, k, R, X)


def gu(m, k, R, X):
    plain = N.Epilogue()
    out0 = torch.zeros(m + 256, 14336, device="cuda", dtype=torch.bfloat16)
    plain.kind, plain.n_valid, plain.m_tokens, plain.out, plain.ldo = N.EPI_BF16, 14336, m, out0.data_ptr(), 14336
    # gate/up
    n = 14336
    Ws = [N.pack(torch.randn(n, k, device="cuda").bfloat16(), 128) for _ in range(3)]
    h = torch.zeros(N.packed_numel(m, n // 2, R), device="cuda", dtype=torch.bfloat16)
    out = torch.zeros(m + 256, n, device="cuda", dtype=torch.bfloat16)
    plain.n_valid, plain.out, plain.ldo = n, out.data_ptr(), n
    sw = N.Epilogue()
    sw.kind, sw.n_valid, sw.m_tokens, sw.out, sw.ldo, sw.pk_rows, sw.pk_kb = N.EPI_SWIGLU, n, m, h.data_ptr(), n // 2, R, n // 256
    sw_rm = N.Epilogue()   # SwiGLU written row-major (isolates the packed-layout store cost)
    sw_rm.kind, sw_rm.n_valid, sw_rm.m_tokens, sw_rm.out, sw_rm.ldo = N.EPI_SWIGLU, n, m, out.data_ptr(), n // 2
    bf_pk = N.Epilogue()   # plain BF16 written packed
    hp = torch.zeros(N.packed_numel(m, n, R), device="cuda", dtype=torch.bfloat16)
    bf_pk.kind, bf_pk.n_valid, bf_pk.m_tokens, bf_pk.out, bf_pk.ldo, bf_pk.pk_rows, bf_pk.pk_kb = \
        N.EPI_BF16, n, m, hp.data_ptr(), n, R, n // 128
    if os.environ.get("GU_ONLY"):
        for name, e in (("gu bf16", plain), ("gu bf16 packed", bf_pk), ("gu swiglu", sw), ("gu swiglu rowmajor", sw_rm)):
            print(f"{name}: {timed(Ws, n, k, X, R, e):.2f} us", flush=True)
            phases(Ws[0], n, k, X, R, e)
        return
    for name, e in (("gu bf16", plain), ("gu swiglu", sw)):
        for um in (64, 1000):
            lib.vlc_set_tuning(9, um)
            print(f"{name} unsplit_min={um}: {timed(Ws, n, k, X, R, e):.2f} us", flush=True)
            phases(Ws[0], n, k, X, R, e)
        lib.vlc_set_tuning(9, 64)


main()
