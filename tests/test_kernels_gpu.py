"""Kernel-level numerics of libvlcache against plain PyTorch fp32 references.

Every op is checked through the C ABI (ctypes), on the same bf16 inputs the
kernel sees, so the only differences are accumulation order and output rounding.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nat(cuda_ok):
    from paper_2512_12977_b200 import _native
    _native.load()
    return _native


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _epi(nat, **kw):
    e = nat.Epilogue()
    for k, v in kw.items():
        setattr(e, k, v)
    return e


def _gemm(nat, W, X, m, epi, splits=1):
    """W [n_pad, k_pad] and X [rows, k_pad] row-major bf16 -> packed operands -> vlc_gemm_bf16."""
    ws = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")
    cnt = torch.zeros(16384, dtype=torch.int32, device="cuda")
    R = nat.row_tile(m, W.shape[0])
    Wp = nat.pack(W, 128)
    Xp = nat.pack(X[:m], R, rows_cap=-(-m // R) * R)
    nat.check(nat.load().vlc_gemm_bf16(Wp.data_ptr(), W.shape[0], W.shape[1], Xp.data_ptr(), -(-m // R) * R, m,
                                       epi, splits, ws.data_ptr(), ws.numel(), cnt.data_ptr(), _stream()),
              "gemm")
    torch.cuda.synchronize()


@pytest.mark.parametrize("n_pad,k_pad,m,splits", [(128, 128, 16, 1), (256, 128, 40, 1), (384, 512, 100, 3),
                                                  (256, 256, 300, 2), (128, 1024, 256, 4), (512, 256, 1000, 1),
                                                  (3584, 3584, 236, 0), (1024, 7168, 112, 0), (10752, 3584, 240, 0),
                                                  (1280, 768, 600, 7), (512, 4096, 40, 0)])
def test_gemm_f32_matches_torch(nat, n_pad, k_pad, m, splits):
    g = torch.Generator(device="cuda").manual_seed(n_pad + m)
    W = torch.randn(n_pad, k_pad, device="cuda", generator=g).bfloat16()
    X = torch.randn(max(256, m), k_pad, device="cuda", generator=g).bfloat16()
    out = torch.full((m, n_pad), float("nan"), device="cuda")
    epi = _epi(nat, kind=nat.EPI_F32, n_valid=n_pad, m_tokens=m, out=out.data_ptr(), ldo=n_pad)
    _gemm(nat, W, X, m, epi, splits)
    ref = X[:m].float() @ W.float().t()
    err = (out - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err


def test_gemm_resid_and_swiglu(nat):
    g = torch.Generator(device="cuda").manual_seed(1)
    n, k, m = 256, 128, 50
    W = torch.randn(n, k, device="cuda", generator=g).bfloat16()
    X = torch.randn(256, k, device="cuda", generator=g).bfloat16()
    x = torch.randn(m, n, device="cuda", generator=g)
    x0 = x.clone()
    _gemm(nat, W, X, m, _epi(nat, kind=nat.EPI_RESID, n_valid=n, m_tokens=m, out=x.data_ptr(), ldo=n), 2)
    acc = X[:m].float() @ W.float().t()
    assert torch.allclose(x, x0 + acc, atol=1e-4, rtol=1e-5)
    h = torch.zeros(m, n // 2, device="cuda", dtype=torch.bfloat16)
    _gemm(nat, W, X, m, _epi(nat, kind=nat.EPI_SWIGLU, n_valid=n, m_tokens=m, out=h.data_ptr(), ldo=n // 2))
    R = nat.row_tile(m)   # packed SwiGLU output (as consumed by the down projection)
    hp = torch.zeros(nat.packed_numel(m, n // 2, R), device="cuda", dtype=torch.bfloat16)
    _gemm(nat, W, X, m, _epi(nat, kind=nat.EPI_SWIGLU, n_valid=n, m_tokens=m, out=hp.data_ptr(), ldo=n // 2,
                             pk_rows=R, pk_kb=-(-(n // 2) // 128)))
    assert torch.equal(nat.unpack(hp, m, n // 2, R), h)
    gate, up = acc[:, 0::2], acc[:, 1::2]
    ref = gate / (1 + torch.exp(-gate)) * up
    assert (h.float() - ref).abs().max().item() <= 2e-2 * ref.abs().max().item()


def _rope_ref(x, pos, hd, base=10000.0):
    half = hd // 2
    inv = base ** (-torch.arange(half, dtype=torch.float32) * (2.0 / hd))
    ang = pos.float().cpu()[:, None] * inv[None]
    c, s = torch.cos(ang).cuda(), torch.sin(ang).cuda()
    n = x.shape[0]
    xh = x.reshape(n, -1, hd)
    a, b = xh[..., :half], xh[..., half:]
    return torch.cat([a * c[:, None] - b * s[:, None], b * c[:, None] + a * s[:, None]], -1).reshape(n, -1)


def _tables(hd, npos, base=10000.0):
    half = hd // 2
    inv = (base ** (-np.arange(half, dtype=np.float32) * (2.0 / hd))).astype(np.float32)
    ang = np.arange(npos, dtype=np.float32)[:, None] * inv
    return (torch.from_numpy(np.cos(ang, dtype=np.float32)).cuda(),
            torch.from_numpy(np.sin(ang, dtype=np.float32)).cuda())


def _perm_rows(kv, hd):
    """device row order for rope pairing: within a head, rows (t, t+hd/2) adjacent."""
    idx = []
    for h in range(kv // hd):
        for t in range(hd // 2):
            idx += [h * hd + t, h * hd + t + hd // 2]
    return torch.tensor(idx)


@pytest.mark.parametrize("hd,heads,m,cs_tab,splits", [
    (128, 3, 37, False, 2), (32, 8, 37, False, 2), (16, 2, 37, False, 2), (128, 3, 37, True, 2),
    (32, 8, 37, True, 2), (128, 4, 300, True, 2), (128, 2, 200, False, 2),
    # one tile per CTA (decoupled rings, staged token metadata), C3-like widths
    (128, 28, 236, True, 0), (128, 28, 236, False, 0), (128, 28, 141, True, 0), (64, 56, 200, True, 0),
    (16, 64, 97, True, 0)])
def test_gemm_qkv_rope_epilogue(nat, hd, heads, m, cs_tab, splits):
    """cs_tab: the interleaved (c0 c1 s0 s1) per-position table the model passes; without it the
    epilogue reads the split cos/sin tables.  The epilogue rotates four pairs per lane (8 features)."""
    kv = hd * heads
    d = 128
    g = torch.Generator(device="cuda").manual_seed(hd)
    Wq, Wk, Wv = (torch.randn(kv, d, device="cuda", generator=g).bfloat16() for _ in range(3))
    perm = _perm_rows(kv, hd).cuda()
    n_pad = ((3 * kv + 127) // 128) * 128
    W = torch.zeros(n_pad, d, device="cuda", dtype=torch.bfloat16)
    W[:kv], W[kv:2 * kv], W[2 * kv:3 * kv] = Wq[perm], Wk[perm], Wv
    X = torch.randn(max(256, m), d, device="cuda", generator=g).bfloat16()
    pos = torch.randperm(500, device="cuda", generator=g)[:m].int()
    qmap = torch.randperm(m, device="cuda", generator=g).int()
    kvmap = (pos + 3).int()
    cos, sin = _tables(hd, 600)
    cs = torch.stack([cos.reshape(600, hd // 4, 2), sin.reshape(600, hd // 4, 2)], 2).reshape(600, hd).contiguous()
    q = torch.zeros(m, kv, device="cuda", dtype=torch.bfloat16)
    kc = torch.zeros(600, kv, device="cuda", dtype=torch.bfloat16)
    vc = torch.zeros_like(kc)
    kpre = torch.zeros(m, kv, device="cuda", dtype=torch.bfloat16)
    epi = _epi(nat, kind=nat.EPI_QKV_ROPE, n_valid=3 * kv, m_tokens=m, out=q.data_ptr(), ldo=kv,
               out2=kc.data_ptr(), ld2=kv, out3=vc.data_ptr(), ld3=kv, out4=kpre.data_ptr(), ld4=kv,
               map1=qmap.data_ptr(), map2=kvmap.data_ptr(), pos=pos.data_ptr(), cos_tab=cos.data_ptr(),
               sin_tab=sin.data_ptr(), tab_ld=hd // 2, hd=hd, seg=kv,
               cs_tab=cs.data_ptr() if cs_tab else None)
    _gemm(nat, W, X, m, epi, splits)
    Xf = X[:m].float()
    qr = _rope_ref(Xf @ Wq.float().t(), pos, hd)
    kr = _rope_ref(Xf @ Wk.float().t(), pos, hd)
    v = Xf @ Wv.float().t()
    tol = lambda r: 1e-2 * r.abs().max().item()
    assert (q[qmap.long()].float() - qr).abs().max().item() < tol(qr)
    assert (kc[kvmap.long()].float() - kr).abs().max().item() < tol(kr)
    assert (vc[kvmap.long()].float() - v).abs().max().item() < tol(v)
    assert (kpre.float() - Xf @ Wk.float().t()).abs().max().item() < tol(v)


def test_gemm_qkv_rope_needs_head_dim_multiple_of_8(nat):
    W = torch.zeros(128, 128, device="cuda", dtype=torch.bfloat16)
    X = torch.zeros(16, 128, device="cuda", dtype=torch.bfloat16)
    z = torch.zeros(64, device="cuda", dtype=torch.int32)
    tab = torch.zeros(64 * 6, device="cuda")
    out = torch.zeros(16, 36, device="cuda", dtype=torch.bfloat16)
    epi = _epi(nat, kind=nat.EPI_QKV_ROPE, n_valid=108, m_tokens=16, out=out.data_ptr(), ldo=36, out2=out.data_ptr(),
               ld2=36, out3=out.data_ptr(), ld3=36, map2=z.data_ptr(), pos=z.data_ptr(), cos_tab=tab.data_ptr(),
               sin_tab=tab.data_ptr(), tab_ld=6, hd=12, seg=36)
    with pytest.raises(nat.NativeError, match="head_dim % 8"):
        _gemm(nat, W, X, 16, epi, 0)


def _attn_ref(q, k, v, qpos, heads, hd, nkeys):
    nq = q.shape[0]
    qh = q.float().reshape(nq, heads, hd).transpose(0, 1)
    kh = k.float()[:nkeys].reshape(nkeys, heads, hd).transpose(0, 1)
    vh = v.float()[:nkeys].reshape(nkeys, heads, hd).transpose(0, 1)
    s = qh @ kh.transpose(1, 2) / math.sqrt(hd)
    vis = torch.arange(nkeys, device=q.device)[None, :] <= qpos.long()[:, None]
    s = s.masked_fill(~vis[None], float("-inf"))
    return (torch.softmax(s, -1) @ vh).transpose(0, 1).reshape(nq, -1)


def test_kv_relocate_matches_torch(nat):
    g = torch.Generator(device="cuda").manual_seed(5)
    L, T, kv, hd, P = 3, 100, 256, 128, 16
    ppl = (T + P - 1) // P
    npages = L * ppl + 5
    kpool = torch.randn(npages * P, kv, device="cuda", generator=g).bfloat16()
    vpool = torch.randn(npages * P, kv, device="cuda", generator=g).bfloat16()
    ptab = torch.randperm(npages, device="cuda", generator=g)[:L * ppl].int()
    kv_rows = 400
    kc = torch.zeros(L, kv_rows, kv, device="cuda", dtype=torch.bfloat16)
    vc = torch.zeros_like(kc)
    cos, sin = _tables(hd, 1000)
    start = 37
    descs, blocks = [], []
    keeps = [10, 5, 0]
    for layer in range(L):
        d = [layer, layer * ppl, keeps[layer], T - keeps[layer], start + keeps[layer], start + keeps[layer], 0, 0]
        for off in range(0, d[3], 8):
            blocks.append([len(descs), off])
        descs.append(d)
    dd = torch.tensor(descs, dtype=torch.int32, device="cuda")
    bb = torch.tensor(blocks, dtype=torch.int32, device="cuda")
    nat.check(nat.load().vlc_kv_relocate(kpool.data_ptr(), vpool.data_ptr(), P, ptab.data_ptr(), kv, hd,
                                         kc.data_ptr(), vc.data_ptr(), kv_rows, dd.data_ptr(), bb.data_ptr(),
                                         len(blocks), cos.data_ptr(), sin.data_ptr(), hd // 2, _stream()),
              "relocate")
    torch.cuda.synchronize()
    for layer in range(L):
        t = torch.arange(keeps[layer], T, device="cuda")
        rows = ptab[layer * ppl + t // P].long() * P + t % P
        pos = start + t
        ref_k = _rope_ref(kpool[rows].float(), pos, hd)
        assert (kc[layer, pos].float() - ref_k).abs().max().item() < 2e-2
        assert torch.equal(vc[layer, pos], vpool[rows])
        assert kc[layer, :start + keeps[layer]].abs().sum().item() == 0


def _paged_case(nat, hd, heads, nkeys, nq, causal, store_every, seed, page_rows=64):
    """Request K/V rows plus a store pool; every `store_every`-th 64-key chunk (0: none) is read from
    a randomly placed store page holding K rotated at the position it was CACHED at, pos - D, with a
    shift D that changes every other 128-key tile (negative ones included); the kernel multiplies such
    chunks against its queries rotated by -D.  The reference rotates the pre-RoPE key straight to its
    position (engine.py:180).  Returns the kernel arguments and the fp32 torch reference."""
    from paper_2512_12977_b200.layout import attention_work, tiles_needed
    kv = heads * hd
    g = torch.Generator(device="cuda").manual_seed(seed)
    layers, layer, kv_rows = 2, 1, nkeys + 64
    kc = torch.randn(layers, kv_rows, kv, device="cuda", generator=g).bfloat16()
    vc = torch.randn(layers, kv_rows, kv, device="cuda", generator=g).bfloat16()
    n_chunks = -(-nkeys // 64)
    npages = n_chunks * 64 // page_rows + 3
    kpool = torch.randn(npages * page_rows, kv, device="cuda", generator=g).bfloat16()
    vpool = torch.randn(npages * page_rows, kv, device="cuda", generator=g).bfloat16()
    ptab = torch.randperm(npages, device="cuda", generator=g).int()
    cos, sin = _tables(hd, nkeys + 64)
    ref_k, ref_v = kc[layer, :nkeys].float().clone(), vc[layer, :nkeys].float().clone()
    kr = kpool.clone()                      # the store's rotated-at-cache-position copy
    half = hd // 2
    inv = 10000.0 ** (-torch.arange(half, device="cuda", dtype=torch.float32) * (2.0 / hd))

    def rope(kf, p):                        # fp32 rotation of [ln, kv] rows to positions p (any sign)
        ang = p.float()[:, None] * inv[None, :]
        cc, ss = torch.cos(ang)[:, None, :], torch.sin(ang)[:, None, :]
        k3 = kf.reshape(len(p), heads, hd)
        a_, b_ = k3[..., :half], k3[..., half:]
        return torch.cat([a_ * cc - b_ * ss, b_ * cc + a_ * ss], -1).reshape(len(p), kv)
    chunks = []
    for ci, c in enumerate(range(0, nkeys, 64)):
        ln = min(64, nkeys - c)
        if store_every and ci % store_every == store_every - 1:
            pti, off = ci * 64 // page_rows, (ci * 64) % page_rows
            rows = ptab[pti].long() * page_rows + off + torch.arange(ln, device="cuda")
            pos = torch.arange(c, c + ln, device="cuda")
            shift = ((ci // 4) % 3) * 37 - 40       # constant over a 128-key tile, new every other tile
            kf = kpool[rows].float()
            ref_k[c:c + ln] = rope(kf, pos).bfloat16().float()
            kr[rows] = rope(kf, pos - shift).bfloat16()
            ref_v[c:c + ln] = vpool[rows].float()
            chunks.append([c, ln | (shift << 8), pti, off])
        else:
            chunks.append([c, ln, c, -1])
    if len(chunks) % 2:
        chunks.append([chunks[-1][0] + 64, chunks[-1][1] & ~0xFF, chunks[-1][2], chunks[-1][3]])
    chunks = np.array(chunks, np.int32)
    if causal:
        qpos = torch.sort(torch.randperm(nkeys, device="cuda", generator=g)[:nq]).values.int()
        qpos[-1] = nkeys - 1
    else:
        qpos = torch.full((nq,), nkeys - 1, dtype=torch.int32, device="cuda")
    q = torch.zeros(max(256, nq + 256), kv, device="cuda", dtype=torch.bfloat16)
    q[:nq] = torch.randn(nq, kv, device="cuda", generator=g).bfloat16()
    rowof = torch.randperm(nq, device="cuda", generator=g).int()
    out = torch.zeros(nq, kv, device="cuda", dtype=torch.bfloat16)
    items, groups = attention_work([(0, 0, nq)], qpos.cpu().numpy(), lambda r, p: tiles_needed(chunks, p), [0],
                                   heads)
    keep = dict(it=torch.from_numpy(items).cuda(), ch=torch.from_numpy(chunks).cuda(),
                ws_o=torch.zeros(max(groups, 1) * 8 * 256 * hd, device="cuda"),
                ws_ml=torch.zeros(max(groups, 1) * 8 * 256 * 2, device="cuda"),
                cnt=torch.zeros(4096, dtype=torch.int32, device="cuda"),
                kc=kc, vc=vc, kpool=kpool, kr=kr, vpool=vpool, ptab=ptab, cos=cos, sin=sin, q=q, qpos=qpos,
                rowof=rowof)
    use_pool = bool(store_every)
    a = nat.AttnPagedArgs(q=q.data_ptr(), q_rows_cap=q.shape[0], kc=kc.data_ptr(), vc=vc.data_ptr(),
                          layers_cap=layers, kv_rows_cap=kv_rows, layer=layer,
                          pool_k=kr.data_ptr() if use_pool else None, pool_v=vpool.data_ptr() if use_pool else None,
                          pool_rows=kpool.shape[0], page_table=ptab.data_ptr(), page_rows=page_rows,
                          cos_tab=cos.data_ptr(), sin_tab=sin.data_ptr(), tab_ld=hd // 2, kv=kv, heads=heads,
                          head_dim=hd, chunks=keep["ch"].data_ptr(), items=keep["it"].data_ptr(),
                          n_items=len(items), qpos=qpos.data_ptr(), rowof=rowof.data_ptr(), out=out.data_ptr(),
                          ldo=kv, pk_rows=0, pk_kb=0, ws_o=keep["ws_o"].data_ptr(), ws_ml=keep["ws_ml"].data_ptr(),
                          ws_slots=groups, counters=keep["cnt"].data_ptr(),
                          scale_log2=math.log2(math.e) / math.sqrt(hd))
    ref = _attn_ref(q[:nq], ref_k, ref_v, qpos, heads, hd, nkeys)
    return a, out, ref, keep


@pytest.mark.parametrize("hd,heads,nkeys,nq,causal,store_every",
                         [(128, 28, 4128, 236, True, 1), (128, 28, 4128, 236, True, 3), (128, 2, 1000, 150, True, 2),
                          (64, 2, 513, 200, True, 2), (32, 8, 288, 44, True, 1), (16, 2, 26, 10, True, 1),
                          (128, 4, 300, 300, True, 0), (128, 3, 256, 256, False, 2), (128, 1, 4128, 600, True, 4),
                          (32, 8, 288, 288, False, 0), (16, 2, 40, 40, True, 0)])
def test_attention_paged_matches_torch(nat, hd, heads, nkeys, nq, causal, store_every):
    """vlc_attn_paged against fp32 torch: request chunks and store chunks (pre-RoPE K rotated in
    shared memory) mixed, causal and bidirectional, split key ranges merged in-kernel."""
    a, out, ref, keep = _paged_case(nat, hd, heads, nkeys, nq, causal, store_every, nkeys + nq + store_every)
    rowof = keep["rowof"]
    for _ in range(2):   # twice: the split-merge counters must be left zeroed for the next launch
        out.zero_()
        nat.check(nat.load().vlc_attn_paged(a, _stream()), "attn_paged")
        torch.cuda.synchronize()
        got = out[rowof.long()].float()
        err = (got - ref).abs().max().item()
        assert err < 2e-2, err
    assert int(keep["cnt"].abs().sum()) == 0
    # packed output (the O-projection's input layout)
    nq, kv = out.shape
    R = nat.row_tile(nq)
    outp = torch.zeros(nat.packed_numel(nq, kv, R), device="cuda", dtype=torch.bfloat16)
    a.out, a.pk_rows, a.pk_kb = outp.data_ptr(), R, -(-kv // 128)
    nat.check(nat.load().vlc_attn_paged(a, _stream()), "attn_paged packed")
    torch.cuda.synchronize()
    assert torch.equal(nat.unpack(outp, nq, kv, R), out)


def test_attention_paged_store_page_size_128(nat):
    """Store pages of 128 rows: a chunk starts mid-page (row offset 64)."""
    a, out, ref, keep = _paged_case(nat, 128, 4, 700, 90, True, 1, 11, page_rows=128)
    nat.check(nat.load().vlc_attn_paged(a, _stream()), "attn_paged")
    torch.cuda.synchronize()
    assert (out[keep["rowof"].long()].float() - ref).abs().max().item() < 2e-2


@pytest.mark.parametrize("n_pad,k_pad,m", [(10752, 3584, 276), (1024, 512, 400), (256, 128, 300), (3584, 7168, 512),
                                           (14336, 3584, 260)])
def test_gemm_wide_token_tile(nat, n_pad, k_pad, m):
    """257..512 tokens of a one-wave GEMM stay ONE wide token tile (two UMMA N chunks into one TMEM
    accumulator, decoupled rings, one k-range per CTA): F32 and RESID (split-K red.add) epilogues."""
    assert nat.row_tile(m, n_pad) == -(-m // 16) * 16
    test_gemm_f32_matches_torch(nat, n_pad, k_pad, m, 0)
    g = torch.Generator(device="cuda").manual_seed(n_pad + m + 5)
    W = torch.randn(n_pad, k_pad, device="cuda", generator=g).bfloat16()
    X = torch.randn(max(512, m), k_pad, device="cuda", generator=g).bfloat16()
    x = torch.randn(m, n_pad, device="cuda", generator=g)
    x0 = x.clone()
    _gemm(nat, W, X, m, _epi(nat, kind=nat.EPI_RESID, n_valid=n_pad, m_tokens=m, out=x.data_ptr(), ldo=n_pad), 0)
    ref = x0 + X[:m].float() @ W.float().t()
    assert (x - ref).abs().max().item() / ref.abs().max().item() < 1e-5


@pytest.mark.parametrize("dec", [0, 1, 3, 12])
@pytest.mark.parametrize("n_pad,k_pad,m", [(10752, 3584, 236), (14336, 3584, 112), (3584, 7168, 236), (3584, 3584, 112)])
def test_gemm_decoupled_rings_and_aligned_split(nat, dec, n_pad, k_pad, m):
    """Schedules of the chain GEMMs: one CTA per tile and tile-aligned split-K (any split count),
    with coupled rings (key 18 = 0) or decoupled weight / activation rings (automatic depth, 3
    activation stages, 2 half-k-block activation stages)."""
    lib = nat.load()
    lib.vlc_set_tuning(18, dec)
    lib.vlc_set_tuning(20, 16)
    try:
        test_gemm_f32_matches_torch(nat, n_pad, k_pad, m, 0)
        g = torch.Generator(device="cuda").manual_seed(n_pad + m + 1)
        W = torch.randn(n_pad, k_pad, device="cuda", generator=g).bfloat16()
        X = torch.randn(max(256, m), k_pad, device="cuda", generator=g).bfloat16()
        x = torch.randn(m, n_pad, device="cuda", generator=g)
        x0 = x.clone()
        _gemm(nat, W, X, m, _epi(nat, kind=nat.EPI_RESID, n_valid=n_pad, m_tokens=m, out=x.data_ptr(), ldo=n_pad), 0)
        ref = x0 + X[:m].float() @ W.float().t()
        assert (x - ref).abs().max().item() / ref.abs().max().item() < 1e-5
    finally:
        lib.vlc_set_tuning(18, 1)
        lib.vlc_set_tuning(20, 16)


@pytest.fixture
def gemm_mode(nat):
    yield lambda mode: nat.load().vlc_set_tuning(7, mode)
    nat.load().vlc_set_tuning(7, 1)


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("n_pad,k_pad,m,ctas", [(256, 256, 40, 0), (512, 1024, 240, 0), (10752, 3584, 236, 0),
                                                (3584, 7168, 236, 0), (768, 256, 44, 5), (1024, 512, 600, 0)])
def test_gemm_tile_modes_f32_resid(nat, gemm_mode, mode, n_pad, k_pad, m, ctas):
    """128-row (mode 1) and 256-row (mode 2) weight tiles, stream-K splits, F32 and RESID
    (red.add) epilogues against torch."""
    gemm_mode(mode)
    g = torch.Generator(device="cuda").manual_seed(n_pad + k_pad + m)
    W = torch.randn(n_pad, k_pad, device="cuda", generator=g).bfloat16()
    X = torch.randn(max(256, m), k_pad, device="cuda", generator=g).bfloat16()
    ref = X[:m].float() @ W.float().t()
    out = torch.full((m, n_pad), float("nan"), device="cuda")
    _gemm(nat, W, X, m, _epi(nat, kind=nat.EPI_F32, n_valid=n_pad, m_tokens=m, out=out.data_ptr(), ldo=n_pad), ctas)
    assert (out - ref).abs().max().item() / ref.abs().max().item() < 1e-5
    x = torch.randn(m, n_pad, device="cuda", generator=g)
    x0 = x.clone()
    _gemm(nat, W, X, m, _epi(nat, kind=nat.EPI_RESID, n_valid=n_pad, m_tokens=m, out=x.data_ptr(), ldo=n_pad), ctas)
    assert ((x - x0) - ref).abs().max().item() / ref.abs().max().item() < 1e-5


@pytest.mark.parametrize("mode", [1, 2])
def test_gemm_tile_modes_swiglu_packed(nat, gemm_mode, mode):
    gemm_mode(mode)
    g = torch.Generator(device="cuda").manual_seed(7)
    n, k, m = 1024, 512, 236
    W = torch.randn(n, k, device="cuda", generator=g).bfloat16()
    X = torch.randn(256, k, device="cuda", generator=g).bfloat16()
    acc = X[:m].float() @ W.float().t()
    R = nat.row_tile(m)
    hp = torch.zeros(nat.packed_numel(m, n // 2, R), device="cuda", dtype=torch.bfloat16)
    _gemm(nat, W, X, m, _epi(nat, kind=nat.EPI_SWIGLU, n_valid=n, m_tokens=m, out=hp.data_ptr(), ldo=n // 2,
                             pk_rows=R, pk_kb=-(-(n // 2) // 128)))
    h = nat.unpack(hp, m, n // 2, R).float()
    gate, up = acc[:, 0::2], acc[:, 1::2]
    ref = gate / (1 + torch.exp(-gate)) * up
    assert (h - ref).abs().max().item() <= 2e-2 * ref.abs().max().item()


@pytest.fixture
def pair_mode(nat):
    nat.load().vlc_set_tuning(10, -32)     # force the CTA-pair kernel from 32-token tiles
    yield
    nat.load().vlc_set_tuning(10, 0)      # the default: pair kernel off


@pytest.mark.parametrize("n_pad,k_pad,m", [(256, 128, 32), (512, 256, 100), (10752, 3584, 236), (2048, 256, 600),
                                           (512, 384, 48)])
def test_gemm_cta_pair_f32(nat, pair_mode, n_pad, k_pad, m):
    """cta_group::2 GEMM (M = 256 over an SM pair, token rows split between the two SMs)."""
    g = torch.Generator(device="cuda").manual_seed(n_pad + m)
    W = torch.randn(n_pad, k_pad, device="cuda", generator=g).bfloat16()
    X = torch.randn(max(256, m), k_pad, device="cuda", generator=g).bfloat16()
    ref = X[:m].float() @ W.float().t()
    out = torch.full((m, n_pad), float("nan"), device="cuda")
    _gemm(nat, W, X, m, _epi(nat, kind=nat.EPI_F32, n_valid=n_pad, m_tokens=m, out=out.data_ptr(), ldo=n_pad), 0)
    assert (out - ref).abs().max().item() / ref.abs().max().item() < 1e-5


@pytest.mark.parametrize("n_pad,k_pad,m", [(38016, 1024, 278), (38144, 512, 500), (76032, 256, 236)])
def test_gemm_multiwave_head_token_tiles(nat, n_pad, k_pad, m):
    """Multi-wave (LM-head-like) GEMM on the default schedule, the CTA-pair stream-K kernel: more than
    256 rows take several token tiles, a weight tile's token tiles being consecutive units."""
    g = torch.Generator(device="cuda").manual_seed(n_pad + m)
    W = torch.randn(n_pad, k_pad, device="cuda", generator=g).bfloat16()
    X = torch.randn(max(256, m), k_pad, device="cuda", generator=g).bfloat16()
    ref = X[:m].float() @ W.float().t()
    out = torch.full((m, n_pad), float("nan"), device="cuda")
    _gemm(nat, W, X, m, _epi(nat, kind=nat.EPI_F32, n_valid=n_pad, m_tokens=m, out=out.data_ptr(), ldo=n_pad), 0)
    assert (out - ref).abs().max().item() / ref.abs().max().item() < 1e-5


def test_gemm_cta_pair_swiglu_packed(nat, pair_mode):
    g = torch.Generator(device="cuda").manual_seed(9)
    n, k, m = 1024, 512, 236
    W = torch.randn(n, k, device="cuda", generator=g).bfloat16()
    X = torch.randn(256, k, device="cuda", generator=g).bfloat16()
    acc = X[:m].float() @ W.float().t()
    R = nat.row_tile(m)
    hp = torch.zeros(nat.packed_numel(m, n // 2, R), device="cuda", dtype=torch.bfloat16)
    _gemm(nat, W, X, m, _epi(nat, kind=nat.EPI_SWIGLU, n_valid=n, m_tokens=m, out=hp.data_ptr(), ldo=n // 2,
                             pk_rows=R, pk_kb=-(-(n // 2) // 128)))
    h = nat.unpack(hp, m, n // 2, R).float()
    gate, up = acc[:, 0::2], acc[:, 1::2]
    ref = gate / (1 + torch.exp(-gate)) * up
    assert (h - ref).abs().max().item() <= 2e-2 * ref.abs().max().item()


@pytest.mark.parametrize("rows,width", [(1, 8), (300, 3584), (5000, 256)])
def test_gather_rows(nat, rows, width):
    """vlc_gather_rows: dst[dst_rows[r]] = src[src_rows[r]] (the merged-KV assembly of ReuseResult.kv)."""
    g = torch.Generator(device="cuda").manual_seed(rows + width)
    src = torch.randn(2 * rows + 3, width, device="cuda", generator=g).bfloat16()
    dst = torch.zeros(rows + 5, width, device="cuda", dtype=torch.bfloat16)
    s_idx = torch.randperm(2 * rows + 3, device="cuda", generator=g)[:rows].int()
    d_idx = torch.randperm(rows + 5, device="cuda", generator=g)[:rows].int()
    nat.check(nat.load().vlc_gather_rows(dst.data_ptr(), d_idx.data_ptr(), src.data_ptr(), s_idx.data_ptr(), rows,
                                         width * 2, _stream()), "gather_rows")
    torch.cuda.synchronize()
    want = torch.zeros_like(dst)
    want[d_idx.long()] = src[s_idx.long()]
    assert torch.equal(dst, want)
