"""Microbenchmark of vlc_attn_paged at the C3 layer shape (hd 128, 28 heads, 4128 keys, 236 queries).
  python tools/attn_paged_bench.py [store_every ...]   random query positions, every k-th chunk from the store
  python tools/attn_paged_bench.py c3 [trace]           the C3 reuse layout (16 + 4 x 1024 + 16 tokens, the
                                                          first 51 tokens of each image and all text recomputed,
                                                          every other image chunk read from the store); with
                                                          `trace`, per-CTA phase stamps of one launch
Timing only (CUDA events over 50 launches, 256 MB L2 flush between launches)."""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
from paper_2512_12977_b200 import _native as nat  # noqa: E402
if os.environ.get("VLC_LIB_VARIANT"):          # experiment builds (tools/build_variant.py)
    nat.LIB_PATH = os.environ["VLC_LIB_VARIANT"]
from paper_2512_12977_b200.layout import attention_work, tiles_needed  # noqa: E402


def c3_case(hd=128, heads=28, T=1024, imgs=4, keep=51, pre=16, post=16, seed=0):
    kv = heads * hd
    n = pre + imgs * T + post
    g = torch.Generator(device="cuda").manual_seed(seed)
    kc = torch.randn(1, n + 64, kv, device="cuda", generator=g).bfloat16()
    vc = torch.randn(1, n + 64, kv, device="cuda", generator=g).bfloat16()
    npages = imgs * T // 64 + 4
    kpool = torch.randn(npages * 64, kv, device="cuda", generator=g).bfloat16()
    vpool = torch.randn(npages * 64, kv, device="cuda", generator=g).bfloat16()
    ptab = torch.randperm(npages, device="cuda", generator=g).int()
    ang = np.arange(n + 64, dtype=np.float32)[:, None] * (10000.0 ** (-np.arange(hd // 2, dtype=np.float32) * 2 / hd))
    cos = torch.from_numpy(np.cos(ang)).cuda()
    sin = torch.from_numpy(np.sin(ang)).cuda()
    chunks = [[c, min(64, pre - c), c, -1] for c in range(0, pre, 64)]
    qpos = list(range(pre))
    for m in range(imgs):
        s0 = pre + m * T
        qpos += list(range(s0, s0 + keep))
        for t0 in range(0, T, 64):
            if t0 >= keep:     # K rotated at its cached position (start 8): shift D = s0 - 8
                chunks.append([s0 + t0, 64 | ((s0 - 8) << 8), m * (T // 64) + t0 // 64, 0])
            else:
                chunks.append([s0 + t0, 64, s0 + t0, -1])
    s1 = pre + imgs * T
    chunks += [[c, min(64, n - c), c, -1] for c in range(s1, n, 64)]
    qpos += list(range(s1, n))
    if len(chunks) % 2:
        chunks.append([chunks[-1][0] + 64, 0, chunks[-1][2], chunks[-1][3]])
    chunks = np.array(chunks, np.int32)
    nq = len(qpos)
    qp = np.array(qpos, np.int32)
    q = torch.randn(nq + 256, kv, device="cuda", generator=g).bfloat16()
    out = torch.zeros(nq, kv, device="cuda", dtype=torch.bfloat16)
    items, groups = attention_work([(0, 0, nq)], qp, lambda r, p: tiles_needed(chunks, p), [0], heads)
    keepb = dict(it=torch.from_numpy(items).cuda(), ch=torch.from_numpy(chunks).cuda(),
                 ws_o=torch.zeros(max(groups, 1) * 8 * 256 * hd, device="cuda"),
                 ws_ml=torch.zeros(max(groups, 1) * 8 * 256 * 2, device="cuda"),
                 cnt=torch.zeros(4096, dtype=torch.int32, device="cuda"), kc=kc, vc=vc, kpool=kpool, vpool=vpool,
                 ptab=ptab, cos=cos, sin=sin, q=q, qpos=torch.from_numpy(qp).cuda(),
                 rowof=torch.arange(nq, dtype=torch.int32, device="cuda"), items=items)
    a = nat.AttnPagedArgs(q=q.data_ptr(), q_rows_cap=q.shape[0], kc=kc.data_ptr(), vc=vc.data_ptr(), layers_cap=1,
                          kv_rows_cap=n + 64, layer=0, pool_k=kpool.data_ptr(), pool_v=vpool.data_ptr(),
                          pool_rows=kpool.shape[0], page_table=ptab.data_ptr(), page_rows=64,
                          cos_tab=cos.data_ptr(), sin_tab=sin.data_ptr(), tab_ld=hd // 2, kv=kv, heads=heads,
                          head_dim=hd, chunks=keepb["ch"].data_ptr(), items=keepb["it"].data_ptr(),
                          n_items=len(items), qpos=keepb["qpos"].data_ptr(), rowof=keepb["rowof"].data_ptr(),
                          out=out.data_ptr(), ldo=kv, pk_rows=0, pk_kb=0, ws_o=keepb["ws_o"].data_ptr(),
                          ws_ml=keepb["ws_ml"].data_ptr(), ws_slots=groups, counters=keepb["cnt"].data_ptr(),
                          scale_log2=math.log2(math.e) / math.sqrt(hd))
    return a, out, keepb


def time_it(a, label, reps=50):
    lib = nat.load()
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(5):
        nat.check(lib.vlc_attn_paged(a, s), "attn")
    torch.cuda.synchronize()
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
    print(f"{label}: items={a.n_items} slots={a.ws_slots}: p50 {ts[len(ts) // 2]:.1f} us min {ts[0]:.1f} us",
          flush=True)


def trace(a, items):
    tr = torch.zeros(a.n_items * 64, dtype=torch.int64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")
    flush.zero_()
    a.trace = tr.data_ptr()
    nat.check(nat.load().vlc_attn_paged(a, torch.cuda.current_stream().cuda_stream), "attn")
    torch.cuda.synchronize()
    a.trace = None
    d = tr.view(-1, 64).cpu().numpy().astype(np.float64)
    t0 = d[:, 0][d[:, 0] > 0].min()
    rel = np.where(d > 0, (d - t0) / 1e3, np.nan)
    nt = items[:, 5] - items[:, 4]
    it = []
    for i in range(len(d)):
        k = min(int(nt[i]), 40)
        if k >= 2:
            it.append((rel[i, 2 + k - 1] - rel[i, 2]) / (k - 1))
    names = {0: "start", 1: "q_landed", 2: "S(0) ready", 50: "loop_end", 51: "out/partial", 52: "merge_go",
             53: "merge_end"}
    for s, nm in names.items():
        col = rel[:, s]
        col = col[~np.isnan(col)]
        if len(col):
            print(f"  {nm:12s} min {col.min():6.2f} med {np.median(col):6.2f} max {col.max():6.2f}")
    for lab, base in (("S ready", 2), ("K landed", 18), ("K rotated", 34)):
        k = int(np.median(nt))
        row = np.nanmedian(rel[nt >= k, base:base + min(k, 16)], axis=0)
        print(f"  {lab:10s} per tile (median CTA): " + " ".join(f"{x:5.2f}" for x in row))
    # per split part (items[:, 7] = part << 8 | nsplit): when each part starts, ends its loop, posts its partial
    part, nsp = items[:, 7] >> 8, items[:, 7] & 0xFF
    for ns_ in sorted(set(nsp.tolist())):
        for p_ in range(ns_):
            sel = (nsp == ns_) & (part == p_)
            if sel.any():
                print(f"  nsplit {ns_} part {p_}: n={sel.sum():3d} tiles {np.median(nt[sel]):4.1f}  S(0) "
                      f"{np.nanmedian(rel[sel, 2]):5.2f}  loop_end {np.nanmedian(rel[sel, 50]):5.2f}  partial "
                      f"{np.nanmedian(rel[sel, 51]):5.2f} (max {np.nanmax(rel[sel, 51]):5.2f})")
    print(f"  per-tile     med {np.median(it):.3f} us  min {np.min(it):.3f} max {np.max(it):.3f}  "
          f"tiles/CTA med {np.median(nt):.0f} max {nt.max()}  total {nt.sum()}")


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "c3":
        a, out, kb = c3_case()
        time_it(a, "C3 layout")
        if "trace" in args:
            trace(a, kb["items"])
    else:
        from test_kernels_gpu import _paged_case  # noqa: E402
        for se in ([int(x) for x in args] or (0, 1)):
            a, out, ref, keep = _paged_case(nat, 128, 28, 4128, 236, True, se, 7)
            time_it(a, f"store_every={se}")
