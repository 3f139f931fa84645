"""GEMM microbenchmark: graph-replayed launches timed with CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_12977_b200 import _native as N  # noqa: E402
if os.environ.get("VLC_LIB_VARIANT"):          # experiment builds (tools/build_variant.py)
    N.LIB_PATH = os.environ["VLC_LIB_VARIANT"]

lib = N.load()
ws = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
cnt = torch.zeros(1 << 16, dtype=torch.int32, device="cuda")




def run(n, k, m, splits, kind=N.EPI_BF16, stages=0, reps=20, coop=1, packed=False, mode=0, red=False):
    nw = max(2, min(8, (1 << 30) // (n * k * 2)))   # rotate > L2 worth of weights
    Ws = [N.pack(torch.randn(n, k, device="cuda").bfloat16(), 128) for _ in range(nw)]
    R = N.row_tile(m, n)
    fn = lib.vlc_gemm_bf16
    X = N.pack(torch.randn(m, k, device="cuda").bfloat16(), R, rows_cap=-(-m // R) * R)
    out = torch.zeros(m + 256, n, device="cuda", dtype=torch.float32)
    e = N.Epilogue()
    e.kind, e.n_valid, e.m_tokens, e.out, e.ldo = kind, n, m, out.data_ptr(), n
    lib.vlc_set_tuning(1, stages)
    lib.vlc_set_tuning(2, coop)
    s = torch.cuda.current_stream().cuda_stream

    def go(W):
        N.check(fn(W.data_ptr(), n, k, X.data_ptr(), -(-m // R) * R, m, e, splits, ws.data_ptr(),
                   ws.numel() * 4, cnt.data_ptr(), torch.cuda.current_stream().cuda_stream), "g")
    go(Ws[0])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for r in range(reps):
            go(Ws[r % nw])
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    g.replay()
    e1.record()
    e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    gbs = (n * k * 2 + m * k * 2) / us / 1e3
    tf = 2 * n * k * m / us / 1e6
    print(f"N={n:6d} K={k:5d} M={m:4d} ctas={splits} pk={int(packed)} mode={mode} st={stages}: {us:8.2f} us  "
          f"{gbs:7.1f} GB/s  {tf:7.1f} TF/s", flush=True)


def phases(n, k, m, ctas, kind=None):
    """Per-CTA phase timestamps of one launch (DRAM-cold weights)."""
    R = N.row_tile(m, n)
    W = N.pack(torch.randn(n, k, device="cuda").bfloat16(), 128)
    X = N.pack(torch.randn(m, k, device="cuda").bfloat16(), R, rows_cap=-(-m // R) * R)
    out = torch.zeros(m + 256, n, device="cuda", dtype=torch.float32)
    e = N.Epilogue()
    e.kind, e.n_valid, e.m_tokens, e.out, e.ldo = N.EPI_BF16 if kind in (None, "pair") else kind, n, m, out.data_ptr(), n
    dbg = torch.zeros(320 * 8, dtype=torch.int64, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for it in range(3):
        flush.add_(1)
        lib.vlc_set_debug_buffer(dbg.data_ptr() if it == 2 else None)
        N.check(lib.vlc_gemm_bf16(W.data_ptr(), n, k, X.data_ptr(), -(-m // R) * R, m, e, ctas, ws.data_ptr(),
                                  ws.numel() * 4, cnt.data_ptr(), torch.cuda.current_stream().cuda_stream), "g")
        torch.cuda.synchronize()
    lib.vlc_set_debug_buffer(None)
    d = dbg.view(320, 8)[:160].cpu().numpy().astype("float64")
    g = d[:, 0] > 0
    d = d[g]
    t0 = d[:, 0].min()
    d = np.where(d > 0, (d - t0) / 1e3, -1.0)
    names = (["start", "prod_go", "prod_done", "acc_full(last)", "owner_go", "acc_full(seg0)", "epi_end", "exit"]
             if kind == "pair" else
             ["start", "prod_go", "prod_done", "acc_full(last)", "partials_done", "fixup_go", "epi_end", "exit"])
    print(f"--- N={n} K={k} M={m} ctas={ctas}: {len(d)} CTAs; us rel. to first start")
    for i, nm in enumerate(names):
        col = d[:, i]
        col = col[col >= 0]
        if not len(col):
            continue
        print(f"  {nm:16s} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f}")


if __name__ == "__main__":
    import numpy as np  # noqa: F811
    mode = sys.argv[1] if len(sys.argv) > 1 else "sweep"
    if mode == "pairphases":      # single-CTA vs CTA-pair kernel, QKV / GU shapes at c = 236
        for pair in (0, 32):
            lib.vlc_set_tuning(10, pair)
            print(f"=== pair threshold {pair}")
            for (n, kk, m, c) in ((10752, 3584, 236, 0), (14336, 3584, 236, 0)):
                phases(n, kk, m, c, kind="pair" if pair else None)
        lib.vlc_set_tuning(10, 0)
    if mode == "pairtile":        # CTA-pair kernel with one 256-row tile per pair (no stream-K) vs single-CTA
        for pair in (0, -16, 0, -16):
            lib.vlc_set_tuning(10, pair)
            print(f"=== pair {pair}", flush=True)
            for (n, kk, m) in ((10752, 3584, 236), (14336, 3584, 236)):
                c = n // 128 if pair else 0
                run(n, kk, m, c)
                if pair:
                    phases(n, kk, m, c, kind="pair")
        lib.vlc_set_tuning(10, 0)
    if mode == "decoupled":       # one-tile GEMMs with decoupled weight / activation rings (key 18)
        for dec in (2, 12, 13, 14, 2, 13):
            lib.vlc_set_tuning(18, dec)
            print(f"-- decoupled {dec}", flush=True)
            for (n, kk, m) in ((10752, 3584, 236), (14336, 3584, 236), (14336, 3584, 112)):
                run(n, kk, m, 0)
        lib.vlc_set_tuning(18, 0)
        lib.vlc_set_tuning(18, 1)
        for (n, kk, m) in ((10752, 3584, 236),):
            phases(n, kk, m, 0)
        lib.vlc_set_tuning(18, 0)
    if mode == "clock":           # SM clock during the decoupled QKV / GU mainloop (cycles / ns)
        for (n, kk, m) in ((10752, 3584, 236), (14336, 3584, 236)):
            R = N.row_tile(m, n)
            W = N.pack(torch.randn(n, kk, device="cuda").bfloat16(), 128)
            X = N.pack(torch.randn(m, kk, device="cuda").bfloat16(), R, rows_cap=-(-m // R) * R)
            out = torch.zeros(m + 256, n, device="cuda", dtype=torch.float32)
            e = N.Epilogue()
            e.kind, e.n_valid, e.m_tokens, e.out, e.ldo = N.EPI_BF16, n, m, out.data_ptr(), n
            dbg = torch.zeros(320 * 8, dtype=torch.int64, device="cuda")
            for it in range(4):
                lib.vlc_set_debug_buffer(dbg.data_ptr() if it == 3 else None)
                N.check(lib.vlc_gemm_bf16(W.data_ptr(), n, kk, X.data_ptr(), -(-m // R) * R, m, e, 0, ws.data_ptr(),
                                          ws.numel() * 4, cnt.data_ptr(), torch.cuda.current_stream().cuda_stream), "g")
                torch.cuda.synchronize()
            lib.vlc_set_debug_buffer(None)
            dd = dbg.view(320, 8).cpu().numpy().astype("float64")
            cyc = dd[160:, 0]
            d = dd[:160]
            ok = cyc > 0
            d, cyc = d[ok], cyc[ok]
            mhz = cyc / (d[:, 6] - d[:, 5]) * 1e3
            print(f"N={n}: mainloop {np.median(d[:, 6] - d[:, 5]) / 1e3:.2f} us, {np.median(cyc):.0f} cycles, "
                  f"SM clock {np.median(mhz):.0f} MHz (min {mhz.min():.0f})", flush=True)
    if mode == "wide":            # 256-row tiles (H = 2) under stream-K over every SM (fix-up path)
        for wide, um in ((1, 64), (2, 64), (1, 1000), (2, 1000)):
            lib.vlc_set_tuning(7, wide)
            lib.vlc_set_tuning(9, um)
            print(f"-- wide {wide} unsplit_min {um}", flush=True)
            for (n, kk, m) in ((10752, 3584, 236), (14336, 3584, 236)):
                run(n, kk, m, 0)
                phases(n, kk, m, 0)
        lib.vlc_set_tuning(7, 1)
        lib.vlc_set_tuning(9, 64)
    if mode == "head":            # LM head: CTA pair (9 waves, last one holds 2 of 594 tiles) vs stream-K
        for pair in (96, 0, 96):
            lib.vlc_set_tuning(10, pair)
            print(f"-- pair {pair}", flush=True)
            run(152064, 3584, 236, 0, kind=N.EPI_F32, reps=6)
        lib.vlc_set_tuning(10, 0)
    if mode == "aligned":         # tile-aligned split-K: divisor splits (key 17 = 1) vs any split (2)
        for al in (1, 2, 1, 2):
            lib.vlc_set_tuning(17, al)
            print(f"-- aligned {al}", flush=True)
            for (n, kk, m) in ((3584, 3584, 236), (3584, 7168, 236)):
                run(n, kk, m, 0, kind=N.EPI_RESID)
        lib.vlc_set_tuning(17, 1)
    if mode == "residctas":       # stream-K RESID GEMMs at fewer CTAs (fewer split segments -> less red.add)
        for c in (148, 128, 112, 96, 74):
            for (n, kk, m) in ((3584, 3584, 236), (3584, 7168, 236)):
                run(n, kk, m, c, kind=N.EPI_RESID)
    if mode == "residphases":     # the stream-K O / down projections (red.add into an fp32 residual)
        for (n, kk, m) in ((3584, 3584, 236), (3584, 7168, 236)):
            run(n, kk, m, 0, kind=N.EPI_RESID)
            phases(n, kk, m, 0, kind=N.EPI_RESID)
    if mode == "phases":
        for (n, kk, m, c) in ((14336, 3584, 240, 112), (14336, 3584, 16, 112), (3584, 3584, 240, 148),
                              (14336, 3584, 240, 148)):
            phases(n, kk, m, c)
    elif mode == "modes":
        for (n, k, m, c) in ((3584, 3584, 16, 28), (3584, 3584, 240, 28), (14336, 3584, 240, 112),
                             (14336, 3584, 128, 112), (14336, 3584, 16, 112), (10752, 3584, 240, 84),
                             (14336, 3584, 240, 148), (10752, 3584, 240, 148), (3584, 3584, 240, 148),
                             (3584, 7168, 240, 148), (152064, 3584, 236, 0), (14336, 3584, 4128, 0)):
            run(n, k, m, c)
        lib.vlc_set_tuning(3, 0)
    elif mode == "packed":
        for (n, k) in ((14336, 3584), (10752, 3584), (3584, 3584), (3584, 7168)):
            for m in (16, 240):
                for pk in (False, True):
                    run(n, k, m, n // 128, packed=pk)
        for pk in (False, True):
            run(3584, 3584, 16, 148, packed=pk)
            run(14336, 3584, 16, 112, packed=pk, stages=12)
    elif mode == "ctas":
        for (n, k) in ((14336, 3584), (10752, 3584), (3584, 3584), (3584, 7168)):
            for m in (16, 240):
                for ctas in sorted({n // 128, 74, 148}):
                    run(n, k, m, ctas)
    else:
        for m in (16, 112, 240):
            for n, k in ((14336, 3584), (10752, 3584), (3584, 3584), (3584, 7168)):
                run(n, k, m, 0, kind=N.EPI_RESID if n == 3584 else N.EPI_BF16)
        run(152064, 3584, 236, 0, kind=N.EPI_F32)
        run(14336, 3584, 4128, 0)
