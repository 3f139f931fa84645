"""CTA-pair GEMM (vlc_set_tuning key 10) vs torch, each case in a subprocess with a timeout;
then timing of the C3 shapes with the pair kernel on/off."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def case(n, k, m, kind):
    import torch
    from paper_2512_12977_b200 import _native as N
    lib = N.load()
    lib.vlc_set_tuning(10, 32)
    g = torch.Generator(device="cuda").manual_seed(n + m)
    W = torch.randn(n, k, device="cuda", generator=g).bfloat16()
    X = torch.randn(max(256, m), k, device="cuda", generator=g).bfloat16()
    R = N.row_tile(m)
    Wp, Xp = N.pack(W, 128), N.pack(X[:m], R, rows_cap=-(-m // R) * R)
    ws = torch.zeros(64 << 20, dtype=torch.float32, device="cuda")
    cnt = torch.zeros(4096, dtype=torch.int32, device="cuda")
    ref = X[:m].float() @ W.float().t()
    e = N.Epilogue()
    if kind == "f32":
        out = torch.full((m, n), float("nan"), device="cuda")
        e.kind, e.n_valid, e.m_tokens, e.out, e.ldo = N.EPI_F32, n, m, out.data_ptr(), n
    else:
        out = torch.zeros(N.packed_numel(m, n // 2, R), device="cuda", dtype=torch.bfloat16)
        e.kind, e.n_valid, e.m_tokens, e.out, e.ldo, e.pk_rows, e.pk_kb = N.EPI_SWIGLU, n, m, out.data_ptr(), n // 2, R, -(-(n // 2) // 128)
    N.check(lib.vlc_gemm_bf16(Wp.data_ptr(), n, k, Xp.data_ptr(), -(-m // R) * R, m, e, 0, ws.data_ptr(),
                              ws.numel() * 4, cnt.data_ptr(), torch.cuda.current_stream().cuda_stream), "g")
    torch.cuda.synchronize()
    if kind == "f32":
        err = ((out - ref).abs().max() / ref.abs().max()).item()
    else:
        h = N.unpack(out, m, n // 2, R).float()
        gt, up = ref[:, 0::2], ref[:, 1::2]
        r2 = gt / (1 + torch.exp(-gt)) * up
        err = ((h - r2).abs().max() / r2.abs().max()).item()
    print(f"err={err:.2e}", flush=True)


def timing():
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import gemm_bench as gb
    N = gb.N
    for mode in (0, 96):
        gb.lib.vlc_set_tuning(10, mode)
        print(f"-- pair threshold {mode}", flush=True)
        for n, k, kind in ((10752, 3584, N.EPI_BF16), (14336, 3584, N.EPI_BF16), (152064, 3584, N.EPI_F32)):
            gb.run(n, k, 236, 0, kind=kind)
    gb.lib.vlc_set_tuning(10, 0)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "case":
        case(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5])
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "timing":
        timing()
        sys.exit(0)
    ok = True
    for c in ((256, 128, 32, "f32"), (512, 256, 100, "f32"), (256, 1024, 240, "f32"), (10752, 3584, 236, "f32"),
              (1024, 512, 236, "swiglu"), (2048, 256, 600, "f32"), (512, 384, 48, "f32")):
        try:
            r = subprocess.run([sys.executable, __file__, "case", *map(str, c)], capture_output=True, text=True,
                               timeout=60)
            res = r.stdout.strip() or r.stderr.strip()[-400:]
        except subprocess.TimeoutExpired:
            res, ok = "HANG", False
        print(c, res, flush=True)
        if "err=" not in res or float(res.split("err=")[1]) > 2e-2:
            ok = False
    if ok:
        subprocess.run([sys.executable, __file__, "timing"], timeout=300)
