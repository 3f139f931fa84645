"""GEMM microbenchmark: graph-replayed launches timed with CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_12977_b200 import _native as N  # noqa: E402

lib = N.load()
ws = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
cnt = torch.zeros(1 << 16, dtype=torch.int32, device="cuda")


def run(n, k, m, splits, kind=N.EPI_BF16, stages=0, reps=20):
    W = torch.randn(n, k, device="cuda").bfloat16()
    X = torch.randn(max(256, m + 256), k, device="cuda").bfloat16()
    out = torch.zeros(m + 256, n, device="cuda", dtype=torch.float32)
    e = N.Epilogue()
    e.kind, e.n_valid, e.m_tokens, e.out, e.ldo = kind, n, m, out.data_ptr(), n
    lib.vlc_set_tuning(1, stages)
    s = torch.cuda.current_stream().cuda_stream

    def go():
        N.check(lib.vlc_gemm_bf16(W.data_ptr(), n, k, X.data_ptr(), X.shape[0], m, e, splits, ws.data_ptr(),
                                  ws.numel() * 4, cnt.data_ptr(), torch.cuda.current_stream().cuda_stream), "g")
    go()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            go()
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
    print(f"N={n:6d} K={k:5d} M={m:4d} splits={splits} kind={kind} stages={stages}: {us:8.2f} us  "
          f"{gbs:7.1f} GB/s  {tf:7.1f} TF/s", flush=True)


if __name__ == "__main__":
    for m in (16, 112, 240):
        for n, k in ((14336, 3584), (10752, 3584), (3584, 3584), (3584, 7168)):
            run(n, k, m, 0, kind=N.EPI_RESID if n == 3584 else N.EPI_BF16)
    for st in (3, 4):
        run(14336, 3584, 240, 0, stages=st)
    run(152064, 3584, 236, 0, kind=N.EPI_F32)
    run(14336, 3584, 4128, 0)
    run(10752, 3584, 4128, 0)
    run(3584, 7168, 4128, 0, kind=N.EPI_RESID)
