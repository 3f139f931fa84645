"""Standalone timing + phase breakdown of the ping-pong attention kernel at the C3 shape."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_12977_b200 import _native as N  # noqa: E402
from paper_2512_12977_b200.layout import attention_work_pp  # noqa: E402

lib = N.load()


ONE = False   # single-query-tile items (attention_work_one) for the tuning-15 = 30/31 kernels


def setup(hd=128, heads=28, nkeys=4128, nq=236, max_ctas=148):
    kv = heads * hd
    g = torch.Generator(device="cuda").manual_seed(1)
    L = 4
    kc = torch.randn(L, nkeys + 64, kv, device="cuda", generator=g).bfloat16()
    vc = torch.randn(L, nkeys + 64, kv, device="cuda", generator=g).bfloat16()
    qpos = np.sort(np.random.default_rng(0).permutation(nkeys)[:nq]).astype(np.int32)
    qpos[-1] = nkeys - 1
    qp = torch.from_numpy(qpos).cuda()
    q = torch.randn(512, kv, device="cuda", generator=g).bfloat16()
    rowof = torch.arange(nq, dtype=torch.int32, device="cuda")
    out = torch.zeros(nq, kv, device="cuda", dtype=torch.bfloat16)
    from paper_2512_12977_b200.layout import attention_work_one
    work = attention_work_one if ONE else attention_work_pp
    it9, groups = work([(0, 0, nq)], qpos, np.array([nkeys]), heads, max_ctas)
    it = torch.from_numpy(np.ascontiguousarray(it9[:, :8])).cuda()
    ws_o = torch.zeros(max(groups, 1) * 8 * 256 * hd, device="cuda")
    ws_ml = torch.zeros(max(groups, 1) * 8 * 256 * 2, device="cuda")
    cnt = torch.zeros(4096, dtype=torch.int32, device="cuda")
    a = N.AttnArgs(q=q.data_ptr(), q_rows_cap=q.shape[0], kc=kc.data_ptr(), vc=vc.data_ptr(), layers_cap=L,
                   kv_rows_cap=nkeys + 64, layer=1, kv=kv, heads=heads, head_dim=hd, items=it.data_ptr(),
                   n_items=it.shape[0], qpos=qp.data_ptr(), rowof=rowof.data_ptr(), out=out.data_ptr(), ldo=kv,
                   ws_o=ws_o.data_ptr(), ws_ml=ws_ml.data_ptr(), ws_slots=groups, comb=0, n_comb=0,
                   scale_log2=math.log2(math.e) / math.sqrt(hd), counters=cnt.data_ptr())
    keep = (kc, vc, q, qp, rowof, out, it, ws_o, ws_ml, cnt)
    return a, keep, it.shape[0]


def run(max_ctas):
    a, keep, n = setup(max_ctas=max_ctas)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        N.check(lib.vlc_attn_pp(a, s), "pp")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20):
        N.check(lib.vlc_attn_pp(a, s), "pp")
    e1.record()
    e1.synchronize()
    print(f"max_ctas={max_ctas}: {n} CTAs, {e0.elapsed_time(e1) * 1e3 / 20:.1f} us/launch", flush=True)
    dbg = torch.zeros(n * 8, dtype=torch.int64, device="cuda")
    lib.vlc_set_debug_buffer(dbg.data_ptr())
    N.check(lib.vlc_attn_pp(a, s), "pp")
    torch.cuda.synchronize()
    lib.vlc_set_debug_buffer(None)
    d = dbg.view(n, 8).cpu().numpy().astype("float64")
    t0 = d[:, 0].min()
    d = np.where(d > 0, (d - t0) / 1e3, np.nan)
    for i, nm in enumerate(["start", "q_loaded", "mma_done", "softmaxA_done", "softmaxB_done", "merge_go", "end"]):
        col = d[:, i]
        col = col[~np.isnan(col)]
        if len(col):
            print(f"   {nm:14s} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f}")


def phases(var=11):
    """VAR 0x400 (tuning 15 = 11): per-phase clock64 cycles summed over all CTAs (one thread per
    query tile for the softmax phases, the MMA thread for its phases)."""
    global ONE
    ONE = var in (30, 31, 32, 33, 34, 35, 36, 37, 38, 39)
    lib.vlc_set_tuning(15, var)
    a, keep, n = setup(max_ctas=148)
    s = torch.cuda.current_stream().cuda_stream
    N.check(lib.vlc_attn_pp(a, s), "pp")
    buf = torch.zeros(512, dtype=torch.int64, device="cuda")
    lib.vlc_set_trace_buffer(buf.data_ptr())
    N.check(lib.vlc_attn_pp(a, s), "pp")
    torch.cuda.synchronize()
    lib.vlc_set_trace_buffer(None)
    b = buf.cpu().numpy()[256:]
    names = ["wait_s", "tmem_ld", "mask_max", "rescale", "exp_pack", "st_arrive"]
    for x in range(2):
        it = max(int(b[x * 8 + 7]), 1)
        print(f"softmax tile {'AB'[x]} ({it} iterations): " +
              " ".join(f"{nm}={b[x * 8 + k] / it:.0f}" for k, nm in enumerate(names)), flush=True)
    for x in range(2):
        print(f"mma tile {'AB'[x]}: " + " ".join(f"{nm}={b[16 + x * 4 + k] / 140:.0f}"
                                              for k, nm in enumerate(["wait_p", "issue_pv", "wait_kv_issue_s"])))
    lib.vlc_set_tuning(15, 0)


if __name__ == "__main__":
  if len(sys.argv) > 1 and sys.argv[1] == "phases":
    phases(int(sys.argv[2]) if len(sys.argv) > 2 else 11)
    sys.exit(0)
  if len(sys.argv) > 1 and sys.argv[1] == "vars":   # softmax variants of the 128-key kernel (key 15)
    for v in [int(x) for x in sys.argv[2:]]:
      ONE = v in (30, 31, 32, 33, 34, 35, 36, 37, 38, 39)
      lib.vlc_set_tuning(15, v)
      print(f"== softmax variant {v}", flush=True)
      run(148)
    sys.exit(0)
  for kt in (64, 128):
    lib.vlc_set_tuning(12, kt)
    print(f"== key tile {kt}", flush=True)
    for mc in (148, 28):
      run(mc)
