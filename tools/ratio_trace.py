"""Per-kernel device time of one C3 reuse prefill at several static recompute ratios (events around each
launch, eager, the stream held on a device-side spin while the host issues; L2 flushed before each pass).
  python tools/ratio_trace.py 0.05 0.06"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2512_12977_b200 as P  # noqa: E402
from paper_2512_12977_b200.engine import _runner, prefill_with_reuse  # noqa: E402
from paper_2512_12977_b200.toydata import make_images, prompt_ids  # noqa: E402

cfg = P.ModelConfig(**bench.CONFIGS["C3"], seed=0)
T, V, L = cfg.tokens_per_image, cfg.vocab_size, cfg.num_layers
model = P.ToyVLM.device_random(cfg, seed=0)
runner = _runner(model)
store = P.CacheStore()
images = make_images(4, cfg.image_side, 1)
P.fill_store(model, store, images, prompt_ids(V, 8, 11))
text = prompt_ids(V, 32, 12)
seq = P.make_sequence(text[:16], 4, T, text[16:])
hashes = [P.hash_image(px) for px in images]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for r in [float(a) for a in sys.argv[1:]] or [0.05, 0.06]:
    req = P.ReuseRequest(seq, hashes, P.plan_static(r, L))
    prefill_with_reuse(model, req, store).last_logits()
    agg = {}
    n = 3
    for _ in range(n):
        runner.tracer = []
        flush.add_(1)
        torch.cuda._sleep(int(40e6))
        prefill_with_reuse(model, req, store)
        torch.cuda.synchronize()
        for name, e0, e1, nb, fl in runner.tracer:
            a = agg.setdefault(name, [0.0, 0])
            a[0] += e0.elapsed_time(e1)
            a[1] += 1
    runner.tracer = None
    tot = sum(v[0] for v in agg.values()) / n
    print(f"ratio {r}: c0 = {req.plan.ratios[0] * 4 * T + 32:.0f} rows, sum of kernels {tot:.3f} ms")
    for name, (ms, cnt) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"   {name:14s} {ms / n:7.3f} ms  {cnt // n:3d} launches  {1e3 * ms / cnt:7.2f} us/launch")
