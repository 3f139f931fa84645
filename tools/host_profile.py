"""Host-side cost of one prefill_with_reuse call at the bench workload (cProfile, no sync)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2512_12977_b200 as P  # noqa: E402
from paper_2512_12977_b200.toydata import make_images, prompt_ids  # noqa: E402

wl = bench.WORKLOADS[os.environ.get("WL", "C3")]
cfg = P.ModelConfig(**bench.CONFIGS[wl["cfg"]], seed=0)
model = P.ToyVLM.device_random(cfg, 0)
store = P.CacheStore()
imgs = make_images(wl["images"], cfg.image_side, 1)
P.fill_store(model, store, imgs, prompt_ids(cfg.vocab_size, 8, 11))
text = prompt_ids(cfg.vocab_size, 32, 12)
seq = P.make_sequence(text[:16], wl["images"], cfg.tokens_per_image, text[16:])
req = P.ReuseRequest(seq, [P.hash_image(p) for p in imgs], P.plan_static(wl["ratio"], cfg.num_layers))
for _ in range(3):
    P.prefill_with_reuse(model, req, store).last_logits()
torch.cuda.synchronize()
for _ in range(5):
    t0 = time.perf_counter()
    r = P.prefill_with_reuse(model, req, store)
    t1 = time.perf_counter()
    r.last_logits()
    t2 = time.perf_counter()
    print(f"issue {1e3 * (t1 - t0):.3f} ms  e2e {1e3 * (t2 - t0):.3f} ms  device {1e3 * r.metrics.compute_seconds:.3f} ms",
          flush=True)
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    P.prefill_with_reuse(model, req, store).last_logits()
pr.disable()
pstats.Stats(pr).sort_stats(os.environ.get("SORT", "cumulative")).print_stats(35)
