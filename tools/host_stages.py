"""Host-side cost of prefill_with_reuse by stage (resolve / layout / metadata pack+upload / graph replay)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2512_12977_b200 as P  # noqa: E402
from paper_2512_12977_b200 import engine as E  # noqa: E402
from paper_2512_12977_b200 import runtime as RT  # noqa: E402
from paper_2512_12977_b200.toydata import make_images, prompt_ids  # noqa: E402

cfg = P.ModelConfig(**bench.CONFIGS["C3"], seed=0)
model = P.ToyVLM.device_random(cfg, 0)
store = P.CacheStore()
imgs = make_images(4, cfg.image_side, 1)
P.fill_store(model, store, imgs, prompt_ids(cfg.vocab_size, 8, 11))
text = prompt_ids(cfg.vocab_size, 32, 12)
seq = P.make_sequence(text[:16], 4, cfg.tokens_per_image, text[16:])
req = P.ReuseRequest(seq, [P.hash_image(p) for p in imgs], P.plan_static(0.05, cfg.num_layers))
for _ in range(3):
    P.prefill_with_reuse(model, req, store).last_logits()
torch.cuda.synchronize()

acc = {}


def wrap(obj, name, key, static=False):
    f = getattr(obj, name)

    def g(*a, **k):
        t0 = time.perf_counter()
        r = f(*a, **k)
        acc[key] = acc.get(key, 0.0) + time.perf_counter() - t0
        return r
    setattr(obj, name, staticmethod(g) if static else g)


wrap(E, "_resolve", "resolve")
wrap(E, "_layout", "layout")
wrap(RT.IntPack, "upload", "upload")
wrap(RT.Runner, "_pack", "pack", static=True)
wrap(torch.cuda.CUDAGraph, "replay", "graph_replay")
wrap(RT.Runner, "_pick_set", "pick_set")
N = 20
t0 = time.perf_counter()
for _ in range(N):
    r = P.prefill_with_reuse(model, req, store)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"total host per call {1e3 * (t1 - t0) / N:.3f} ms")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"  {k:14s} {1e3 * v / N:.3f} ms")
