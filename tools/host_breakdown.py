"""Wall-clock breakdown of the host side of prefill_with_reuse (no sync inside): monkeypatched
perf_counter checkpoints around the engine / runner stages."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2512_12977_b200 as P  # noqa: E402
from paper_2512_12977_b200 import engine as E  # noqa: E402
from paper_2512_12977_b200 import layout as LY  # noqa: E402
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


wrap(E, "_resolve", "engine._resolve")
wrap(E, "_layout", "engine._layout")
wrap(LY, "structure_of", "layout.structure_of")
wrap(E, "_merged_kv_loader", "engine._merged_kv_loader")
wrap(RT.Runner, "prefill", "runner.prefill")
wrap(RT.Runner, "_pack", "runner._pack", static=True)
wrap(RT.Runner, "_pick_set", "runner._pick_set")
wrap(RT.IntPack, "upload_segments", "IntPack.upload_segments")
wrap(torch.cuda.CUDAGraph, "replay", "graph.replay")
wrap(RT.Workspace, "get", "Workspace.get")
wrap(E, "_runner", "engine._runner")
wrap(E, "prefill_batch_with_reuse", "engine.prefill_batch_with_reuse")
N = 50
for _ in range(N):
    r = P.prefill_with_reuse(model, req, store)
    torch.cuda.synchronize()
acc.clear()
tot = 0.0
for _ in range(N):
    t0 = time.perf_counter()
    r = P.prefill_with_reuse(model, req, store)
    tot += time.perf_counter() - t0
    torch.cuda.synchronize()
print(f"prefill_with_reuse host {1e3 * tot / N:.3f} ms per call")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"  {k:32s} {1e3 * v / N:.3f} ms")
# end to end as the bench measures it: API call -> last-row logits on the host
e2e, host = [], []
for _ in range(N):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = P.prefill_with_reuse(model, req, store)
    t1 = time.perf_counter()
    r.last_logits()
    t2 = time.perf_counter()
    e2e.append(t2 - t0)
    host.append(t1 - t0)
ev = []
for _ in range(N):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    P.prefill_with_reuse(model, req, store)
    e1.record()
    e1.synchronize()
    ev.append(e0.elapsed_time(e1))
print(f"e2e p50 {1e3 * np.median(e2e):.3f} ms (host issue {1e3 * np.median(host):.3f} ms), device events p50 "
      f"{np.median(ev):.3f} ms (no L2 flush)")
