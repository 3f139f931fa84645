"""One C3 reuse prefill under cudaProfilerStart/Stop (for `ncu --profile-from-start off`),
plus host-issue timing of prefill_with_reuse (no sync)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2512_12977_b200 as P  # noqa: E402
from paper_2512_12977_b200.engine import prefill_with_reuse  # noqa: E402
from paper_2512_12977_b200.toydata import make_images, prompt_ids  # noqa: E402

wl = bench.WORKLOADS[os.environ.get("WL", "C3")]
ratio = float(os.environ.get("RATIO", wl["ratio"]))
cfg = P.ModelConfig(**bench.CONFIGS[wl["cfg"]], seed=0)
model = P.ToyVLM.device_random(cfg, 0)
store = P.CacheStore()
imgs = make_images(wl["images"], cfg.image_side, 1)
P.fill_store(model, store, imgs, prompt_ids(cfg.vocab_size, 8, 11))
text = prompt_ids(cfg.vocab_size, 32, 12)
seq = P.make_sequence(text[:16], wl["images"], cfg.tokens_per_image, text[16:])
req = P.ReuseRequest(seq, [P.hash_image(p) for p in imgs], P.plan_static(ratio, cfg.num_layers))
for _ in range(3):
    prefill_with_reuse(model, req, store)
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter()
    prefill_with_reuse(model, req, store)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"host issue {1e3 * (t1 - t0):.2f} ms, issue+drain {1e3 * (t2 - t0):.2f} ms", flush=True)
torch.cuda.profiler.start()
prefill_with_reuse(model, req, store)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
