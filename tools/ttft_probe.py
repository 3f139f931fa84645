"""p50 device TTFT of the C3 reuse prefill (bench.py's measurement, no baselines) -- for A/B runs of
environment knobs (VLC_* tuning / VLC_EXPERIMENT_SKIP=<kernel names>)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2512_12977_b200 as P  # noqa: E402
from paper_2512_12977_b200.toydata import make_images, prompt_ids  # noqa: E402

ratio = float(sys.argv[1]) if len(sys.argv) > 1 else 0.05
cfg = P.ModelConfig(**bench.CONFIGS["C3"], seed=0)
model = P.ToyVLM.device_random(cfg, 0)
store = P.CacheStore()
imgs = make_images(4, cfg.image_side, 1)
P.fill_store(model, store, imgs, prompt_ids(cfg.vocab_size, 8, 11))
text = prompt_ids(cfg.vocab_size, 32, 12)
seq = P.make_sequence(text[:16], 4, cfg.tokens_per_image, text[16:])
req = P.ReuseRequest(seq, [P.hash_image(p) for p in imgs], P.plan_static(ratio, cfg.num_layers))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    P.prefill_with_reuse(model, req, store)
torch.cuda.synchronize()
ts = []
for _ in range(30):
    flush.fill_(1)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    P.prefill_with_reuse(model, req, store)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"{os.environ.get('TAG', '')} ttft p50 {np.median(ts):.3f} ms  min {min(ts):.3f}", flush=True)
