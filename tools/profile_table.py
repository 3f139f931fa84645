"""Profile a sensitivity table on the device for the bench model (configs[3]) and write it to
gpurun_out/<workload>_sensitivity_table.json (committed as profiles/..., read by bench.py's layer-aware vs
uniform comparison).

Protocol = the reference's (sensitivity.py:88-178) through paper_2512_12977_b200.sensitivity.profile:
per proxy sample (image, original prompt, neutral prompt), the neutral-prompt KV is injected at every
layer except the first floor(r*T) image tokens of the probed layer; score = logit MSE vs the
same-context greedy continuation, averaged over samples.  Each sample's table is kept too, so the
per-cell standard error says whether a layer's gain S(0) - S(r) is above the sample noise."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2512_12977_b200 as P  # noqa: E402
from paper_2512_12977_b200 import sensitivity as S  # noqa: E402
from paper_2512_12977_b200.toydata import make_image, prompt_ids  # noqa: E402

wl = os.environ.get("WL", "C3")
cfg = P.ModelConfig(**bench.CONFIGS[bench.WORKLOADS[wl]["cfg"]], seed=0)
model = P.ToyVLM.device_random(cfg, seed=0)
V = cfg.vocab_size
n_samples = int(os.environ.get("SAMPLES", "8"))
max_new = int(os.environ.get("MAX_NEW", "4"))
grid = tuple(float(g) for g in os.environ.get("GRID", "0.02,0.04,0.06,0.08,0.1").split(","))
t0 = time.time()
per = []
for k in range(n_samples):
    smp = S.ProxySample(make_image(cfg.image_side, 400 + k), prompt_ids(V, 10, 500 + k), prompt_ids(V, 10, 0xD00D))
    t = S.profile(model, [smp], grid, max_new=max_new)
    per.append((t.baseline, t.scores))
    print(f"sample {k}: {time.time() - t0:.0f} s", flush=True)
dt = time.time() - t0
base = float(np.mean([b for b, _ in per]))
sc = np.mean([s for _, s in per], axis=0)
# gain of each layer at the largest grid ratio, per sample, and its standard error over samples
gains = np.array([b - s[:, -1] for b, s in per])                 # [samples, L]
se = gains.std(axis=0, ddof=1) / np.sqrt(len(per)) if len(per) > 1 else np.zeros(cfg.num_layers)
out = {"workload": wl, "model": "device_random seed 0", "model_fingerprint": model.fingerprint,
       "grid": list(grid), "baseline": base, "scores": sc.tolist(), "samples": n_samples, "max_new": max_new,
       "per_sample_baseline": [b for b, _ in per], "per_sample_scores": [s.tolist() for _, s in per],
       "gain_at_max_ratio": gains.mean(axis=0).tolist(), "gain_se": se.tolist(),
       "layers_gain_above_2se": int((gains.mean(axis=0) > 2 * se).sum()), "profile_seconds": round(dt, 1)}
path = os.path.join(ROOT, "gpurun_out", f"{wl.lower()}_sensitivity_table.json")
os.makedirs(os.path.dirname(path), exist_ok=True)
json.dump(out, open(path, "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if "scores" not in k and "per_sample" not in k}), flush=True)
