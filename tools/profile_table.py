"""Profile a sensitivity table on the device for the bench model (configs[3]) and write it to
profiles/<workload>_sensitivity_table.json (read by bench.py's layer-aware vs uniform comparison).

Protocol = the reference's (sensitivity.py:88-178) through paper_2512_12977_b200.sensitivity.profile:
per proxy sample (image, original prompt, neutral prompt), the neutral-prompt KV is injected at every
layer except the first floor(r*T) image tokens of the probed layer; score = logit MSE vs the
same-context greedy continuation, averaged over samples."""
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
n_samples = int(os.environ.get("SAMPLES", "3"))
samples = [S.ProxySample(make_image(cfg.image_side, 400 + k), prompt_ids(V, 10, 500 + k), prompt_ids(V, 10, 0xD00D))
           for k in range(n_samples)]
grid = (0.01, 0.02, 0.04, 0.06, 0.08, 0.1)
t0 = time.time()
table = S.profile(model, samples, grid, max_new=4)
dt = time.time() - t0
out = {"workload": wl, "model": "device_random seed 0", "model_fingerprint": model.fingerprint,
       "grid": list(grid), "baseline": table.baseline, "scores": table.scores.tolist(), "samples": n_samples,
       "max_new": 4, "profile_seconds": round(dt, 1)}
path = os.path.join(ROOT, "gpurun_out", f"{wl.lower()}_sensitivity_table.json")
os.makedirs(os.path.dirname(path), exist_ok=True)
json.dump(out, open(path, "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "scores"}), flush=True)
print(np.array(table.scores).round(4))
