"""Run-to-run spread of serial calls vs results of two concurrent threads (C1 scene)."""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_12977_b200 as P  # noqa: E402
from scenes import Scene  # noqa: E402

sc = Scene(P, "C1", 2, export=False)
L = sc.cfg.num_layers
plans = [P.plan_static(0.05, L), P.RecomputePlan((0.3, 0.2, 0.1, 0.0)), P.plan_static(0.0, L),
         P.RecomputePlan((1.0, 0.1, 0.1, 0.0))]
ser = [[P.prefill_with_reuse(sc.model, sc.request(p), sc.store).logits for p in plans] for _ in range(3)]
for k in range(len(plans)):
    print("plan", k, "serial spread", max(float(np.max(np.abs(ser[r][k] - ser[0][k]))) for r in range(3)))
out = {}


def worker(tid):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for rep in range(6):
            k = (tid + rep) % len(plans)
            res = P.prefill_with_reuse(sc.model, sc.request(plans[k]), sc.store)
            out[(tid, rep)] = (k, res.logits)


th = [threading.Thread(target=worker, args=(t,)) for t in range(2)]
[t.start() for t in th]
[t.join() for t in th]
for (tid, rep), (k, lg) in sorted(out.items()):
    d = np.abs(lg - ser[0][k])
    print(f"thread {tid} rep {rep} plan {k}: max diff {d.max():.3e} rows>1e-4 {np.flatnonzero(d.max(1) > 1e-4)[:10]}")
