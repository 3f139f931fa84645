"""One C1 reuse prefill (configs[0]) plus a C2-width 2-layer one, for compute-sanitizer.

Run eagerly (VLC_DEBUG_SYNC=1 -> every launch synchronised, no CUDA graph) so the sanitizer sees each
kernel of the chain: embed, kv_relocate, RMSNorm, the tcgen05 GEMMs (one-tile, split-K red.add,
stream-K fix-up), the attention (split-KV in-kernel merge), the CTA-pair LM head, the store page
writes of the device miss path.  Checks the result against the oracle so a sanitizer run that
silently changed the arithmetic shows up too.

  compute-sanitizer --tool memcheck  python tools/sanitize_chain.py
  compute-sanitizer --tool racecheck python tools/sanitize_chain.py
  compute-sanitizer --tool synccheck python tools/sanitize_chain.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ.setdefault("VLC_DEBUG_SYNC", "1")

import numpy as np  # noqa: E402

import paper_2512_12977_b200 as P  # noqa: E402
from oracle import kvreuse_oracle as O  # noqa: E402
from scenes import CONFIGS, Scene  # noqa: E402

CONFIGS["C2x2"] = dict(CONFIGS["C2"], num_layers=2)


def main():
    for name, n_img, ratios in (("C1", 2, (0.05,) * 4), ("C1", 1, (1.0, 0.1, 0.1, 0.0)), ("C2x2", 1, (0.03, 0.02))):
        sc = Scene(P, name, n_img)
        oc, w, ids, segs, keys, enc, kv = sc.oracle_inputs()
        res = P.prefill_with_reuse(sc.model, sc.request(P.RecomputePlan(ratios)), sc.store)
        ref = O.reuse_prefill(oc, w, ids, segs, keys, ratios, enc, kv)
        err = O.rel_err(res.logits, ref.logits)
        ok = np.array_equal(res.positions, ref.rows) and err <= 2e-2
        print(f"{name} images={n_img} plan={ratios[:2]}..: rel_err={err:.3e} rows_equal="
              f"{np.array_equal(res.positions, ref.rows)} {'OK' if ok else 'MISMATCH'}", flush=True)
        if not ok:
            sys.exit(1)


if __name__ == "__main__":
    main()
