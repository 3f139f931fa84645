"""Generate golden fixtures from the REAL reference package (kvreuse 0.1.0).

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs tests/golden/*.npz.  These pin the CPU oracle (oracle/kvreuse_oracle.py)
to the reference; the oracle in turn is the checker for the CUDA path.
"""
import os
import sys

import numpy as np

REF = os.environ.get("VLC_REF_PATH", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from kvreuse import ModelConfig, init_model  # noqa: E402
from kvreuse.bench import fill_store  # noqa: E402
from kvreuse.engine import ReuseRequest, count_flops, prefill_with_reuse  # noqa: E402
from kvreuse.model import (encode_image, generate, make_sequence, prefill_full,  # noqa: E402
                           weight_checksum)
from kvreuse.planner import BudgetSpec, plan_bruteforce, plan_greedy  # noqa: E402
from kvreuse.plans import RecomputePlan, build_masks, plan_static  # noqa: E402
from kvreuse.sensitivity import SensitivityTable  # noqa: E402
from kvreuse.store import CacheStore, hash_image  # noqa: E402
from kvreuse.toydata import make_image, make_images, prompt_ids  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

SMALL = dict(num_layers=4, num_heads=2, model_dim=32, kv_dim=32, vocab_size=97,
             patch_size=4, tokens_per_image=16, seed=7)
C1 = dict(num_layers=4, num_heads=8, model_dim=256, kv_dim=256, vocab_size=4096,
          patch_size=4, tokens_per_image=256, seed=0)


def small_scene():
    cfg = ModelConfig(**SMALL)
    m = init_model(cfg)
    img = make_image(16, 3)
    prefix, suffix = prompt_ids(97, 6, 1), prompt_ids(97, 4, 2)
    store = CacheStore()
    fill_store(m, store, [img], prefix)
    h = hash_image(img)
    out = {"fingerprint": np.array(m.fingerprint, dtype=np.uint64),
           "checksum": np.frombuffer(bytes.fromhex(weight_checksum(m)), np.uint8),
           "img": img, "prefix": np.array(prefix), "suffix": np.array(suffix),
           "image_hash": np.frombuffer(bytes.fromhex(h.hex), np.uint8)}
    emb = encode_image(m, img)
    out["emb"] = emb
    out["enc_zero_head"] = encode_image(m, np.zeros((16, 16), np.float32))[0, :4]
    seq_same = make_sequence(prefix, 1, 16, suffix=suffix)
    mis_prefix = prompt_ids(97, 6, 99)
    seq_mis = make_sequence(mis_prefix, 1, 16, suffix=suffix)
    cases = {
        "full": (seq_same, plan_static(1.0, 4)),
        "r0_same": (seq_same, plan_static(0.0, 4)),
        "r0_mis": (seq_mis, plan_static(0.0, 4)),
        "mixed_mis": (seq_mis, RecomputePlan((0.3, 0.2, 0.1, 0.0))),
    }
    for name, (seq, plan) in cases.items():
        res = prefill_with_reuse(m, ReuseRequest(seq, [h], plan), store)
        out[f"{name}_rows"] = res.positions
        out[f"{name}_logits"] = res.logits
        out[f"{name}_keys"] = res.kv.keys
        out[f"{name}_values"] = res.kv.values
        out[f"{name}_counts"] = np.array(res.metrics.computed_per_layer)
    full_mis, _ = prefill_full(m, seq_mis, [emb])
    out["full_mis_logits"] = full_mis
    res = prefill_with_reuse(m, ReuseRequest(seq_same, [h], plan_static(0.0, 4), images=[img]),
                             CacheStore())
    out["miss_logits"] = res.logits
    out["miss_metrics"] = np.array([res.metrics.fallback_images, res.metrics.encoder_misses])
    ids, _ = generate(m, seq_same, [emb], 8)
    out["generate_ids"] = np.array(ids)
    fl = count_flops(seq_mis, RecomputePlan((0.3, 0.2, 0.1, 0.0)), cfg, encoder_cached=False)
    out["flops_mixed"] = np.array([fl.encoder, fl.attention, fl.mlp], dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "small_scene.npz"), **out)


def c1_scene():
    """BASELINE configs[0]: L4 d256 H8, 256 cached image tokens + 32 text, r=0.05."""
    cfg = ModelConfig(**C1)
    m = init_model(cfg)
    T, V = cfg.tokens_per_image, cfg.vocab_size
    imgs = make_images(1, cfg.image_side, 1)
    store = CacheStore()
    fill_store(m, store, imgs, prompt_ids(V, 8, 11))
    text = prompt_ids(V, 32, 12)
    seq = make_sequence(text[:16], 1, T, suffix=text[16:])
    res = prefill_with_reuse(m, ReuseRequest(seq, [hash_image(p) for p in imgs],
                                             plan_static(0.05, 4)), store)
    out = {"fingerprint": np.array(m.fingerprint, dtype=np.uint64),
           "rows": res.positions, "logits": res.logits,
           "counts": np.array(res.metrics.computed_per_layer),
           "keys_l0": res.kv.keys[0], "keys_l3": res.kv.keys[3],
           "values_l0": res.kv.values[0], "values_l3": res.kv.values[3]}
    np.savez_compressed(os.path.join(OUT, "c1_scene.npz"), **out)


def masks_and_plans():
    out = {}
    rng = np.random.default_rng(123)
    for t in range(20):
        L = int(rng.integers(1, 7))
        units = sorted(rng.integers(0, 151, size=L).tolist(), reverse=True)
        ratios = tuple(u * 0.002 for u in units)
        if rng.random() < 0.2:
            ratios = (1.0,) + ratios[1:]
        n_text_pre, n_img, n_suf = int(rng.integers(0, 5)), int(rng.integers(0, 4)), int(rng.integers(0, 4))
        T = int([16, 64, 256][rng.integers(0, 3)])
        seq = make_sequence(list(range(1, n_text_pre + 1)), n_img, T, suffix=list(range(n_suf)))
        if len(seq) == 0:
            continue
        mk = build_masks(RecomputePlan(ratios), seq)
        out[f"m{t}_ratios"] = np.array(ratios)
        out[f"m{t}_layout"] = np.array([n_text_pre, n_img, n_suf, T])
        out[f"m{t}_mask"] = mk.layers
    # allocator: greedy / brute force on random and diminishing tables
    for t in range(30):
        g = np.random.default_rng(500 + t)
        L = int(g.integers(2, 6))
        grid = (0.1, 0.2, 0.3) if t % 2 else (0.002, 0.01, 0.03, 0.05)
        scores = g.uniform(0.0, 1.0, size=(L, len(grid)))
        if t % 3 == 0:
            scores = np.sort(scores, axis=1)[:, ::-1].copy()
        base = float(g.uniform(0.5, 1.5))
        tbl = SensitivityTable(scores, grid, base, 1, 0)
        p = float(g.uniform(0, L * max(grid)))
        out[f"p{t}_scores"] = scores
        out[f"p{t}_grid"] = np.array(grid)
        out[f"p{t}_meta"] = np.array([base, p])
        out[f"p{t}_greedy"] = np.array(plan_greedy(tbl, BudgetSpec(p)).ratios)
        if L <= 6 and len(grid) <= 8:
            out[f"p{t}_brute"] = np.array(plan_bruteforce(tbl, BudgetSpec(p)).ratios)
    # 28-layer greedy at 3% mean budget on a pinned diminishing table (C2 plan)
    g = np.random.default_rng(2025)
    grid = tuple((k + 1) * 0.002 for k in range(50))
    gains = np.sort(g.uniform(0.001, 0.05, size=(28, len(grid))), axis=1)[:, ::-1]
    gains = gains * np.linspace(2.0, 0.5, 28)[:, None]
    scores = np.maximum(1.0 - np.cumsum(gains, axis=1), 0.0)
    tbl = SensitivityTable(scores, grid, 1.0, 1, 0)
    out["c2_table"] = scores
    out["c2_grid"] = np.array(grid)
    out["c2_plan"] = np.array(plan_greedy(tbl, BudgetSpec(0.03 * 28)).ratios)
    np.savez_compressed(os.path.join(OUT, "plans_masks.npz"), **out)


if __name__ == "__main__":
    small_scene()
    c1_scene()
    masks_and_plans()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))
