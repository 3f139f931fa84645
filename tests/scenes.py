"""Shared scene builders for the full-scale parity tests and bench.py's parity / CPU legs.

A *scene* is the benchmark setup of BASELINE configs[1] / configs[2]: a device model with
random-init weights, a store filled by the device cache-miss path (each image cached under an
8-token prefix, bench.py:98-104 of the reference) and the live request that reuses the images at
SHIFTED positions (16-token prefix, 16-token suffix).  `oracle_inputs` hands the CPU side exactly
what the device holds: the weights (bf16 values widened to fp32, reference names and layout) and
the stored encoder rows / pre-RoPE K/V (bf16 pages widened to fp32).
"""
from __future__ import annotations

import numpy as np

CONFIGS = {
    "C1": dict(num_layers=4, num_heads=8, model_dim=256, kv_dim=256, vocab_size=4096, patch_size=4,
               tokens_per_image=256),
    "C2": dict(num_layers=28, num_heads=12, model_dim=1536, kv_dim=1536, vocab_size=151936, patch_size=4,
               tokens_per_image=1024),
    "C3": dict(num_layers=28, num_heads=28, model_dim=3584, kv_dim=3584, vocab_size=152064, patch_size=4,
               tokens_per_image=1024),
}


class Scene:
    def __init__(self, P, name: str, n_images: int, seed: int = 0, export: bool = True, image_seed: int = 1,
                 tp_group=None):
        from paper_2512_12977_b200.toydata import make_images, prompt_ids
        self.P, self.name = P, name
        self.kw = dict(CONFIGS[name], seed=seed)
        self.cfg = P.ModelConfig(**self.kw)
        self.w = {} if export else None
        self.model = P.ToyVLM.device_random(self.cfg, seed=seed, export=self.w, tp_group=tp_group)
        V, T = self.cfg.vocab_size, self.cfg.tokens_per_image
        self.images = make_images(n_images, self.cfg.image_side, image_seed)
        self.store = P.CacheStore()
        P.fill_store(self.model, self.store, self.images, prompt_ids(V, 8, 11))   # device miss path
        self.hashes = [P.hash_image(px) for px in self.images]
        self.text = prompt_ids(V, 32, 12)
        self.seq = P.make_sequence(self.text[:16], n_images, T, self.text[16:])

    def request(self, plan):
        return self.P.ReuseRequest(self.seq, self.hashes, plan)

    def oracle_inputs(self):
        """(oracle Cfg, weights, ids, segs, hash keys, encoder store, KV store) for
        oracle.reuse_prefill -- or, with the same data, the reference's prefill_with_reuse."""
        from oracle import kvreuse_oracle as O
        oc = O.Cfg(**self.kw)
        ids, segs = O.layout(self.text[:16], len(self.images), self.cfg.tokens_per_image, self.text[16:])
        keys = [h.hex for h in self.hashes]
        enc, kv = {}, {}
        for h in self.hashes:
            e = self.store.get_encoder(h)
            k = self.store.get_kv(h)
            enc[h.hex] = np.ascontiguousarray(e.embeddings, dtype=np.float32)
            kv[h.hex] = O.KVEntry(k.keys, k.values, k.origin_position)
        return oc, self.w, ids, segs, keys, enc, kv


def rel_err_layers(actual, expected) -> float:
    """rel_err (max|a - e| / max|e|, the reference's metric) over [L, n, kv] arrays, layer by
    layer to bound the float64 transient."""
    num, den = 0.0, 1e-6
    for i in range(expected.shape[0]):
        e = np.asarray(expected[i], np.float64)
        num = max(num, float(np.max(np.abs(np.asarray(actual[i], np.float64) - e))))
        den = max(den, float(np.max(np.abs(e))))
    return num / den
