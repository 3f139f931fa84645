"""End-to-end parity of the device reuse prefill against the CPU oracle.

Tolerance: the oracle runs on the SAME bf16-rounded weights;
indices / hit-miss decisions must be bit-exact; logits and recomputed K/V within
rel_err <= 2e-2 (max|a-e| / max|e|, the reference's metric, conftest.py:25-28)
with the last row's top-1 token identical.
"""
import numpy as np
import pytest

from conftest import rel_err
from oracle import kvreuse_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 2e-2

SMALL = dict(num_layers=4, num_heads=2, model_dim=32, kv_dim=32, vocab_size=97, patch_size=4,
             tokens_per_image=16, seed=7)
C1 = dict(num_layers=4, num_heads=8, model_dim=256, kv_dim=256, vocab_size=4096, patch_size=4,
          tokens_per_image=256, seed=0)


def _models(cfg_kw):
    import paper_2512_12977_b200 as P
    ocfg = O.Cfg(**cfg_kw)
    w = {k: O.bf16_round(v) for k, v in O.make_weights(ocfg).items()}
    return P, ocfg, w, P.ToyVLM(P.ModelConfig(**cfg_kw), w)


class Scene:
    """Oracle store + device store filled from the SAME oracle KV (isolates the reuse path)."""

    def __init__(self, cfg_kw, n_images, cache_prefix, seed_img=1):
        self.P, self.ocfg, self.w, self.model = _models(cfg_kw)
        P, ocfg = self.P, self.ocfg
        T = ocfg.tokens_per_image
        self.images = O.images(n_images, ocfg.side, seed_img)
        self.enc, self.kv = {}, {}
        for px in self.images:
            ids, segs = O.layout(cache_prefix, 1, T)
            O.fill_one(ocfg, self.w, ids, segs, [px], self.enc, self.kv)
        self.store = P.CacheStore()
        fp = self.model.fingerprint
        for px in self.images:
            h = O.sha256_hex(px)
            self.store.put_encoder(P.EncoderCacheEntry(P.ImageHash(h), self.enc[h], fp))
            e = self.kv[h]
            self.store.put_kv(P.KVCacheEntry(P.ImageHash(h), e.keys, e.values, e.origin_position, fp))

    def run(self, prefix, suffix, ratios, images=None, store=None, oracle_stores=None):
        P, ocfg = self.P, self.ocfg
        T = ocfg.tokens_per_image
        n_img = len(self.images)
        ids, segs = O.layout(prefix, n_img, T, suffix)
        hashes = [O.sha256_hex(px) for px in self.images]
        enc, kv = oracle_stores if oracle_stores is not None else (self.enc, self.kv)
        ref = O.reuse_prefill(ocfg, self.w, ids, segs, hashes, ratios, enc, kv, images=images)
        seq = P.make_sequence(prefix, n_img, T, suffix)
        req = P.ReuseRequest(seq, [P.hash_image(px) for px in self.images], P.RecomputePlan(tuple(ratios)),
                             images=images)
        got = P.prefill_with_reuse(self.model, req, self.store if store is None else store)
        return ref, got


def _check(ref, got, tol=TOL, check_top1=True):
    assert np.array_equal(got.positions, ref.rows)
    assert got.metrics.computed_per_layer == ref.counts
    assert got.metrics.encoder_misses == ref.encoder_misses
    assert got.metrics.fallback_images == ref.fallback_images
    e = rel_err(got.logits, ref.logits)
    assert e <= tol, f"logits rel_err {e}"
    if check_top1:
        assert int(np.argmax(got.logits[-1])) == int(np.argmax(ref.logits[-1]))
    ek = rel_err(got.kv.keys, ref.keys)
    ev = rel_err(got.kv.values, ref.values)
    assert ek <= tol and ev <= tol, (ek, ev)
    return e


@pytest.fixture(scope="module")
def small(cuda_ok):
    return Scene(SMALL, 1, O.prompt(97, 6, 1))


@pytest.mark.parametrize("ratios", [(1.0,) * 4, (0.0,) * 4, (0.3, 0.2, 0.1, 0.0), (0.3, 0.3, 0.3, 0.3)])
@pytest.mark.parametrize("same_prefix", [True, False])
def test_small_reuse_parity(small, ratios, same_prefix):
    prefix = O.prompt(97, 6, 1) if same_prefix else O.prompt(97, 6, 99)
    ref, got = small.run(prefix, O.prompt(97, 4, 2), ratios)
    _check(ref, got)


def test_small_all_miss_fallback(small):
    P = small.P
    ref, got = small.run(O.prompt(97, 6, 1), O.prompt(97, 4, 2), (0.0,) * 4, images=small.images,
                         store=P.CacheStore(), oracle_stores=({}, {}))
    assert (got.metrics.fallback_images, got.metrics.encoder_misses) == (1, 1)
    _check(ref, got)


def test_small_errors(small):
    P = small.P
    seq = P.make_sequence(O.prompt(97, 6, 1), 1, 16)
    h = [P.hash_image(small.images[0])]
    with pytest.raises(P.InputError):
        P.prefill_with_reuse(small.model, P.ReuseRequest(seq, h, P.plan_static(0.0, 4)), P.CacheStore())
    with pytest.raises(P.PlanError):
        P.prefill_with_reuse(small.model, P.ReuseRequest(seq, h, P.RecomputePlan((0.003, 0, 0, 0))), small.store)
    with pytest.raises(P.InputError):
        P.prefill_with_reuse(small.model, P.ReuseRequest(seq, h, P.plan_static(0.1, 3)), small.store)
    other = P.ToyVLM(P.ModelConfig(**{**SMALL, "seed": 11}))
    with pytest.raises(P.StaleCacheError):
        P.prefill_with_reuse(other, P.ReuseRequest(seq, h, P.plan_static(0.0, 4)), small.store)


def test_small_device_fill_then_reuse(small):
    """Miss path on device (GPU encoder + dense prefill + store write-back), then reuse."""
    P = small.P
    store = P.CacheStore()
    P.fill_store(small.model, store, small.images, O.prompt(97, 6, 1))
    assert len(store) == 2
    ref, got = small.run(O.prompt(97, 6, 99), O.prompt(97, 4, 2), (0.3, 0.2, 0.1, 0.0), store=store)
    _check(ref, got, tol=3e-2)
    emb = store.get_encoder(P.hash_image(small.images[0])).embeddings
    assert rel_err(emb, small.enc[O.sha256_hex(small.images[0])]) <= TOL


def test_small_prefill_full_and_encoder(small):
    P = small.P
    T = 16
    ids, segs = O.layout(O.prompt(97, 6, 1), 1, T, O.prompt(97, 4, 2))
    emb = O.encode(small.ocfg, small.w, small.images[0])
    ref_logits, ref_k, ref_v = O.dense_prefill(small.ocfg, small.w, ids, segs, [emb])
    seq = P.make_sequence(O.prompt(97, 6, 1), 1, T, O.prompt(97, 4, 2))
    logits, kv = P.prefill_full(small.model, seq, [emb])
    assert rel_err(logits, ref_logits) <= TOL
    assert rel_err(kv.keys, ref_k) <= TOL and rel_err(kv.values, ref_v) <= TOL
    assert rel_err(P.encode_image(small.model, small.images[0]), emb) <= TOL


@pytest.fixture(scope="module")
def c1(cuda_ok):
    return Scene(C1, 1, O.prompt(4096, 8, 11))


@pytest.mark.parametrize("r", [0.05, 0.0, 0.3, 1.0])
def test_c1_reuse_parity(c1, r):
    """BASELINE configs[0]: 4 layers d256 H8, 256 cached image tokens + 32 text, 5% recompute."""
    text = O.prompt(4096, 32, 12)
    ref, got = c1.run(text[:16], text[16:], (r,) * 4)
    _check(ref, got)


def test_c1_dynamic_plan_and_last_logits(c1):
    text = O.prompt(4096, 32, 12)
    ref, got = c1.run(text[:16], text[16:], (0.1, 0.05, 0.05, 0.002))
    _check(ref, got)
    assert np.allclose(got.last_logits(), got.logits[-1])


def test_c1_multi_image_shifted(cuda_ok):
    sc = Scene({**C1, "seed": 3}, 3, O.prompt(4096, 8, 11), seed_img=4)
    text = O.prompt(4096, 20, 5)
    ref, got = sc.run(text[:7], text[7:], (0.05, 0.05, 0.04, 0.02))
    _check(ref, got)
