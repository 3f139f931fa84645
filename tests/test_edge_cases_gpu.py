"""Edge cases of the reuse prefill on the device vs the CPU oracle (bf16-rounded weights):
text-only and image-only requests, one image repeated inside a request, a hit next to a miss
(encoder miss with pixels + KV fallback for that image only), the grid extremes 0.002 and 0.3."""
import numpy as np
import pytest

from conftest import rel_err
from oracle import kvreuse_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

KW = dict(num_layers=3, num_heads=4, model_dim=128, kv_dim=128, vocab_size=501, patch_size=4,
          tokens_per_image=64, seed=5)


@pytest.fixture(scope="module")
def env(cuda_ok):
    import paper_2512_12977_b200 as P
    oc = O.Cfg(**KW)
    w = {k: O.bf16_round(v) for k, v in O.make_weights(oc).items()}
    model = P.ToyVLM(P.ModelConfig(**KW), w)
    imgs = O.images(2, oc.side, 9)
    enc, kv = {}, {}
    for px in imgs[:1]:                                 # only image 0 is cached
        ids0, segs0 = O.layout(O.prompt(501, 5, 3), 1, 64)
        O.fill_one(oc, w, ids0, segs0, [px], enc, kv)
    store = P.CacheStore()
    h0 = O.sha256_hex(imgs[0])
    store.put_encoder(P.EncoderCacheEntry(P.ImageHash(h0), enc[h0], model.fingerprint))
    store.put_kv(P.KVCacheEntry(P.ImageHash(h0), kv[h0].keys, kv[h0].values, 5, model.fingerprint))
    return P, oc, w, model, imgs, enc, kv, store


def _run(env, prefix, img_idx, suffix, ratios, pixels=False):
    P, oc, w, model, imgs, enc, kv, store = env
    T = oc.tokens_per_image
    ims = [imgs[i] for i in img_idx]
    ids, segs = O.layout(prefix, len(ims), T, suffix)
    hs = [O.sha256_hex(px) for px in ims]
    px = ims if pixels else None
    ref = O.reuse_prefill(oc, w, ids, segs, hs, ratios, dict(enc), dict(kv), images=px)
    seq = P.make_sequence(prefix, len(ims), T, suffix)
    got = P.prefill_with_reuse(model, P.ReuseRequest(seq, [P.ImageHash(h) for h in hs], P.RecomputePlan(ratios),
                                                     images=px), store)
    assert np.array_equal(got.positions, ref.rows)
    assert got.metrics.computed_per_layer == ref.counts
    assert (got.metrics.encoder_misses, got.metrics.fallback_images) == (ref.encoder_misses, ref.fallback_images)
    assert rel_err(got.logits, ref.logits) <= 2e-2
    assert int(np.argmax(got.logits[-1])) == int(np.argmax(ref.logits[-1]))
    assert rel_err(got.kv.keys, ref.keys) <= 2e-2 and rel_err(got.kv.values, ref.values) <= 2e-2
    return got


def test_text_only(env):
    got = _run(env, O.prompt(501, 37, 1), [], [], (0.05, 0.05, 0.0))
    assert len(got.positions) == 37


def test_image_only(env):
    _run(env, [], [0], [], (0.1, 0.05, 0.02))


def test_no_rows_at_a_layer(env):
    """Image-only request whose plan recomputes nothing at the last layer: the reference raises a
    NumPy reshape error there (zero rows); the device path returns an empty logits block."""
    P, oc, w, model, imgs, enc, kv, store = env
    seq = P.make_sequence([], 1, 64)
    got = P.prefill_with_reuse(model, P.ReuseRequest(seq, [P.hash_image(imgs[0])], P.RecomputePlan((0.1, 0.05, 0.0))),
                               store)
    assert got.logits.shape == (0, 501) and len(got.positions) == 0
    assert got.metrics.computed_per_layer == [6, 3, 0]


def test_same_image_twice(env):
    _run(env, O.prompt(501, 4, 2), [0, 0], O.prompt(501, 3, 4), (0.3, 0.1, 0.002))


def test_hit_next_to_miss(env):
    got = _run(env, O.prompt(501, 6, 6), [0, 1], O.prompt(501, 5, 7), (0.05, 0.05, 0.05), pixels=True)
    assert got.metrics.encoder_misses == 1 and got.metrics.fallback_images == 1


@pytest.mark.parametrize("r", [0.002, 0.3])
def test_grid_extremes(env, r):
    _run(env, O.prompt(501, 9, 8), [0], O.prompt(501, 9, 9), (r,) * 3)


@pytest.mark.parametrize("npre,nsuf", [(150, 100), (300, 260)])
def test_wide_and_multi_token_tiles(env, npre, nsuf):
    """Long text around repeated cached images: 257..512 computed rows run every one-wave GEMM as ONE
    wide token tile (two UMMA N chunks), > 512 rows as several token tiles; parity with the oracle."""
    got = _run(env, O.prompt(501, npre, 11), [0, 0, 0], O.prompt(501, nsuf, 12), (0.3, 0.3, 0.1))
    assert max(got.metrics.computed_per_layer) > 256
