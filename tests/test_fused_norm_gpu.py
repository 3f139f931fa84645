"""RMSNorm fused into the residual projections' tail (vlc_epilogue.norm_*, VLC_FUSED_NORM=1):
the reuse prefill with the fused norms against the CPU oracle (configs[0]-like) and against the
separate-launch chain at the C3 width."""
import numpy as np
import pytest

from conftest import rel_err
from oracle import kvreuse_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

KW = dict(num_layers=4, num_heads=8, model_dim=256, kv_dim=256, vocab_size=4096, patch_size=4,
          tokens_per_image=256, seed=0)


@pytest.fixture
def fused():
    from paper_2512_12977_b200 import runtime as RT
    old = RT._FUSED_NORM
    RT._FUSED_NORM = True
    yield
    RT._FUSED_NORM = old


def test_fused_norm_matches_oracle(cuda_ok, fused):
    import paper_2512_12977_b200 as P
    oc = O.Cfg(**KW)
    w = {k: O.bf16_round(v) for k, v in O.make_weights(oc).items()}
    model = P.ToyVLM(P.ModelConfig(**KW), w)
    V, T = oc.vocab_size, oc.tokens_per_image
    img = O.images(1, oc.side, 1)
    enc, kv = {}, {}
    ids0, segs0 = O.layout(O.prompt(V, 8, 11), 1, T)
    O.fill_one(oc, w, ids0, segs0, img, enc, kv)
    h = O.sha256_hex(img[0])
    store = P.CacheStore()
    store.put_encoder(P.EncoderCacheEntry(P.ImageHash(h), enc[h], model.fingerprint))
    store.put_kv(P.KVCacheEntry(P.ImageHash(h), kv[h].keys, kv[h].values, 8, model.fingerprint))
    text = O.prompt(V, 32, 12)
    ids, segs = O.layout(text[:16], 1, T, text[16:])
    ratios = (0.1, 0.05, 0.05, 0.02)                     # depth-packed rows: c shrinks per layer
    ref = O.reuse_prefill(oc, w, ids, segs, [h], ratios, enc, kv)
    req = P.ReuseRequest(P.make_sequence(text[:16], 1, T, text[16:]), [P.ImageHash(h)], P.RecomputePlan(ratios))
    for _ in range(2):                                   # eager, then the captured graph
        got = P.prefill_with_reuse(model, req, store)
        assert np.array_equal(got.positions, ref.rows)
        assert rel_err(got.logits, ref.logits) <= 2e-2
        assert int(np.argmax(got.logits[-1])) == int(np.argmax(ref.logits[-1]))
        assert rel_err(got.kv.keys, ref.keys) <= 2e-2


@pytest.mark.timeout(900)
def test_fused_norm_equals_separate_norm_c3(cuda_ok):
    import paper_2512_12977_b200 as P
    from paper_2512_12977_b200 import runtime as RT
    from paper_2512_12977_b200.toydata import make_images, prompt_ids
    cfg = P.ModelConfig(num_layers=28, num_heads=28, model_dim=3584, kv_dim=3584, vocab_size=152064, patch_size=4,
                        tokens_per_image=1024, seed=0)
    model = P.ToyVLM.device_random(cfg, seed=0)
    imgs = make_images(2, cfg.image_side, 1)
    store = P.CacheStore()
    P.fill_store(model, store, imgs, prompt_ids(cfg.vocab_size, 8, 11))
    text = prompt_ids(cfg.vocab_size, 32, 12)
    req = P.ReuseRequest(P.make_sequence(text[:16], 2, cfg.tokens_per_image, text[16:]),
                         [P.hash_image(p) for p in imgs], P.plan_static(0.05, cfg.num_layers))
    old = RT._FUSED_NORM
    try:
        RT._FUSED_NORM = False
        a = P.prefill_with_reuse(model, req, store).logits
        RT._FUSED_NORM = True
        model._runner.graphs.clear()
        b = P.prefill_with_reuse(model, req, store).logits
    finally:
        RT._FUSED_NORM = old
        model._runner.graphs.clear()
    assert rel_err(b, a) <= 2e-2
    assert int(np.argmax(a[-1])) == int(np.argmax(b[-1]))
