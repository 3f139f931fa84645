"""Pin the CPU oracle to the real reference (golden vectors + reference pins)."""
import numpy as np
import pytest

from conftest import golden, rel_err
from oracle import kvreuse_oracle as O

SMALL = O.Cfg(num_layers=4, num_heads=2, model_dim=32, kv_dim=32, vocab_size=97,
              patch_size=4, tokens_per_image=16, seed=7)
C1 = O.Cfg(num_layers=4, num_heads=8, model_dim=256, kv_dim=256, vocab_size=4096,
           patch_size=4, tokens_per_image=256, seed=0)


@pytest.fixture(scope="module")
def small():
    g = golden("small_scene.npz")
    w = O.make_weights(SMALL)
    enc, kv = {}, {}
    ids, segs = O.layout(list(g["prefix"]), 1, 16)
    O.fill_one(SMALL, w, ids, segs, [g["img"]], enc, kv)
    return g, w, enc, kv


def test_weights_fingerprint_matches_reference(small):
    g, w, _, _ = small
    assert O.fingerprint(SMALL, w) == int(g["fingerprint"])


def test_hash_pins():
    # test_store.py:45-49 and :70-74
    assert O.sha256_hex(np.arange(4, dtype=np.uint8)) == \
        "054edec1d0211f624fed0cbca9d4f9400b0e491c43742af2c5b0abebf0c990d8"
    a = np.arange(4, dtype=np.uint8).reshape(2, 2)
    assert O.sha256_many([a, a + 9]) == \
        "62fc9e9e103929bf2f07998578a063e5d66343e8ad009b976361947cfde871b3"


def test_encoder_pins(small):
    g, w, _, _ = small
    assert np.array_equal(O.encode(SMALL, w, g["img"]), g["emb"])
    head = O.encode(SMALL, w, np.zeros((16, 16), np.float32))[0, :4]
    # test_model.py:63-68 pin
    assert np.allclose(head, [-0.2425854, 1.10859, -1.0661058, 0.9320958], atol=1e-6)
    assert np.allclose(head, g["enc_zero_head"], atol=0)


@pytest.mark.parametrize("case,prefix_key,ratios", [
    ("full", "prefix", (1.0,) * 4), ("r0_same", "prefix", (0.0,) * 4),
    ("r0_mis", None, (0.0,) * 4), ("mixed_mis", None, (0.3, 0.2, 0.1, 0.0))])
def test_reuse_prefill_matches_reference(small, case, prefix_key, ratios):
    g, w, enc, kv = small
    prefix = list(g["prefix"]) if prefix_key else O.prompt(97, 6, 99)
    ids, segs = O.layout(prefix, 1, 16, list(g["suffix"]))
    h = O.sha256_hex(g["img"])
    out = O.reuse_prefill(SMALL, w, ids, segs, [h], ratios, enc, kv)
    assert np.array_equal(out.rows, g[f"{case}_rows"])
    assert out.counts == list(g[f"{case}_counts"])
    assert rel_err(out.logits, g[f"{case}_logits"]) <= 1e-6
    assert rel_err(out.keys, g[f"{case}_keys"]) <= 1e-6
    assert rel_err(out.values, g[f"{case}_values"]) <= 1e-6


def test_mismatched_mse_regression_pin(small):
    # test_engine.py:53-62: MSE 0.0774246963810249 (rel 1e-4)
    g, w, enc, kv = small
    ids, segs = O.layout(O.prompt(97, 6, 99), 1, 16, list(g["suffix"]))
    out = O.reuse_prefill(SMALL, w, ids, segs, [O.sha256_hex(g["img"])], (0.0,) * 4, enc, kv)
    full, _, _ = O.dense_prefill(SMALL, w, ids, segs, [g["emb"]])
    mse = float(np.mean((out.logits[-1].astype(np.float64) - full[-1]) ** 2))
    assert mse == pytest.approx(0.0774246963810249, rel=1e-4)


def test_miss_fallback(small):
    g, w, _, _ = small
    ids, segs = O.layout(list(g["prefix"]), 1, 16, list(g["suffix"]))
    out = O.reuse_prefill(SMALL, w, ids, segs, [O.sha256_hex(g["img"])], (0.0,) * 4, {}, {},
                          images=[g["img"]])
    assert (out.fallback_images, out.encoder_misses) == tuple(g["miss_metrics"])
    assert rel_err(out.logits, g["miss_logits"]) <= 1e-6


def test_flops_pin(small):
    g, _, _, _ = small
    ids, segs = O.layout(O.prompt(97, 6, 99), 1, 16, list(g["suffix"]))
    counts = O.compute_masks((0.3, 0.2, 0.1, 0.0), len(ids), segs).sum(1)
    assert O.flops(SMALL, counts, len(ids), 1) == tuple(g["flops_mixed"])


def test_c1_reuse_matches_reference():
    g = golden("c1_scene.npz")
    w = O.make_weights(C1)
    assert O.fingerprint(C1, w) == int(g["fingerprint"])
    T, V = 256, 4096
    imgs = O.images(1, C1.side, 1)
    enc, kv = {}, {}
    ids0, segs0 = O.layout(O.prompt(V, 8, 11), 1, T)
    O.fill_one(C1, w, ids0, segs0, imgs, enc, kv)
    text = O.prompt(V, 32, 12)
    ids, segs = O.layout(text[:16], 1, T, text[16:])
    out = O.reuse_prefill(C1, w, ids, segs, [O.sha256_hex(imgs[0])], (0.05,) * 4, enc, kv)
    assert np.array_equal(out.rows, g["rows"])
    assert out.counts == list(g["counts"])
    assert rel_err(out.logits, g["logits"]) <= 1e-5
    for l in (0, 3):
        assert rel_err(out.keys[l], g[f"keys_l{l}"]) <= 1e-5
        assert rel_err(out.values[l], g[f"values_l{l}"]) <= 1e-5


def test_masks_and_planner_match_reference():
    g = golden("plans_masks.npz")
    for key in g.files:
        if key.endswith("_mask"):
            t = key[:-5]
            pre, nimg, suf, T = (int(v) for v in g[t + "_layout"])
            ids, segs = O.layout(list(range(1, pre + 1)), nimg, T, list(range(suf)))
            assert np.array_equal(O.compute_masks(tuple(g[t + "_ratios"]), len(ids), segs), g[key])
        if key.endswith("_greedy"):
            t = key[:-7]
            base, p = g[t + "_meta"]
            grid = tuple(float(x) for x in g[t + "_grid"])
            assert O.greedy(g[t + "_scores"], grid, base, p) == tuple(g[key])
            if t + "_brute" in g.files:
                assert O.brute(g[t + "_scores"], grid, base, p) == tuple(g[t + "_brute"])
    grid = tuple(float(x) for x in g["c2_grid"])
    assert O.greedy(g["c2_table"], grid, 1.0, 0.03 * 28) == tuple(g["c2_plan"])


def test_decode_pins(small):
    """Oracle decode (engine.py:204-232) against the reference: generate golden of the small scene
    (full prefill + 8 greedy steps) and the pinned continuation after the mismatched-prefix r=0
    reuse (test_engine.py:177-184)."""
    g, w, enc, kv = small
    ids, segs = O.layout(list(g["prefix"]), 1, 16, list(g["suffix"]))
    logits, K, V = O.dense_prefill(SMALL, w, ids, segs, [g["emb"]])
    got, step_logits, _ = O.decode(SMALL, w, K, V, max_new=8, initial_logits=logits[-1])
    assert got == list(g["generate_ids"])
    assert [int(np.argmax(r)) for r in step_logits] == got
    got2, _, _ = O.decode(SMALL, w, g["r0_mis_keys"], g["r0_mis_values"], max_new=8,
                          initial_logits=g["r0_mis_logits"][-1])
    assert got2 == [92, 3, 88, 83, 83, 83, 83, 83]


def test_decode_teacher_forced_tail_matches_prefill(small):
    """Tail tokens teacher-forced over a shorter prefill reproduce the longer prefill's rows."""
    g, w, _, _ = small
    suffix = list(g["suffix"])
    ids, segs = O.layout(list(g["prefix"]), 1, 16)
    _, K, V = O.dense_prefill(SMALL, w, ids, segs, [g["emb"]])
    _, _, tail = O.decode(SMALL, w, K, V, tail_ids=suffix)
    ids_full, segs_full = O.layout(list(g["prefix"]), 1, 16, suffix)
    full, _, _ = O.dense_prefill(SMALL, w, ids_full, segs_full, [g["emb"]])
    assert rel_err(tail, full[-len(suffix):]) <= 1e-5


def test_forward_injected_matches_reuse_golden(small):
    """engine.py:239-283 restated: the dense injected path with the plan's stale mask reproduces the
    reference's skip-path logits at the computed rows (test_engine.py:65-80)."""
    g, w, enc, kv = small
    ids, segs = O.layout(O.prompt(97, 6, 99), 1, 16, list(g["suffix"]))
    n = len(ids)
    h = O.sha256_hex(g["img"])
    ik = np.zeros((4, n, 32), np.float32)
    iv = np.zeros_like(ik)
    start = O.image_spans(segs)[0][0]
    ik[:, start:start + 16], iv[:, start:start + 16] = kv[h].keys, kv[h].values
    uc = ~O.compute_masks((0.3, 0.2, 0.1, 0.0), n, segs)
    uc[:, :start] = False
    uc[:, start + 16:] = False
    logits, caps = O.forward_injected(SMALL, w, ids, segs, [g["emb"]], ik, iv, uc, capture_layers=(1, -1))
    rows = g["mixed_mis_rows"]
    assert rel_err(logits[rows], g["mixed_mis_logits"]) <= 1e-5
    assert sorted(caps) == [1, 3] and caps[1].shape == (n, 32)


def test_profile_fixture_pinned():
    """sensitivity.py:156-178 restated; the reference's regression pin (test_sensitivity.py:127-139)."""
    w = O.make_weights(SMALL)
    samples = [(O.image(16, 400 + k), O.prompt(97, 10, 500 + k), O.neutral_prompt(97, 10)) for k in range(5)]
    scores, base = O.profile(SMALL, w, samples, (0.1, 0.2, 0.3), max_new=6)
    assert base == pytest.approx(0.05434575974372617, rel=1e-6)
    expected = [[0.05434575974372617, 0.05434575974372617, 0.05434575974372617],
                [0.053952849361164124, 0.05491019159272694, 0.05474442593760177],
                [0.05204071848618812, 0.04659527542216396, 0.04360329238478551],
                [0.051986565840154916, 0.04302598720114376, 0.04084225128826289]]
    assert np.allclose(scores, expected, rtol=1e-6)
