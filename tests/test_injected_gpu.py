"""Dense forward with injected KV (engine.py:239-283) and the sensitivity-profiling protocol
(sensitivity.py:88-178) on the device, against the oracle restatements that are pinned to the
reference (tests/test_oracle_golden.py: skip-path equality, profile fixture pin)."""
import numpy as np
import pytest

from conftest import golden, rel_err
from oracle import kvreuse_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SMALL = dict(num_layers=4, num_heads=2, model_dim=32, kv_dim=32, vocab_size=97, patch_size=4,
             tokens_per_image=16, seed=7)


@pytest.fixture(scope="module")
def scene(cuda_ok):
    import paper_2512_12977_b200 as P
    oc = O.Cfg(**SMALL)
    w = {k: O.bf16_round(v) for k, v in O.make_weights(oc).items()}
    return P, oc, w, P.ToyVLM(P.ModelConfig(**SMALL), w)


def test_injected_matches_oracle_and_skip_path(scene):
    P, oc, w, model = scene
    g = golden("small_scene.npz")
    enc, kv = {}, {}
    ids0, segs0 = O.layout(list(g["prefix"]), 1, 16)
    O.fill_one(oc, w, ids0, segs0, [g["img"]], enc, kv)
    h = O.sha256_hex(g["img"])
    prefix, suffix = O.prompt(97, 6, 99), list(g["suffix"])
    ids, segs = O.layout(prefix, 1, 16, suffix)
    n = len(ids)
    seq = P.make_sequence(prefix, 1, 16, suffix)
    plan = P.RecomputePlan((0.3, 0.2, 0.1, 0.0))
    uc = P.plan_to_use_cached(plan, seq)
    ik = np.zeros((4, n, 32), np.float32)
    iv = np.zeros_like(ik)
    ik[:, 6:22], iv[:, 6:22] = kv[h].keys, kv[h].values
    ref, ref_caps = O.forward_injected(oc, w, ids, segs, [enc[h]], ik, iv, uc, capture_layers=(1, -1))
    got, caps = P.forward_injected(model, seq, [enc[h]], ik, iv, uc, capture_layers=(1, -1))
    assert rel_err(got, ref) <= 2e-2
    assert sorted(caps) == [1, 3]
    for i in (1, 3):
        assert rel_err(caps[i], ref_caps[i]) <= 2e-2
    # the skip path (prefill_with_reuse) equals the injected path at its computed rows
    store = P.CacheStore()
    store.put_encoder(P.EncoderCacheEntry(P.ImageHash(h), enc[h], model.fingerprint))
    store.put_kv(P.KVCacheEntry(P.ImageHash(h), kv[h].keys, kv[h].values, 6, model.fingerprint))
    res = P.prefill_with_reuse(model, P.ReuseRequest(seq, [P.ImageHash(h)], plan), store)
    assert rel_err(res.logits, got[res.positions]) <= 2e-2
    # no mask = dense prefill
    dense, _ = P.prefill_full(model, seq, [enc[h]])
    plain, _ = P.forward_injected(model, seq, [enc[h]])
    assert rel_err(plain, dense) <= 1e-5
    with pytest.raises(P.InputError):
        P.forward_injected(model, seq, [enc[h]], use_cached=uc)


def test_profile_matches_oracle(scene):
    """Device sensitivity profile vs the oracle's (pinned to the reference fixture on fp32 weights)
    on the same bf16 weights; the allocator's plan from either table is the same."""
    P, oc, w, model = scene
    from paper_2512_12977_b200 import sensitivity as S
    samples = [(O.image(16, 400 + k), O.prompt(97, 10, 500 + k), O.neutral_prompt(97, 10)) for k in range(3)]
    grid = (0.1, 0.2, 0.3)
    ref_scores, ref_base = O.profile(oc, w, samples, grid, max_new=6)
    table = S.profile(model, [S.ProxySample(*s) for s in samples], grid, max_new=6)
    assert table.baseline == pytest.approx(ref_base, rel=0.1)
    assert np.allclose(table.scores, ref_scores, rtol=0.1, atol=1e-3)
    # control: identical prompts -> no mismatch anywhere
    ctrl = S.profile(model, [S.ProxySample(O.image(16, 200), O.prompt(97, 10, 300), O.prompt(97, 10, 300))],
                     (0.1,), max_new=4)
    assert ctrl.baseline <= 1e-3 and float(ctrl.scores.max()) <= 1e-3
    ref_table = P.SensitivityTable(ref_scores, grid, ref_base, 3, model.fingerprint)
    budget = P.BudgetSpec(0.3)
    assert P.plan_greedy(table, budget).ratios == P.plan_greedy(ref_table, budget).ratios
