"""Decode over merged KV on the device (reference engine.py:204-232, model.py:392-464) against the
oracle's restatement (pinned to the reference's generate golden and the mismatched-reuse
continuation in tests/test_oracle_golden.py)."""
import numpy as np
import pytest

from conftest import golden, rel_err
from oracle import kvreuse_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SMALL = dict(num_layers=4, num_heads=2, model_dim=32, kv_dim=32, vocab_size=97, patch_size=4,
             tokens_per_image=16, seed=7)
C1 = dict(num_layers=4, num_heads=8, model_dim=256, kv_dim=256, vocab_size=4096, patch_size=4,
          tokens_per_image=256, seed=0)


def _setup(kw, prefix, suffix, img):
    import paper_2512_12977_b200 as P
    oc = O.Cfg(**kw)
    w = {k: O.bf16_round(v) for k, v in O.make_weights(oc).items()}
    model = P.ToyVLM(P.ModelConfig(**kw), w)
    T = oc.tokens_per_image
    enc, kv = {}, {}
    ids0, segs0 = O.layout(prefix, 1, T)
    O.fill_one(oc, w, ids0, segs0, [img], enc, kv)
    h = O.sha256_hex(img)
    store = P.CacheStore()
    store.put_encoder(P.EncoderCacheEntry(P.ImageHash(h), enc[h], model.fingerprint))
    store.put_kv(P.KVCacheEntry(P.ImageHash(h), kv[h].keys, kv[h].values, len(prefix), model.fingerprint))
    return P, oc, w, model, store, enc, kv, h


@pytest.mark.parametrize("kw,steps", [(SMALL, 8), (C1, 6)])
def test_decode_after_reuse_matches_oracle(cuda_ok, kw, steps):
    g = golden("small_scene.npz")
    V, T = kw["vocab_size"], kw["tokens_per_image"]
    img = g["img"] if kw is SMALL else O.images(1, 4 * 16, 1)[0]
    prefix = list(g["prefix"]) if kw is SMALL else O.prompt(V, 8, 11)
    P, oc, w, model, store, enc, kv, h = _setup(kw, prefix, None, img)
    text = O.prompt(V, 10, 99)
    ids, segs = O.layout(text[:6], 1, T, text[6:])
    plan = (0.0,) * kw["num_layers"]
    ref = O.reuse_prefill(oc, w, ids, segs, [h], plan, enc, kv)
    ref_ids, ref_steps, _ = O.decode(oc, w, ref.keys, ref.values, max_new=steps, initial_logits=ref.logits[-1])
    res = P.prefill_with_reuse(model, P.ReuseRequest(P.make_sequence(text[:6], 1, T, text[6:]), [P.ImageHash(h)],
                                                     P.RecomputePlan(plan)), store)
    # (a) same merged KV as the oracle, the oracle's greedy tokens teacher-forced: every step's
    # distribution within tolerance (greedy ids themselves may flip at a near-tie after a few
    # steps: bf16 KV vs the fp32 oracle)
    forced = P.decode_with_merged_kv(model, P.KVTensors(ref.keys, ref.values), tail_ids=ref_ids[:-1])
    assert rel_err(forced.tail_logits, ref_steps[1:]) <= 2e-2
    for got_row, ref_row, ref_id in zip(forced.tail_logits, ref_steps[1:], ref_ids[1:]):
        if _margin(ref_row) > 5e-3:                    # a decided step: same greedy token
            assert int(np.argmax(got_row)) == ref_id
    # (b) the whole device pipeline: reuse prefill -> greedy decode from its own merged KV and last
    # row; ids agree with the oracle's up to the first near-tie of the oracle's distribution
    dec = P.decode_with_merged_kv(model, res.kv, max_new=steps, initial_logits=res.logits[-1])
    k = _first_tie(ref_steps, tol=5e-3)
    assert dec.ids[:k] == ref_ids[:k], (k, dec.ids, ref_ids)
    assert rel_err(dec.step_logits[:max(k, 1)], ref_steps[:max(k, 1)]) <= 2e-2


def _margin(row):
    top = np.sort(row)[-2:]
    return float(top[1] - top[0]) / float(np.abs(row).max())


def _first_tie(steps, tol=2e-2):
    for t, row in enumerate(steps):
        if _margin(row) <= tol:
            return t
    return len(steps)
