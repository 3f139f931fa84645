"""Store persistence interop on the GPU: a store persisted by the REAL reference loads into the
HBM store and drives a reuse prefill that matches the oracle; our persist round-trips."""
import json

import numpy as np
import pytest

from conftest import GOLDEN, golden, rel_err
from oracle import kvreuse_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SMALL = dict(num_layers=4, num_heads=2, model_dim=32, kv_dim=32, vocab_size=97, patch_size=4,
             tokens_per_image=16, seed=7)


def test_load_reference_store_and_reuse(cuda_ok, tmp_path):
    import os
    import paper_2512_12977_b200 as P
    store = P.CacheStore.load(os.path.join(GOLDEN, "ref_store"))
    oc = O.Cfg(**SMALL)
    w = O.make_weights(oc)                                   # reference fp32 weights: fingerprint matches
    model = P.ToyVLM(P.ModelConfig(**SMALL), w)
    g = golden("small_scene.npz")
    h = P.hash_image(g["img"])
    enc, kvs = {}, {}
    ids0, segs0 = O.layout(list(g["prefix"]), 1, 16)
    O.fill_one(oc, w, ids0, segs0, [g["img"]], enc, kvs)
    e = store.get_encoder(h, expected_fingerprint=model.fingerprint)
    assert np.array_equal(e.embeddings, enc[h.hex])          # fp32 slots: exact
    kv = store.get_kv(h, expected_fingerprint=model.fingerprint)
    assert kv.origin_position == 6
    assert rel_err(kv.keys, kvs[h.hex].keys) <= 4e-3         # bf16 pages
    assert rel_err(kv.values, kvs[h.hex].values) <= 4e-3
    with pytest.raises(P.StaleCacheError):
        store.get_kv(h, expected_fingerprint=model.fingerprint ^ 1)
    # reuse prefill from the loaded store vs the oracle on the same cached data
    text = O.prompt(97, 10, 4)
    ids, segs = O.layout(text[:6], 1, 16, text[6:])
    w_b = {k: O.bf16_round(v) for k, v in w.items()}          # what the device computes with
    ref = O.reuse_prefill(oc, w_b, ids, segs, [h.hex], (0.3, 0.2, 0.1, 0.0), enc, kvs)
    got = P.prefill_with_reuse(model, P.ReuseRequest(P.make_sequence(text[:6], 1, 16, text[6:]), [h],
                                                     P.RecomputePlan((0.3, 0.2, 0.1, 0.0))), store)
    assert np.array_equal(got.positions, ref.rows)
    assert rel_err(got.logits, ref.logits) <= 2e-2
    # our persist writes the reference format and round-trips
    out = tmp_path / "ours"
    store.persist(out)
    m = json.loads((out / "manifest.json").read_text())
    ref_m = json.loads(open(os.path.join(GOLDEN, "ref_store", "manifest.json")).read())
    assert m["format"] == ref_m["format"] and sorted(m["entries"]) == sorted(ref_m["entries"])
    enc_key = f"encoder/{h.hex}"
    assert m["entries"][enc_key]["sha256"] == ref_m["entries"][enc_key]["sha256"]   # fp32 embeddings identical
    back = P.CacheStore.load(out)
    assert np.array_equal(back.get_kv(h).keys, kv.keys)
    assert np.array_equal(back.get_encoder(h).embeddings, e.embeddings)
