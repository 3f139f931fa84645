"""Host-side logic of the drop-in (no GPU): plans, masks, allocator, hashing, sequences,
error contract and the device layout planner, each checked against the CPU oracle and
the reference's golden vectors / known-answer pins."""
import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2512_12977_b200 as P
from conftest import golden
from oracle import kvreuse_oracle as O
from paper_2512_12977_b200.layout import SRC_STORE, RequestSpec, build_layout
from paper_2512_12977_b200.plans import layer_keep

GRID = tuple(round((k + 1) * 0.002, 3) for k in range(150))


# ---------------------------------------------------------------- plans (plans.py:21-114)

def test_recompute_count_pins():
    # test_plans.py:45-49
    assert P.recompute_count(0.05, 256) == 12
    assert P.recompute_count(0.03, 1024) == 30
    assert P.recompute_count(0.3, 16) == 4
    assert P.recompute_count(1.0, 16) == 16
    assert P.recompute_count(0.0, 16) == 0
    for r in (0.02, 0.03, 0.04, 0.05):
        assert P.recompute_count(r, 1024) == O.keep_count(r, 1024)


def test_ratio_units_pins():
    from paper_2512_12977_b200.plans import ratio_units
    assert ratio_units(0.0) == 0
    assert ratio_units(0.002) == 1
    assert ratio_units(0.3) == 150
    with pytest.raises(P.PlanError):
        ratio_units(0.003)


@pytest.mark.parametrize("ratios,needle", [
    ((0.1, 0.2), "layer 2"), ((0.003,), "layer 1"), ((1.0, 0.5), "layer 2"), ((), "no layers"),
    ((0.302,), "layer 1"), ((-0.1,), "layer 1")])
def test_validate_plan_reports_first_violation(ratios, needle):
    msg = P.validate_plan(P.RecomputePlan(ratios))
    assert msg is not None and needle in msg
    with pytest.raises(P.PlanError):
        P.build_masks(P.RecomputePlan(ratios), P.make_sequence([1, 2], 1, 16))


def test_masks_match_reference_goldens():
    g = golden("plans_masks.npz")
    n = 0
    for key in g.files:
        if not key.endswith("_mask"):
            continue
        t = key[:-5]
        pre, nimg, suf, T = (int(v) for v in g[t + "_layout"])
        seq = P.make_sequence(list(range(1, pre + 1)), nimg, T, list(range(suf)))
        m = P.build_masks(P.RecomputePlan(tuple(float(r) for r in g[t + "_ratios"])), seq)
        assert np.array_equal(m.layers, g[key]), t
        n += 1
    assert n == 20


def test_engine_count_pins():
    # test_engine.py:144-151: plan (0.3,0.2,0.1,0.0) on T=16, 6+4 text -> [14,13,11,10], mean 0.15
    seq = P.make_sequence(list(range(6)), 1, 16, [1, 2, 3, 4])
    plan = P.RecomputePlan((0.3, 0.2, 0.1, 0.0))
    assert P.build_masks(plan, seq).computed_counts == [14, 13, 11, 10]
    assert P.mean_ratio(plan) == pytest.approx(0.15)
    # test_engine.py:49: r=0 positions = text only
    m = P.build_masks(P.plan_static(0.0, 4), seq)
    assert list(np.flatnonzero(m.layers[-1])) == [0, 1, 2, 3, 4, 5, 22, 23, 24, 25]


@settings(max_examples=60, deadline=None)
@given(st.lists(st.integers(0, 150), min_size=1, max_size=8), st.integers(0, 3), st.integers(0, 5),
       st.integers(0, 5), st.sampled_from([4, 16, 64]))
def test_masks_property_vs_oracle(units, nimg, pre, suf, T):
    ratios = tuple(sorted((u * 0.002 for u in units), reverse=True))
    ratios = tuple(round(r, 3) for r in ratios)
    seq = P.make_sequence(list(range(pre)), nimg, T, list(range(suf)))
    m = P.build_masks(P.RecomputePlan(ratios), seq).layers
    ids, segs = O.layout(list(range(pre)), nimg, T, list(range(suf)))
    assert np.array_equal(m, O.compute_masks(ratios, len(ids), segs))
    # invariants (test_plans.py:86-106): text always computed, nested across layers
    img = seq.image_mask()
    assert m[:, ~img].all()
    assert (m[1:] <= m[:-1]).all()


# ---------------------------------------------------------------- allocator (planner.py:29-146)

def _table(scores, grid, base):
    return P.SensitivityTable(np.asarray(scores), tuple(float(x) for x in grid), float(base), 1, 0)


def test_planner_matches_reference_goldens():
    g = golden("plans_masks.npz")
    n = 0
    for key in g.files:
        if not key.endswith("_greedy"):
            continue
        t = key[:-7]
        base, p = (float(v) for v in g[t + "_meta"])
        tab = _table(g[t + "_scores"], g[t + "_grid"], base)
        assert P.plan_greedy(tab, P.BudgetSpec(p)).ratios == tuple(float(v) for v in g[key]), t
        if t + "_brute" in g.files:
            assert P.plan_bruteforce(tab, P.BudgetSpec(p)).ratios == tuple(float(v) for v in g[t + "_brute"]), t
        n += 1
    assert n == 30
    tab = _table(g["c2_table"], g["c2_grid"], 1.0)
    plan = P.plan_greedy(tab, P.BudgetSpec(0.03 * 28))
    assert plan.ratios == tuple(float(v) for v in g["c2_plan"])
    assert P.validate_plan(plan) is None


@settings(max_examples=40, deadline=None)
@given(st.integers(1, 5), st.integers(1, 4), st.integers(0, 2 ** 31 - 1), st.floats(0.0, 1.0))
def test_greedy_vs_oracle_random_tables(L, G, seed, frac):
    rng = np.random.default_rng(seed)
    grid = tuple(sorted(rng.choice(np.arange(1, 151), G, replace=False) * 0.002))
    grid = tuple(round(x, 3) for x in grid)
    scores = rng.random((L, G))
    base = 1.0 + rng.random()
    p = round(frac * L * max(grid), 6)
    tab = _table(scores, grid, base)
    got = P.plan_greedy(tab, P.BudgetSpec(p))
    assert got.ratios == O.greedy(scores, grid, base, p)
    brute = P.plan_bruteforce(tab, P.BudgetSpec(p))
    assert brute.ratios == O.brute(scores, grid, base, p)
    assert P.objective(tab, brute) <= P.objective(tab, got) + 1e-12


def test_planner_tie_break_and_budget_errors():
    # tie -> shallowest layer (test_planner.py:91-103)
    tab = _table([[0.5, 0.2], [0.5, 0.2]], (0.1, 0.2), 1.0)
    assert P.plan_greedy(tab, P.BudgetSpec(0.1)).ratios == (0.1, 0.0)
    with pytest.raises(P.InputError):
        P.plan_greedy(tab, P.BudgetSpec(-0.1))
    with pytest.raises(P.InputError):
        P.plan_greedy(tab, P.BudgetSpec(0.5))          # > L * max(grid)
    with pytest.raises(P.InputError):
        P.plan_greedy(tab, P.BudgetSpec(0.2, grid=(0.05,)))   # grid point not profiled


def test_sensitivity_table_contract():
    tab = _table([[0.3, 0.1]], (0.002, 0.004), 0.9)
    assert tab.score(0, 0.0) == 0.9
    assert tab.score(0, 0.004) == pytest.approx(0.1)
    with pytest.raises(P.InputError):
        tab.score(0, 0.006)
    with pytest.raises(P.InputError):
        _table([[0.3, 0.1]], (0.004, 0.002), 0.9)
    with pytest.raises(P.InputError):
        _table([[-0.3, 0.1]], (0.002, 0.004), 0.9)


# ---------------------------------------------------------------- hashing (store.py:29-61)

def test_hash_pins():
    # test_store.py:45-49 and :70-74
    assert P.hash_image(np.arange(4, dtype=np.uint8)).hex == \
        "054edec1d0211f624fed0cbca9d4f9400b0e491c43742af2c5b0abebf0c990d8"
    a = np.arange(4, dtype=np.uint8).reshape(2, 2)
    assert P.hash_request([a, a + 9]).hex == \
        "62fc9e9e103929bf2f07998578a063e5d66343e8ad009b976361947cfde871b3"
    assert P.hash_request([a, a + 9]) != P.hash_request([a + 9, a])        # order-sensitive
    g = golden("small_scene.npz")
    assert P.hash_image(g["img"]).hex == bytes(g["image_hash"]).hex()
    for bad in ("ABC", "0" * 63, "G" * 64):
        with pytest.raises(P.InputError):
            P.ImageHash(bad)
    with pytest.raises(P.InputError):
        P.hash_image(np.zeros(0, np.float32))


def test_hash_matches_oracle_on_toydata():
    from paper_2512_12977_b200.toydata import make_images
    for px, opx in zip(make_images(3, 64, 1), O.images(3, 64, 1)):
        assert np.array_equal(px, opx)
        assert P.hash_image(px).hex == O.sha256_hex(opx)


# ---------------------------------------------------------------- sequences / FLOPs / config

def test_sequence_validation_errors():
    seq = P.make_sequence([1, 2, 3], 2, 16, [4])
    assert len(seq) == 3 + 32 + 1
    assert [s.start for s in seq.image_segments] == [3, 19]
    with pytest.raises(P.InputError):
        seq.validate(8)
    bad = P.TokenSequence(seq.ids[:-1], seq.segments)
    with pytest.raises(P.InputError):
        bad.validate(16)


def test_count_flops_matches_reference_pin():
    g = golden("small_scene.npz")
    cfg = P.ModelConfig(num_layers=4, num_heads=2, model_dim=32, kv_dim=32, vocab_size=97, patch_size=4,
                        tokens_per_image=16, seed=7)
    seq = P.make_sequence(O.prompt(97, 6, 99), 1, 16, list(g["suffix"]))
    f = P.count_flops(seq, P.RecomputePlan((0.3, 0.2, 0.1, 0.0)), cfg, encoder_cached=False)
    assert (f.encoder, f.attention, f.mlp) == tuple(int(v) for v in g["flops_mixed"])


def test_model_config_and_fingerprint_match_reference():
    g = golden("small_scene.npz")
    cfg = P.ModelConfig(num_layers=4, num_heads=2, model_dim=32, kv_dim=32, vocab_size=97, patch_size=4,
                        tokens_per_image=16, seed=7)
    m = P.init_model(cfg)
    assert m.fingerprint == int(g["fingerprint"])
    with pytest.raises(P.ConfigError):
        P.ModelConfig(num_layers=4, num_heads=3, model_dim=32, kv_dim=32, vocab_size=97, patch_size=4,
                      tokens_per_image=16)
    with pytest.raises(P.ConfigError):
        P.ModelConfig(num_layers=4, num_heads=2, model_dim=32, kv_dim=32, vocab_size=97, patch_size=4,
                      tokens_per_image=15)


# ---------------------------------------------------------------- device layout planner (host side)

def _spec(pre, T, nimg, suf, ratios, hits=None):
    seq = P.make_sequence(list(range(1, pre + 1)), nimg, T, list(range(1, suf + 1)))
    plan = P.RecomputePlan(ratios)
    keep = np.repeat(layer_keep(plan, T)[:, None], nimg, axis=1).astype(np.int32)
    hits = hits if hits is not None else [True] * nimg
    for m, h in enumerate(hits):
        if not h:
            keep[:, m] = T
    segs = seq.image_segments
    L = len(ratios)
    tpos = np.array([p for s in seq.segments if s.kind == "text" for p in range(s.start, s.start + s.length)])
    pages = [np.arange(L * -(-T // 64), dtype=np.int32).reshape(L, -1) + 1000 * m if h else None
             for m, h in enumerate(hits)]
    spec = RequestSpec(n=len(seq), text_pos=tpos, text_ids=tpos % 7,
                       images=[(s.start, s.length) for s in segs], keep=keep,
                       kv_hit=[bool(h and (keep[:, m] < T).any()) for m, h in enumerate(hits)],
                       enc_src=[(SRC_STORE, m * T) for m in range(nimg)], page_rows=pages)
    return seq, plan, spec


@pytest.mark.parametrize("pre,T,nimg,suf,ratios,hits", [
    (16, 256, 1, 16, (0.05,) * 4, None),
    (6, 16, 1, 4, (0.3, 0.2, 0.1, 0.0), None),
    (16, 64, 3, 16, (0.3, 0.1, 0.1, 0.0), [True, False, True]),
    (0, 64, 2, 0, (1.0, 1.0), None),
    (5, 16, 0, 0, (0.0, 0.0), None),
    (4, 32, 2, 4, (1.0, 0.1, 0.1, 0.0), None),     # full first layer, reuse below it
])
def test_layout_rows_match_masks(pre, T, nimg, suf, ratios, hits):
    seq, plan, spec = _spec(pre, T, nimg, suf, ratios, hits)
    L = len(ratios)
    lay = build_layout([spec], L, heads=2)
    masks = P.build_masks(plan, seq).layers.copy()
    for m, h in enumerate(hits or [True] * nimg):
        if not h:
            s = seq.image_segments[m]
            masks[:, s.start:s.start + s.length] = True
    for i in range(L):
        ci = int(lay.c[i])
        assert ci == masks[i].sum()
        # layer i works on the packed prefix [0, c_i): exactly the reference's rows
        assert sorted(lay.row_pos[:ci].tolist()) == list(np.flatnonzero(masks[i]))
        # queries of layer i are position-sorted and point back at prefix rows
        qp = lay.qpos[i, :ci]
        assert (np.diff(qp) >= 0).all()
    assert np.array_equal(lay.positions[0], np.flatnonzero(masks[-1]))
    # reused (layer, token) rows: the store chunks' rows are read in place by the attention, the
    # rest of each keep boundary's chunk is relocated (exactly once)
    from paper_2512_12977_b200.layout import relocated_ranges
    want = sum(e - k for i in range(L) for _, k, e in relocated_ranges(spec, i))
    assert lay.reloc_tokens == want
    store = sum(int(c[1]) & 0xFF for ch in lay.attn_chunks for c in ch if c[3] >= 0 and c[1] & 0xFF > 0)
    assert store + want == int((~masks).sum())


@pytest.mark.parametrize("nq,nkeys,heads,reqs", [(236, 4128, 28, 1), (62, 1056, 12, 1), (44, 288, 8, 1),
                                            (600, 4128, 1, 1), (300, 300, 4, 1), (40, 300, 8, 3)])
def test_attention_work_items_cover_every_visible_key(nq, nkeys, heads, reqs):
    """Work items of vlc_attn_paged: every (query tile, head) covers the 128-key tiles holding its
    causal keys [0, last query position] exactly once across its splits; query tiles are <= 128
    rows; split groups fit the co-residency budget (<= 148 CTAs) and <= 8 parts; the parts of a
    group have consecutive indices with the group size in every item."""
    import numpy as np
    from paper_2512_12977_b200.layout import attention_work, contiguous_chunks, tiles_needed
    rng = np.random.default_rng(nq + nkeys)
    ranges, qpos, q0, lists = [], [], 0, []
    for r in range(reqs):
        pos = np.sort(rng.permutation(nkeys)[:nq]).astype(np.int32)
        pos[-1] = nkeys - 1
        ranges.append((r, q0, nq))
        qpos.append(pos)
        lists.append(contiguous_chunks(r * nkeys, nkeys))
        q0 += nq
    qpos = np.concatenate(qpos)
    chunk0 = np.cumsum([0] + [len(x) for x in lists[:-1]])
    it, groups = attention_work(ranges, qpos, lambda r, p: tiles_needed(lists[r], p), chunk0, heads)
    assert (it[:, 1] <= 128).all() and (it[:, 1] > 0).all()
    if groups:
        assert len(it) <= 148
    parts = {}
    for row in it:
        t0, nqt, h, c0, tb, te, grp, pk = (int(v) for v in row)
        p, ns = pk >> 8, pk & 0xFF
        assert 1 <= ns <= 8 and 0 <= p < ns
        assert (grp < 0) == (ns == 1)
        parts.setdefault((c0, t0, h), []).append((tb, te, p, ns, nqt))
    for (c0, t0, h), lst in parts.items():
        req = int(np.searchsorted(chunk0, c0, side="right") - 1)
        lst.sort()
        ns = lst[0][3]
        assert len(lst) == ns and [x[2] for x in lst] == list(range(ns))
        assert lst[0][0] == 0
        for a, b in zip(lst, lst[1:]):
            assert a[1] == b[0]
        nqt = lst[0][4]
        last = int(qpos[t0 + nqt - 1])
        ch = lists[req]
        te = lst[-1][1]
        # the tiles reach the last visible key and stop at the first tile wholly past it
        assert ch[2 * te - 2:2 * te, 0].min() <= last
        assert 2 * te >= len(ch) or ch[2 * te, 0] > last
    for r, q0_, cnt in ranges:
        for h in range(heads):
            rows = sorted(t0 + i for (c0, t0, hh), lst in parts.items() if c0 == chunk0[r] and hh == h
                          for i in range(lst[0][4]))
            assert rows == list(range(q0_, q0_ + cnt))


@pytest.mark.parametrize("pre,T,nimg,suf,ratios,P", [
    (16, 1024, 4, 16, (0.05, 0.02, 0.0), 64), (16, 256, 2, 16, (0.3, 0.1, 0.0), 64),
    (6, 16, 1, 4, (0.3, 0.2, 0.1, 0.0), 16), (16, 256, 1, 16, (1.0, 0.25, 0.1), 128),
    (3, 300, 2, 5, (0.5, 0.2, 0.0), 64), (16, 256, 1, 16, (0.1, 0.0), 48)])
def test_key_chunks_cover_every_key_once(pre, T, nimg, suf, ratios, P):
    """vlc_attn_paged's key chunks of each layer: positions 0 .. n-1 exactly once, in order; a store
    chunk only for cached rows (t >= keep) that sit inside one page; every cached row of a hit
    image is either read from the store or relocated into the request rows -- never both, never
    neither -- and the relocated rows are exactly the cached rows of request-row chunks.  A store
    chunk carries its image's shift D = new start - cached start above the 8-bit length, and no 128-key
    tile pairs store chunks of two different shifts (the kernel rotates its queries once per tile)."""
    import numpy as np
    from paper_2512_12977_b200.layout import relocated_ranges, request_chunks
    seq, plan, spec = _spec(pre, T, nimg, suf, ratios, None)
    spec.page_tokens = P
    ppl = -(-T // P)
    spec.page_rows = [np.arange(len(ratios) * ppl, dtype=np.int32).reshape(len(ratios), ppl) for _ in range(nimg)]
    base = {m: m * len(ratios) * ppl for m in range(nimg)}
    # cached starts before and after the new ones: positive and negative shifts D
    spec.origin = [s0 + (8 - 13 * m) for m, (s0, _) in enumerate(spec.images)]
    for i in range(len(ratios)):
        ch = request_chunks(spec, i, 1000, base).copy()
        assert len(ch) % 2 == 0
        shift = ch[:, 1] >> 8
        ch[:, 1] &= 0xFF
        for a, b, sa, sb in zip(ch[0::2], ch[1::2], shift[0::2], shift[1::2]):
            if a[3] >= 0 and b[3] >= 0:
                assert sa == sb
        assert (np.diff(ch[:, 0]) >= 0).all()
        real = ch[ch[:, 1] > 0]
        rshift = shift[ch[:, 1] > 0]
        covered = np.concatenate([np.arange(c[0], c[0] + c[1]) for c in real])
        assert np.array_equal(covered, np.arange(spec.n))
        reloc = {m: (k, e) for m, k, e in relocated_ranges(spec, i)}
        for m, (start, Tm) in enumerate(spec.images):
            k = int(spec.keep[i, m])
            store_rows, req_rows = set(), set()
            for c, sh in zip(real, rshift):
                if not (start <= c[0] < start + Tm):
                    continue
                t = set(range(c[0] - start, c[0] - start + c[1]))
                if c[3] >= 0:
                    assert sh == start - spec.origin[m]
                    assert min(t) >= k and c[3] + c[1] <= P
                    assert c[2] == base[m] + i * ppl + (c[0] - start) // P
                    store_rows |= t
                else:
                    assert c[2] == 1000 + c[0]
                    req_rows |= t
            cached = set(range(k, Tm))
            relocated = set(range(*reloc[m])) if m in reloc else set()
            assert store_rows.isdisjoint(relocated) and store_rows | relocated == cached
            assert relocated == cached & req_rows


def test_int_pack_template_and_patches():
    """Per-call metadata: the structural template is shared and left unmodified; the per-call
    segments (token ids / page ids) travel as patches that the full upload applies."""
    import numpy as np
    from paper_2512_12977_b200.runtime import IntPack
    pk = IntPack()
    pk.add("src", np.arange(10))
    pk.add("pages", np.arange(5) + 100)
    pk.add("rest", np.arange(7) + 1000)
    tpl = np.concatenate(pk.parts)
    q = IntPack()
    q.host, q.off = tpl, dict(pk.off)
    q.patches = {"src": np.full(10, -1, np.int32), "pages": np.full(5, -2, np.int32)}
    full = q._full_host()
    o, n = q.off["src"]
    assert (full[o:o + n] == -1).all()
    o, n = q.off["pages"]
    assert (full[o:o + n] == -2).all()
    o, n = q.off["rest"]
    assert (full[o:o + n] == np.arange(7) + 1000).all()
    assert (tpl == np.concatenate(pk.parts)).all()          # template untouched
    # every view keeps 16-byte alignment
    assert all(off % 4 == 0 for off, _ in q.off.values())


def test_reuse_result_is_freed_without_gc():
    """A dropped ReuseResult must die by reference count: the runner keeps only weak references
    to live results and copies out (detaches) those still alive when their workspace set comes
    round again -- a reference cycle would keep every result alive until a GC pass and make each
    call copy the previous result's logits and merged KV."""
    import gc
    import threading
    import weakref
    from paper_2512_12977_b200.engine import ReuseMetrics, ReuseResult
    from paper_2512_12977_b200.model import KVTensors
    gc.disable()
    try:
        res = ReuseResult(np.arange(3), object(), KVTensors(loader=lambda: (None, None)), ReuseMetrics(),
                          threading.RLock())
        ref = weakref.ref(res)
        del res
        assert ref() is None
    finally:
        gc.enable()


def test_query_tiles_minimise_scanned_key_tiles():
    """layout.query_tiles: exact minimum of sum(key tiles of each tile's last query) + 1 per tile
    over every cut into <= rows-row tiles (brute force on small cases); C3 at 5% cuts at the gap
    before image 2 instead of at row 128 (45 instead of 53 key tiles per head)."""
    import itertools

    import numpy as np
    from paper_2512_12977_b200.layout import query_tiles
    rng = np.random.default_rng(5)
    for _ in range(40):
        n, rows = int(rng.integers(1, 11)), int(rng.integers(1, 5))
        pos = np.sort(rng.choice(200, n, replace=False))
        tiles = lambda p: p // 16 + 1          # noqa: E731
        got = query_tiles(pos, tiles, rows=rows)
        assert got[0][0] == 0 and got[-1][1] == n and all(b - a <= rows for a, b in got)
        assert all(x[1] == y[0] for x, y in zip(got, got[1:]))
        best = min(sum(tiles(pos[b - 1]) + 1 for a, b in zip((0,) + c, c + (n,)))
                   for k in range(n) for c in itertools.combinations(range(1, n), k)
                   if all(b - a <= rows for a, b in zip((0,) + c, c + (n,))))
        assert sum(tiles(pos[b - 1]) + 1 for a, b in got) == best
    # C3: 16 text + 4 images x 51 leading tokens (+ their store / request split chunk) + 16 text
    pos = np.concatenate([np.arange(16), 16 + np.arange(51), 1040 + np.arange(51), 2064 + np.arange(51),
                          3088 + np.arange(51), 4112 + np.arange(16)])
    tiles = lambda p: -(-(p // 64 + 1 + (p > 66) + (p > 1090) + (p > 2114) + (p > 3138)) // 2)   # noqa: E731
    got = query_tiles(pos, tiles)
    assert sum(tiles(pos[b - 1]) for a, b in got) == 44 and len(got) == 2
    assert tiles(pos[127]) + tiles(pos[-1]) == 53
