"""CPU oracle for the VLCache cache-reuse prefill path -- TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy float32, the arithmetic of the reference
package `kvreuse` 0.1.0 (/root/reference/pkg/src/kvreuse) on the hot path named
by BASELINE.json's north_star.  Every function cites the reference file:line it
follows.  It is the *checker*: only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import it.  The
product package `paper_2512_12977_b200` never imports it and has no CPU
fallback.

Parity pinning: `tests/golden/make_golden.py` runs the real reference (importable
in the build container from /root/reference/pkg/src) and commits its outputs to
`tests/golden/*.npz`; `tests/test_oracle_golden.py` checks this restatement
against those vectors plus the reference's own known-answer pins (sha256
vectors, decode ids, MSE regression value, encoder head values).  Status:
parity PINNED against the reference.

Layout of the restatement (no classes beyond small records, to keep it a
restatement rather than a copy):
  * sequences / plans / masks        plans.py:21-114, model.py:35-106
  * weights + fingerprint            model.py:165-250
  * primitives                       model.py:129-163, 257-291
  * encoder / embeddings / dense     model.py:302-389
  * reuse prefill                    engine.py:119-190
  * work accounting                  engine.py:39-85
  * allocator                        planner.py:29-146, sensitivity.py:42-81
"""

from __future__ import annotations

import hashlib
import json
import math
from dataclasses import dataclass

import numpy as np

F32 = np.float32
EPS = F32(1e-6)                    # model.py:26
STEP = 0.002                       # plans.py:21
TOP = 0.300                        # plans.py:22


# --------------------------------------------------------------------------
# configuration record (config.py:47-92)

@dataclass(frozen=True)
class Cfg:
    num_layers: int
    num_heads: int
    model_dim: int
    kv_dim: int
    vocab_size: int
    patch_size: int
    tokens_per_image: int
    rope_base: float = 10000.0
    seed: int = 0

    @property
    def head_dim(self):            # config.py:81-83
        return self.kv_dim // self.num_heads

    @property
    def hidden(self):              # config.py:90-92
        return 2 * self.model_dim

    @property
    def side(self):                # config.py:85-88
        return self.patch_size * math.isqrt(self.tokens_per_image)

    def as_json(self):             # model.py:243-250 (same key set, sorted dump)
        return json.dumps({
            "num_layers": self.num_layers, "num_heads": self.num_heads,
            "model_dim": self.model_dim, "kv_dim": self.kv_dim,
            "vocab_size": self.vocab_size, "patch_size": self.patch_size,
            "tokens_per_image": self.tokens_per_image,
            "rope_base": self.rope_base, "seed": self.seed}, sort_keys=True)


# --------------------------------------------------------------------------
# token layout: list of (kind, start, length) with kind 'text' | 'image'
# (model.py:35-106; image positions carry id -1, model.py:47-48)

def layout(prefix, n_images, T, suffix=()):
    ids, segs = [], []
    if len(prefix):
        segs.append(("text", 0, len(prefix)))
        ids += [int(t) for t in prefix]
    for _ in range(n_images):
        segs.append(("image", len(ids), T))
        ids += [-1] * T
    if len(suffix):
        segs.append(("text", len(ids), len(suffix)))
        ids += [int(t) for t in suffix]
    return ids, segs


def image_spans(segs):
    return [(s, n) for kind, s, n in segs if kind == "image"]


# --------------------------------------------------------------------------
# plans and masks (plans.py:31-114)

def plan_problem(ratios, step=STEP):
    """First violation or None (plans.py:55-73)."""
    if len(ratios) == 0:
        return "plan has no layers"
    last = None
    for layer, r in enumerate(ratios, 1):
        if r < 0.0 or r > 1.0:
            return f"layer {layer}: ratio {r} outside [0, 1]"
        if r != 0.0 and r != 1.0:
            k = round(r / step)
            if not (1 <= k <= round(TOP / step) and abs(r - k * step) <= 1e-9):
                return f"layer {layer}: ratio {r} off the grid"
        if last is not None and r > last + 1e-12:
            return f"layer {layer}: ratio {r} exceeds layer {layer - 1}'s {last}"
        last = r
    return None


def grid_units(r, step=STEP):
    """plans.py:31-38; raises ValueError off-grid."""
    if r == 0.0:
        return 0
    k = round(r / step)
    if k < 1 or abs(r - k * step) > 1e-9:
        raise ValueError(f"ratio {r} off grid")
    return int(k)


def keep_count(r, T):
    """plans.py:89-90."""
    return math.floor(r * T + 1e-9)


def compute_masks(ratios, n, segs):
    """bool [L, n]; plans.py:104-114."""
    m = np.ones((len(ratios), n), dtype=bool)
    for start, length in image_spans(segs):
        for layer, r in enumerate(ratios):
            m[layer, start + keep_count(r, length):start + length] = False
    return m


# --------------------------------------------------------------------------
# weights (model.py:165-210) and fingerprint (model.py:221-240)

_BLOCK = ("attn_norm", "wq", "wk", "wv", "wo", "mlp_norm", "w_gate", "w_up", "w_down")


def make_weights(cfg: Cfg):
    """Draw order must follow model.py:173-195 exactly (single PCG64 stream)."""
    g = np.random.default_rng(np.random.PCG64(cfg.seed))
    d, kv, h = cfg.model_dim, cfg.kv_dim, cfg.hidden
    pp = cfg.patch_size ** 2

    def scaled(shape, fan):
        return (g.standard_normal(shape) / np.sqrt(fan)).astype(F32)

    def block():
        out = {}
        for name in _BLOCK:                      # model.py:198-210
            if name.endswith("norm"):
                out[name] = np.ones(d, F32)
                continue
            shape, fan = {"wq": ((d, kv), d), "wk": ((d, kv), d), "wv": ((d, kv), d),
                          "wo": ((kv, d), kv), "w_gate": ((d, h), d),
                          "w_up": ((d, h), d), "w_down": ((h, d), h)}[name]
            out[name] = scaled(shape, fan)
        return out

    w = {"embed": g.standard_normal((cfg.vocab_size, d)).astype(F32)}
    w["head"] = scaled((d, cfg.vocab_size), d)
    w["final_norm"] = np.ones(d, F32)
    w["enc_patch_w"] = scaled((pp, d), pp)
    w["enc_patch_b"] = scaled((d,), d)
    w["enc_pos"] = g.standard_normal((cfg.tokens_per_image, d)).astype(F32)
    w["enc_out_norm"] = np.ones(d, F32)
    for k, v in block().items():
        w["enc_" + k] = v
    for i in range(cfg.num_layers):
        for k, v in block().items():
            w[f"l{i}_{k}"] = v
    return w


def fingerprint(cfg: Cfg, w):
    """First 8 bytes of sha256(config json + sorted name/bytes), big endian."""
    s = hashlib.sha256(cfg.as_json().encode())
    for name in sorted(w):
        s.update(name.encode())
        s.update(w[name].tobytes())
    return int.from_bytes(bytes.fromhex(s.hexdigest())[:8], "big")


def bf16_round(a):
    """Round-to-nearest-even to bfloat16, returned as float32 (test helper)."""
    u = np.ascontiguousarray(a, dtype=F32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(F32).reshape(np.shape(a))


# --------------------------------------------------------------------------
# primitives

def rope_tables(pos, hd, base):
    """model.py:129-134: fp32 inv_freq, fp32 angles, fp32 cos/sin."""
    half = hd // 2
    inv = base ** (-np.arange(half, dtype=F32) * (2.0 / hd))
    ang = np.asarray(pos, dtype=F32)[..., None] * inv
    return np.cos(ang, dtype=F32), np.sin(ang, dtype=F32)


def rope(x, pos, hd, base):
    """Half-split rotation of every head block (model.py:137-163)."""
    x = np.asarray(x, dtype=F32)
    p = np.atleast_1d(np.asarray(pos))
    if p.shape[0] == 1 and x.shape[0] != 1:
        p = np.broadcast_to(p, (x.shape[0],))
    c, s = rope_tables(p, hd, base)
    n = x.shape[0]
    xh = x.reshape(n, -1, hd)
    lo, hi = xh[..., : hd // 2], xh[..., hd // 2:]
    c, s = c[:, None, :], s[:, None, :]
    return np.concatenate((lo * c - hi * s, hi * c + lo * s), axis=-1).reshape(x.shape).astype(F32)


def rmsnorm(x, g):
    """model.py:257-259."""
    return (x / np.sqrt(np.mean(np.square(x), axis=-1, keepdims=True) + EPS)) * g


def mlp(x, wg, wu, wd):
    """SwiGLU, silu(a) = a / (1 + exp(-a)) (model.py:262-265)."""
    a = x @ wg
    return ((a / (F32(1.0) + np.exp(-a))) * (x @ wu)) @ wd


def attend(q, k, v, visible, H):
    """Masked softmax attention, scores fp32 (model.py:268-291)."""
    nq, nk = q.shape[0], k.shape[0]
    hd = q.shape[1] // H
    qh = q.reshape(nq, H, hd).transpose(1, 0, 2)
    kh = k.reshape(nk, H, hd).transpose(1, 0, 2)
    vh = v.reshape(nk, H, hd).transpose(1, 0, 2)
    sc = qh @ kh.transpose(0, 2, 1)
    sc *= F32(1.0 / np.sqrt(hd))
    sc = np.where(visible[None], sc, F32(-np.inf))
    sc -= sc.max(axis=-1, keepdims=True)
    np.exp(sc, out=sc)
    sc /= sc.sum(axis=-1, keepdims=True)
    return (sc @ vh).transpose(1, 0, 2).reshape(nq, -1)


# --------------------------------------------------------------------------
# encoder, embeddings, dense prefill (model.py:302-389)

def encode(cfg: Cfg, w, pixels):
    px = np.asarray(pixels, dtype=F32)
    p = cfg.patch_size
    hh, ww = px.shape
    T = (hh // p) * (ww // p)
    if px.ndim != 2 or hh % p or ww % p or T != cfg.tokens_per_image:
        raise ValueError("bad pixel grid")
    pt = px.reshape(hh // p, p, ww // p, p).transpose(0, 2, 1, 3).reshape(T, p * p)
    x = pt @ w["enc_patch_w"] + w["enc_patch_b"] + w["enc_pos"]
    xn = rmsnorm(x, w["enc_attn_norm"])
    a = attend(xn @ w["enc_wq"], xn @ w["enc_wk"], xn @ w["enc_wv"],
               np.ones((T, T), dtype=bool), cfg.num_heads)
    x = x + a @ w["enc_wo"]
    x = x + mlp(rmsnorm(x, w["enc_mlp_norm"]), w["enc_w_gate"], w["enc_w_up"], w["enc_w_down"])
    return rmsnorm(x, w["enc_out_norm"]).astype(F32)


def embed(cfg: Cfg, w, ids, segs, image_embeds):
    """model.py:339-359."""
    x = np.zeros((len(ids), cfg.model_dim), dtype=F32)
    for pos, tok in enumerate(ids):
        if tok >= 0:
            x[pos] = w["embed"][tok]
    for (start, length), e in zip(image_spans(segs), image_embeds):
        x[start:start + length] = np.asarray(e, dtype=F32)
    return x


def _layer_w(w, i):
    return [w[f"l{i}_{k}"] for k in _BLOCK]


def dense_prefill(cfg: Cfg, w, ids, segs, image_embeds):
    """model.py:362-389: logits [n, V] and pre-RoPE K, V [L, n, kv]."""
    x = embed(cfg, w, ids, segs, image_embeds)
    n = x.shape[0]
    pos = np.arange(n)
    K = np.empty((cfg.num_layers, n, cfg.kv_dim), F32)
    V = np.empty_like(K)
    vis = np.tril(np.ones((n, n), dtype=bool))
    hd, base = cfg.head_dim, cfg.rope_base
    for i in range(cfg.num_layers):
        g1, wq, wk, wv, wo, g2, wg, wu, wd = _layer_w(w, i)
        xn = rmsnorm(x, g1)
        q, k, v = xn @ wq, xn @ wk, xn @ wv
        K[i], V[i] = k, v
        x = x + attend(rope(q, pos, hd, base), rope(k, pos, hd, base), v, vis,
                       cfg.num_heads) @ wo
        x = x + mlp(rmsnorm(x, g2), wg, wu, wd)
    logits = rmsnorm(x, w["final_norm"]) @ w["head"]
    return logits.astype(F32), K, V


# --------------------------------------------------------------------------
# store records used by the oracle (store.py:64-155 semantics: miss -> None)

@dataclass
class KVEntry:
    keys: np.ndarray        # [L, T, kv] pre-RoPE
    values: np.ndarray
    origin_position: int


def sha256_hex(arr):
    """store.py:43-51: sha256 of C-order raw bytes."""
    b = np.ascontiguousarray(arr)
    if b.size == 0:
        raise ValueError("empty")
    return hashlib.sha256(b.tobytes()).hexdigest()


def sha256_many(arrs):
    """store.py:54-61."""
    s = hashlib.sha256()
    for a in arrs:
        s.update(np.ascontiguousarray(a).tobytes())
    return s.hexdigest()


def fill_one(cfg, w, ids, segs, images, enc_store, kv_store):
    """Cache-miss fill of one request (bench.py:82-95)."""
    embs = [encode(cfg, w, px) for px in images]
    _, K, V = dense_prefill(cfg, w, ids, segs, embs)
    for (start, length), px, e in zip(image_spans(segs), images, embs):
        key = sha256_hex(px)
        enc_store[key] = e
        kv_store[key] = KVEntry(K[:, start:start + length].copy(),
                                V[:, start:start + length].copy(), start)
    return embs


# --------------------------------------------------------------------------
# reuse prefill (engine.py:119-190)

@dataclass
class ReuseOut:
    rows: np.ndarray
    logits: np.ndarray
    keys: np.ndarray
    values: np.ndarray
    counts: list
    encoder_misses: int
    fallback_images: int


def reuse_prefill(cfg: Cfg, w, ids, segs, hashes, ratios, enc_store, kv_store,
                  images=None, timings=None):
    """`timings` (optional dict) receives wall seconds of resolve / embed / each layer / head
    (used only by bench.py's bounded CPU-baseline sample)."""
    import time
    t_start = time.perf_counter()
    if plan_problem(ratios) is not None or len(ratios) != cfg.num_layers:
        raise ValueError("bad plan")
    spans = image_spans(segs)
    n, L, kvd = len(ids), cfg.num_layers, cfg.kv_dim
    mask = compute_masks(ratios, n, segs)
    Kc = np.zeros((L, n, kvd), F32)
    Vc = np.zeros_like(Kc)
    embs, misses, fallbacks = [], 0, 0
    for m, (start, length) in enumerate(spans):          # engine.py:140-159
        e = enc_store.get(hashes[m])
        if e is None:
            misses += 1
            if images is None or images[m] is None:
                raise KeyError("miss without pixels")
            e = encode(cfg, w, images[m])
        embs.append(e)
        ent = kv_store.get(hashes[m])
        if ent is not None:
            Kc[:, start:start + length] = ent.keys
            Vc[:, start:start + length] = ent.values
        elif not mask[:, start:start + length].all():
            fallbacks += 1
            mask[:, start:start + length] = True
    counts = [int(r.sum()) for r in mask]
    t_res = time.perf_counter()
    x_all = embed(cfg, w, ids, segs, embs)
    t_emb = time.perf_counter()
    per_layer = []
    allpos = np.arange(n)
    hd, base = cfg.head_dim, cfg.rope_base
    rows = None
    for i in range(L):                                    # engine.py:172-186
        g1, wq, wk, wv, wo, g2, wg, wu, wd = _layer_w(w, i)
        rows = np.flatnonzero(mask[i])
        x = x_all[rows]
        xn = rmsnorm(x, g1)
        q = xn @ wq
        Kc[i, rows] = xn @ wk
        Vc[i, rows] = xn @ wv
        a = attend(rope(q, rows, hd, base), rope(Kc[i], allpos, hd, base), Vc[i],
                   rows[:, None] >= allpos[None, :], cfg.num_heads)
        x = x + a @ wo
        x = x + mlp(rmsnorm(x, g2), wg, wu, wd)
        x_all[rows] = x
        per_layer.append(time.perf_counter())
    logits = (rmsnorm(x_all[rows], w["final_norm"]) @ w["head"]).astype(F32)
    if timings is not None:
        marks = [t_emb] + per_layer
        timings.update(resolve=t_res - t_start, embed=t_emb - t_res,
                       layers=[b - a for a, b in zip(marks[:-1], marks[1:])],
                       head=time.perf_counter() - marks[-1])
    return ReuseOut(rows, logits, Kc, Vc, counts, misses, fallbacks)


# --------------------------------------------------------------------------
# work accounting (engine.py:39-85)

# --------------------------------------------------------------------------
# dense forward with injected KV and the sensitivity protocol (engine.py:239-292,
# sensitivity.py:88-178)

def forward_injected(cfg: Cfg, w, ids, segs, image_embeds, inject_k=None, inject_v=None, use_cached=None,
                     capture_layers=()):
    """Teacher-forced dense forward; at (layer, position) with use_cached, attention sees the
    injected pre-RoPE K/V (rotated to the current position) instead of the fresh projections
    (engine.py:239-283).  Returns (logits [n, V], {layer: attention block output [n, d]})."""
    x = embed(cfg, w, ids, segs, image_embeds)
    n = x.shape[0]
    pos = np.arange(n)
    L = cfg.num_layers
    if use_cached is None:
        use_cached = np.zeros((L, n), dtype=bool)
    vis = np.tril(np.ones((n, n), dtype=bool))
    hd, base = cfg.head_dim, cfg.rope_base
    caps = {}
    for i in range(L):
        an, wq, wk, wv, wo, mn, wg, wu, wd = _layer_w(w, i)
        xn = rmsnorm(x, an)
        q, k, v = xn @ wq, xn @ wk, xn @ wv
        if use_cached[i].any():
            sel = use_cached[i][:, None]
            k = np.where(sel, inject_k[i], k)
            v = np.where(sel, inject_v[i], v)
        a = attend(rope(q, pos, hd, base), rope(k, pos, hd, base), v, vis, cfg.num_heads) @ wo
        if i in capture_layers or (i - L) in capture_layers:
            caps[i] = a
        x = x + a
        x = x + mlp(rmsnorm(x, mn), wg, wu, wd)
    return (rmsnorm(x, w["final_norm"]) @ w["head"]).astype(F32), caps


def neutral_prompt(V, length):
    """toydata.py:36-38 (fixed seed 0xD00D)."""
    return prompt(V, length, 0xD00D)


def profile(cfg: Cfg, w, samples, grid, max_new=8):
    """sensitivity.py:88-178: per sample, the image's KV under the neutral prompt, the greedy
    baseline under the original prompt, then teacher-forced logits with the neutral KV injected at
    every layer except the first floor(r*T) image tokens of the probed layer; mean logit MSE per
    (layer, ratio).  samples: [(image, original_prompt, neutral_prompt)].
    Returns (scores [L, |grid|] f64, baseline f64)."""
    grid = tuple(sorted(float(g) for g in grid))
    L, T = cfg.num_layers, cfg.tokens_per_image
    totals = np.zeros((L, len(grid)), np.float64)
    base_total = 0.0
    for img, orig, neutral in samples:
        emb = encode(cfg, w, img)
        ids_n, segs_n = layout(list(neutral), 1, T)
        _, Kn, Vn = dense_prefill(cfg, w, ids_n, segs_n, [emb])          # build_mismatched_kv
        s0 = image_spans(segs_n)[0][0]
        mk, mv = Kn[:, s0:s0 + T], Vn[:, s0:s0 + T]
        ids_o, segs_o = layout(list(orig), 1, T)                       # baseline_decode
        lo, Ko, Vo = dense_prefill(cfg, w, ids_o, segs_o, [emb])
        gen, z_orig, _ = decode(cfg, w, Ko, Vo, max_new=max_new, initial_logits=lo[-1])

        def reuse(layer, r):                                           # reuse_logits
            ids, segs = layout(list(orig), 1, T, gen)
            n = len(ids)
            start = image_spans(segs)[0][0]
            ik = np.zeros((L, n, cfg.kv_dim), F32)
            iv = np.zeros_like(ik)
            ik[:, start:start + T], iv[:, start:start + T] = mk, mv
            uc = np.zeros((L, n), dtype=bool)
            uc[:, start:start + T] = True
            uc[layer, start:start + keep_count(r, T)] = False
            lg, _ = forward_injected(cfg, w, ids, segs, [emb], ik, iv, uc)
            first = start + T - 1
            return lg[first:first + len(gen)]

        def mse(a, b):
            return float(np.mean(np.square(np.asarray(a, np.float64) - np.asarray(b, np.float64))))
        base_total += mse(z_orig, reuse(0, 0.0))
        for i in range(L):
            for j, r in enumerate(grid):
                totals[i, j] += mse(z_orig, reuse(i, r))
    return totals / len(samples), base_total / len(samples)


# --------------------------------------------------------------------------
# decode over merged KV (engine.py:204-232, model.py:392-464)

def decode(cfg: Cfg, w, keys, values, tail_ids=(), max_new=0, initial_logits=None):
    """Greedy decode attending over merged pre-RoPE KV [L, n0, kv]: keys rotated at their request
    positions once (model.py:403-411), each step appends one token at the next position
    (model.py:413-439); tail tokens teacher-forced first, then greedy (engine.py:204-232,
    model.py:442-456).  Returns (ids, step_logits, tail_logits)."""
    L, n0 = keys.shape[0], keys.shape[1]
    cap = n0 + len(tail_ids) + max_new
    hd, base = cfg.head_dim, cfg.rope_base
    k_rot = np.zeros((L, cap, cfg.kv_dim), F32)
    v = np.zeros_like(k_rot)
    for i in range(L):
        k_rot[i, :n0] = rope(keys[i], np.arange(n0), hd, base)
        v[i, :n0] = values[i]
    state = {"n": n0}

    def step(tok):
        pos = state["n"]
        x = w["embed"][tok].astype(F32).copy()
        for i in range(L):
            an, wq, wk, wv, wo, mn, wg, wu, wd = _layer_w(w, i)
            xn = rmsnorm(x, an)
            k_rot[i, pos] = rope((xn @ wk)[None], [pos], hd, base)[0]
            v[i, pos] = xn @ wv
            q = rope((xn @ wq)[None], [pos], hd, base)
            a = attend(q, k_rot[i, :pos + 1], v[i, :pos + 1], np.ones((1, pos + 1), dtype=bool), cfg.num_heads)[0]
            x = x + a @ wo
            x = x + mlp(rmsnorm(x, mn), wg, wu, wd)
        state["n"] += 1
        return (rmsnorm(x, w["final_norm"]) @ w["head"]).astype(F32)

    tail_logits = np.empty((len(tail_ids), cfg.vocab_size), F32)
    cur = initial_logits
    for j, tok in enumerate(tail_ids):
        cur = step(int(tok))
        tail_logits[j] = cur
    ids, step_logits = [], np.empty((max_new, cfg.vocab_size), F32)
    for t in range(max_new):
        step_logits[t] = cur
        tok = int(np.argmax(cur))
        ids.append(tok)
        cur = step(tok)
    return ids, step_logits, tail_logits


def flops(cfg: Cfg, counts, n, encoded_images=0):
    d, kv, h, T = cfg.model_dim, cfg.kv_dim, cfg.hidden, cfg.tokens_per_image

    def attn(c, keys):
        return 2 * (3 * c * d * kv + 2 * c * keys * kv + c * kv * d)

    def ffn(c):
        return 6 * c * d * h

    enc = 2 * T * cfg.patch_size ** 2 * d + attn(T, T) + ffn(T)
    return (encoded_images * enc, sum(attn(c, n) for c in counts), sum(ffn(c) for c in counts))


# --------------------------------------------------------------------------
# allocator (planner.py:29-146; table lookup sensitivity.py:71-78)

def table_score(scores, grid, baseline, layer, r):
    if r == 0.0:
        return float(baseline)
    for j, g in enumerate(grid):
        if abs(g - r) <= 1e-9:
            return float(scores[layer, j])
    raise KeyError(r)


def greedy(scores, grid, baseline, p_target):
    """Single-step raises, best (gain/cost, -layer), integer unit budget."""
    L = scores.shape[0]
    if p_target < 0 or p_target > L * max(grid) + 1e-9:
        raise ValueError("infeasible budget")
    units = [grid_units(g) for g in grid]
    cap = int((p_target + 1e-9) / STEP)
    lvl = [-1] * L
    used = 0

    def ratio(l):
        return grid[l] if l >= 0 else 0.0

    while True:
        pick = None
        for i in range(L):
            nx = lvl[i] + 1
            if nx >= len(grid):
                continue
            if i and grid[nx] > ratio(lvl[i - 1]) + 1e-12:
                continue
            cost = units[nx] - (units[lvl[i]] if lvl[i] >= 0 else 0)
            if used + cost > cap:
                continue
            gain = (table_score(scores, grid, baseline, i, ratio(lvl[i]))
                    - table_score(scores, grid, baseline, i, grid[nx]))
            if gain <= 0:
                continue
            key = (gain / cost, -i)
            if pick is None or key > pick[0]:
                pick = (key, i, cost)
        if pick is None:
            break
        lvl[pick[1]] += 1
        used += pick[2]
    return tuple(ratio(l) for l in lvl)


def brute(scores, grid, baseline, p_target):
    """Exhaustive minimiser, lexicographically smallest tie (planner.py:105-141)."""
    L = scores.shape[0]
    units = [grid_units(g) for g in grid]
    cap = int((p_target + 1e-9) / STEP)
    best = [None, None]

    def go(layer, top, used, obj, acc):
        if layer == L:
            if best[0] is None or obj < best[0] or (obj == best[0] and acc < best[1]):
                best[0], best[1] = obj, acc
            return
        for lv in range(-1, top + 1):
            c = units[lv] if lv >= 0 else 0
            if used + c > cap:
                break
            r = grid[lv] if lv >= 0 else 0.0
            go(layer + 1, lv, used + c, obj + table_score(scores, grid, baseline, layer, r),
               acc + (r,))

    go(0, len(grid) - 1, 0, 0.0, ())
    return best[1]


# --------------------------------------------------------------------------
# seeded inputs (toydata.py:12-24)

def image(side, seed):
    return np.random.default_rng(np.random.PCG64(seed)).random((side, side), dtype=F32)


def images(count, side, seed):
    return [image(side, seed * 1000 + i) for i in range(count)]


def prompt(V, length, seed):
    return [int(t) for t in np.random.default_rng(np.random.PCG64(seed)).integers(0, V, size=length)]


def rel_err(a, e):
    """conftest.py:25-28."""
    return float(np.max(np.abs(np.asarray(a) - np.asarray(e)))) / max(1e-6, float(np.max(np.abs(e))))
