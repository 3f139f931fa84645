"""Host planning of one reuse-prefill launch (pure numpy; no device needed).

The reference recomputes, at layer i, the rows `flatnonzero(mask[i])` and keeps
one hidden state per position (engine.py:166-186).  On the device the hidden
states of the computed tokens are PACKED so that every layer's computed set is a
PREFIX of one buffer: tokens are ordered by how many layers they survive
(text: all L; image token t of image m: #{i : keep[i][m] > t}, a prefix of the
layers because keep is non-increasing), then by (request, position).  Layer i
then works on rows [0, c_i) -- no gathers or scatters of hidden states between
layers.  Attention needs queries ordered by position per request (causal
masking by absolute position, reference `rows[:, None] >= positions[None, :]`),
so each layer also gets a sorted query order (qdst / qpos / rowof).

Everything here depends only on (sequence layout, plan, which images hit the KV
cache), so it is cached and reused across requests with the same structure.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import os

import numpy as np

SRC_TEXT, SRC_STORE, SRC_SCRATCH = 0, 1, 2


@dataclass
class RequestSpec:
    n: int                        # sequence length
    text_pos: np.ndarray          # positions of text tokens
    text_ids: np.ndarray          # their ids
    images: list                  # [(start, T)] per image segment
    keep: np.ndarray              # int32 [L, n_images] recomputed leading tokens per layer
    kv_hit: list                  # per image: True if cached KV is reused (relocated)
    enc_src: list                 # per image: (SRC_STORE|SRC_SCRATCH, row base)
    page_rows: list = field(default_factory=list)  # per image: int32 [L, ppl] page ids (kv_hit only)


@dataclass
class Layout:
    L: int
    heads: int
    c: np.ndarray                 # int32 [L] computed rows per layer (prefix lengths)
    kv_rows: int                  # total KV-cache rows (sum of n)
    kvoff: np.ndarray             # int32 [R] first KV row of each request
    # per packed row (length c[0])
    row_req: np.ndarray
    row_pos: np.ndarray
    row_kv: np.ndarray
    row_src: np.ndarray           # int32 [c0, 2] (kind, index)
    # per layer sorted query order: [L, c0] (only first c[i] meaningful)
    qdst: np.ndarray
    qpos: np.ndarray
    rowof: np.ndarray
    q_ranges: list                # per layer: list of (req, q0, count)
    # attention work (per layer) + combine entries
    attn_items: list              # per layer: int32 [n, 8]
    comb_items: list              # per layer: int32 [m, 8]
    attn_slots: int               # max partial slots over layers
    # relocation
    reloc_descs: np.ndarray       # int32 [d, 8]
    reloc_blocks: np.ndarray      # int32 [b, 2]
    reloc_layer_blocks: np.ndarray  # int32 [L+1] block offsets per layer (descs sorted by layer)
    reloc_tokens: int             # total relocated token rows (all layers)
    page_table: np.ndarray        # int32 flat page ids referenced by reloc_descs
    # outputs
    row_text: np.ndarray          # int32 [c0] index into the concatenated text ids (-1: image row)
    row_img: np.ndarray           # int32 [c0] global image index (-1: text row)
    row_t: np.ndarray             # int32 [c0] token index inside its image
    final_rows: np.ndarray        # int32 [c_L] packed rows in (req, pos) order
    positions: list               # per request: int64 positions with logits (reference `rows`)
    logit_ranges: list            # per request: (start, count) into the logits rows

    def structure_key(self) -> bytes:
        """Everything that shapes the launch chain (not the token ids / page ids it reads)."""
        import hashlib
        h = hashlib.sha1()
        for a in (self.c, self.kvoff, self.row_pos, self.row_kv, self.qdst, self.qpos, self.rowof,
                  self.reloc_descs, self.reloc_blocks, self.final_rows, self.row_src[:, 0]):
            h.update(np.ascontiguousarray(a).tobytes())
            h.update(b"|")
        for a in self.attn_items + self.comb_items:
            h.update(np.ascontiguousarray(a).tobytes())
        h.update(f"{len(self.page_table)}|{self.kv_rows}|{self.attn_slots}".encode())
        return h.digest()


RELOC_TOK = 8


def _depths(spec: RequestSpec, L: int, text_base: int, img_base: int):
    """(positions, depth, src kind, src index, text ref, image ref, t) of every token
    computed at layer 0."""
    nt = len(spec.text_pos)
    pos = [spec.text_pos.astype(np.int64)]
    dep = [np.full(nt, L, dtype=np.int64)]
    kind = [np.full(nt, SRC_TEXT, dtype=np.int64)]
    idx = [spec.text_ids.astype(np.int64)]
    tref = [text_base + np.arange(nt)]
    iref = [np.full(nt, -1)]
    tt = [np.zeros(nt, dtype=np.int64)]
    for m, (start, T) in enumerate(spec.images):
        k0 = int(spec.keep[0, m])
        if k0 == 0:
            continue
        t = np.arange(k0)
        d = (spec.keep[:, m][None, :] > t[:, None]).sum(axis=1)
        pos.append(start + t)
        dep.append(d)
        kind.append(np.full(k0, spec.enc_src[m][0], dtype=np.int64))
        idx.append(spec.enc_src[m][1] + t)
        tref.append(np.full(k0, -1))
        iref.append(np.full(k0, img_base + m))
        tt.append(t)
    return tuple(np.concatenate(a) for a in (pos, dep, kind, idx, tref, iref, tt))


def attention_work(q_ranges, qpos, n_req, heads, target_items: int):
    """Split (request, head, 128-query tile) key ranges into <= target_items CTAs.

    Returns (items int32 [n, 8], comb int32 [m, 8], slots)."""
    tiles = []
    for req, q0, cnt in q_ranges:
        for t0 in range(q0, q0 + cnt, 128):
            nq = min(128, q0 + cnt - t0)
            kend = int(qpos[t0 + nq - 1]) + 1
            kend = min(kend, int(n_req[req]))
            tiles.append((req, t0, nq, kend))
    total = sum((kend + 127) // 128 for _, _, _, kend in tiles) * heads
    chunk = max(2, -(-total // max(1, target_items)))
    items, comb, slot = [], [], 0
    for h in range(heads):
        for req, t0, nq, kend in tiles:
            nt = (kend + 127) // 128
            ns = -(-nt // chunk)
            if ns <= 1:
                items.append([t0, nq, h, 0, 0, kend, -1, req])
                continue
            bounds = [min(kend, (nt * s // ns) * 128) for s in range(ns)] + [kend]
            for s in range(ns):
                items.append([t0, nq, h, 0, bounds[s], bounds[s + 1], slot + s, req])
            comb.append([t0, nq, h, slot, ns, 0, 0, 0])
            slot += ns
    it = np.array(items, dtype=np.int32).reshape(-1, 8)
    cb = np.array(comb, dtype=np.int32).reshape(-1, 8)
    return it, cb, slot


# Attention work decomposition (and the matching vlc_attn_pp kernel, tuning key 15): single 128-query
# tiles per CTA with S double-buffered (default; measured 31.7 -> 26.8 us per C3 layer) or the
# two-tile ping-pong kernel (VLC_ATTN_ONE=0).  The two must agree: two-tile items (up to 256 queries)
# on the single-tile kernel would drop queries 128..255.
ATTN_ONE_TILE = bool(int(os.environ.get("VLC_ATTN_ONE", "1")))


def attn_kernel_variant() -> int:
    """vlc_set_tuning(15, .) value matching ATTN_ONE_TILE (39: single tile, two softmax threads per row,
    each column half with its own max / sum / O accumulator;
    0: ping-pong)."""
    return 39 if ATTN_ONE_TILE else 0


def attention_work(q_ranges, qpos, n_req, heads, max_ctas: int = 148):
    """Work items for vlc_attn_pp in the configured decomposition (ATTN_ONE_TILE)."""
    fn = attention_work_one if ATTN_ONE_TILE else attention_work_pp
    return fn(q_ranges, qpos, n_req, heads, max_ctas)


def attention_work_one(q_ranges, qpos, n_req, heads, max_ctas: int = 148):
    """Work items of the single-query-tile attention kernel (vlc_attn_pp, tuning 15 = 30): one CTA
    per (request, head, <= 128 sorted queries, key range).  Key ranges are split so every CTA gets
    about the same number of 128-key tiles (a query tile's keys end at its last query's position, so
    late tiles get more splits); <= 8 splits per tile, all CTAs co-resident when anything is split.

    Returns (items int32 [n, 9], n_groups)."""
    units = []
    for h in range(heads):
        for req, q0, cnt in q_ranges:
            for t0 in range(q0, q0 + cnt, 128):
                nq = min(128, q0 + cnt - t0)
                kend = min(int(qpos[t0 + nq - 1]) + 1, int(n_req[req]))
                units.append((req, t0, nq, kend, h, max(1, -(-kend // 128))))
    total = sum(u[5] for u in units)
    if len(units) >= max_ctas:
        ns = [1] * len(units)
    else:
        target = max(1, -(-total // max_ctas))
        while True:
            ns = [max(1, min(8, -(-u[5] // target))) for u in units]
            if sum(ns) <= max_ctas:
                break
            target += 1
    items, group = [], 0
    for (req, t0, nq, kend, h, tiles), n in zip(units, ns):
        n = min(n, tiles)
        if n == 1:
            items.append([t0, nq, h, 0, 0, kend, -1, (0 << 8) | 1, req])
            continue
        bounds = [min(kend, (tiles * sidx // n) * 128) for sidx in range(n)] + [kend]
        for sidx in range(n):
            items.append([t0, nq, h, 0, bounds[sidx], bounds[sidx + 1], group, (sidx << 8) | n, req])
        group += 1
    return np.array(items, dtype=np.int32).reshape(-1, 9), group


def attention_work_pp(q_ranges, qpos, n_req, heads, max_ctas: int = 148):
    """Work items of the ping-pong attention kernel (include/vlcache.h vlc_attn_pp): one CTA per
    (request, head, <=256 sorted queries, key range).  When there are few (query-pair, head)
    units the key range is split so the grid fills the SMs; split groups merge in-kernel, which
    requires every CTA co-resident, hence total CTAs <= max_ctas whenever anything is split.

    Returns (items int32 [n, 8], n_groups)."""
    pairs = []
    for req, q0, cnt in q_ranges:
        for t0 in range(q0, q0 + cnt, 256):
            nq = min(256, q0 + cnt - t0)
            kend = min(int(qpos[t0 + nq - 1]) + 1, int(n_req[req]))
            pairs.append((req, t0, nq, kend))
    units = len(pairs) * heads
    ns_max = max(1, min(8, max_ctas // max(1, units)))
    items, group = [], 0
    for h in range(heads):
        for req, t0, nq, kend in pairs:
            tiles = (kend + 63) // 64
            ns = max(1, min(ns_max, tiles // 2))
            if ns == 1:
                items.append([t0, nq, h, 0, 0, kend, -1, (0 << 8) | 1, req])
                continue
            # even key-tile split: a CTA's time follows its key-tile count (each iteration serves
            # both query tiles), not the query-tile x key-tile work (measured: work-balanced splits
            # leave the single-tile tail CTAs 1.7x slower)
            bounds = [min(kend, (tiles * s // ns) * 64) for s in range(ns)] + [kend]
            for s in range(ns):
                items.append([t0, nq, h, 0, bounds[s], bounds[s + 1], group, (s << 8) | ns, req])
            group += 1
    it = np.array(items, dtype=np.int32).reshape(-1, 9)
    return it, group


def build_layout(specs: list[RequestSpec], L: int, heads: int, target_items: int = 296) -> Layout:
    R = len(specs)
    n_req = np.array([s.n for s in specs], dtype=np.int64)
    kvoff = np.concatenate([[0], np.cumsum(n_req)[:-1]]).astype(np.int64)
    cols = [[] for _ in range(8)]
    tb = ib = 0
    for r, spec in enumerate(specs):
        parts = _depths(spec, L, tb, ib)
        for k, a in enumerate(parts):
            cols[k].append(a)
        cols[7].append(np.full(len(parts[0]), r))
        tb += len(spec.text_pos)
        ib += len(spec.images)
    pos, dep, kind, idx, tref, iref, tt, req = (np.concatenate(a) for a in cols)
    order = np.lexsort((pos, req, -dep))            # depth desc, then request, then position
    pos, dep, kind, idx, tref, iref, tt, req = (a[order] for a in (pos, dep, kind, idx, tref, iref, tt, req))
    c0 = len(pos)
    c = np.array([(dep > i).sum() for i in range(L)], dtype=np.int32)
    row_kv = kvoff[req] + pos

    qdst = np.zeros((L, c0), dtype=np.int32)
    qpos = np.zeros((L, c0), dtype=np.int32)
    rowof = np.zeros((L, c0), dtype=np.int32)
    q_ranges, attn_items, comb_items = [], [], []
    slots = 0
    for i in range(L):
        ci = int(c[i])
        srt = np.lexsort((pos[:ci], req[:ci]))       # (req, pos) order of the active prefix
        qdst[i, srt] = np.arange(ci)
        qpos[i, :ci] = pos[srt]
        rowof[i, :ci] = srt
        rq = req[srt]
        ranges = []
        for r in range(R):
            sel = np.flatnonzero(rq == r)
            if len(sel):
                ranges.append((r, int(sel[0]), len(sel)))
        q_ranges.append(ranges)
        it9, groups = attention_work(ranges, qpos[i], n_req, heads)
        it9[:, 3] = kvoff[it9[:, 8]]
        attn_items.append(np.ascontiguousarray(it9[:, :8]))
        comb_items.append(np.zeros((0, 8), dtype=np.int32))
        slots = max(slots, groups)

    # relocation descriptors, grouped by layer
    descs, blocks, layer_blocks, pages, ntok_total = [], [], [0], [], 0
    page_base = {}
    for r, spec in enumerate(specs):
        for m, (start, T) in enumerate(spec.images):
            if spec.kv_hit[m]:
                page_base[(r, m)] = sum(len(p) for p in pages)
                pages.append(np.asarray(spec.page_rows[m], dtype=np.int32).reshape(-1))
    for i in range(L):
        for r, spec in enumerate(specs):
            for m, (start, T) in enumerate(spec.images):
                if not spec.kv_hit[m]:
                    continue
                k = int(spec.keep[i, m])
                ntok = T - k
                if ntok <= 0:
                    continue
                ppl = np.asarray(spec.page_rows[m]).shape[1]
                d = [i, page_base[(r, m)] + i * ppl, k, ntok, int(kvoff[r]) + start + k, start + k, 0, 0]
                for off in range(0, ntok, RELOC_TOK):
                    blocks.append([len(descs), off])
                descs.append(d)
                ntok_total += ntok
        layer_blocks.append(len(blocks))

    last = int(c[L - 1])
    final_rows = rowof[L - 1, :last].copy()
    positions, logit_ranges = [], []
    fr_req = req[final_rows]
    for r in range(R):
        sel = np.flatnonzero(fr_req == r)
        positions.append(pos[final_rows[sel]].astype(np.int64))
        logit_ranges.append((int(sel[0]) if len(sel) else 0, len(sel)))

    src = np.stack([kind, idx], axis=1).astype(np.int32)
    src[kind == SRC_TEXT, 1] = idx[kind == SRC_TEXT]
    return Layout(L=L, heads=heads, c=c, kv_rows=int(n_req.sum()), kvoff=kvoff.astype(np.int32),
                  row_req=req.astype(np.int32), row_pos=pos.astype(np.int32), row_kv=row_kv.astype(np.int32),
                  row_src=src, qdst=qdst, qpos=qpos, rowof=rowof, q_ranges=q_ranges,
                  attn_items=attn_items, comb_items=comb_items, attn_slots=slots,
                  reloc_descs=np.array(descs, dtype=np.int32).reshape(-1, 8),
                  reloc_blocks=np.array(blocks, dtype=np.int32).reshape(-1, 2),
                  reloc_layer_blocks=np.array(layer_blocks, dtype=np.int32), reloc_tokens=ntok_total,
                  page_table=(np.concatenate(pages) if pages else np.zeros(1, np.int32)).astype(np.int32),
                  row_text=tref.astype(np.int32), row_img=iref.astype(np.int32), row_t=tt.astype(np.int32),
                  final_rows=final_rows, positions=positions, logit_ranges=logit_ranges)


def structure_of(specs: list[RequestSpec], L: int, heads: int):
    """Cache key of the launch structure of a batch (independent of ids and page ids)."""
    key = [L, heads]
    for s in specs:
        key.append((s.n, np.asarray(s.text_pos, np.int64).tobytes(), tuple(s.images),
                     np.asarray(s.keep, np.int32).tobytes(), tuple(bool(h) for h in s.kv_hit),
                     tuple(int(k) for k, _ in s.enc_src),
                     tuple(0 if p is None else np.asarray(p).shape[1] for p in s.page_rows)))
    return tuple(key)


def with_data(lay: Layout, specs: list[RequestSpec]) -> Layout:
    """Copy of a cached structural layout carrying this batch's token ids, encoder rows
    and store pages."""
    import copy
    out = copy.copy(lay)
    text = np.concatenate([np.asarray(s.text_ids, np.int64) for s in specs]) if specs else np.zeros(0)
    base = np.array([b for s in specs for _, b in s.enc_src], dtype=np.int64)
    src = lay.row_src.copy()
    t_rows = lay.row_text >= 0
    src[t_rows, 1] = text[lay.row_text[t_rows]]
    i_rows = ~t_rows
    src[i_rows, 1] = base[lay.row_img[i_rows]] + lay.row_t[i_rows]
    out.row_src = src
    pages = [np.asarray(s.page_rows[m], np.int32).reshape(-1) for s in specs
             for m in range(len(s.images)) if s.kv_hit[m]]
    out.page_table = np.concatenate(pages) if pages else np.zeros(1, np.int32)
    return out
