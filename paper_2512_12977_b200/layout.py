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
    page_tokens: int = 64         # token rows per store page
    origin: list = field(default_factory=list)     # per image: position its cached KV was computed at


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
    # attention work (per layer): key chunks + work items of vlc_attn_paged
    attn_chunks: list             # per layer: int32 [n_chunks, 4] {pos0, len, a, b} (all requests)
    attn_items: list              # per layer: int32 [n, 8]
    attn_slots: int               # max split groups over layers
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
        for a in self.attn_items + self.attn_chunks:
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


CHUNK = 64        # keys per attention chunk (vlc_attn_paged); a 128-key tile is two chunks


def contiguous_chunks(row0: int, n: int) -> np.ndarray:
    """Chunks of a request whose n keys (positions 0..n-1) all sit in request rows row0.. ."""
    out = [[c, min(CHUNK, n - c), row0 + c, -1] for c in range(0, n, CHUNK)]
    return _pad_even(out)


def _pad_even(out):
    if len(out) % 2:          # a masked (len 0) chunk that reads valid memory: the previous source
        last = out[-1]
        out.append([last[0] + CHUNK, last[1] & ~0xFF, last[2], last[3]])
    return np.array(out, dtype=np.int32).reshape(-1, 4)


def chunk_shift(ch) -> int:
    """D of a store chunk (its image's new start - cached start), packed above the 8-bit length."""
    return int(ch[1]) >> 8


def store_chunks_ok(T: int, P: int) -> bool:
    """A 64-key chunk of an image lies inside one store page (else the layer's cached rows are
    relocated into the request rows instead of being read from the store)."""
    return P % CHUNK == 0 or T <= P


def request_chunks(spec: RequestSpec, i: int, kvoff: int, page_base: dict) -> np.ndarray:
    """Key chunks of one request at layer i, in position order (vlc_attn_paged, include/vlcache.h):
    text runs and recomputed image chunks from the request rows; image chunks at or past the
    layer's keep count straight from the store page (a = page-table index, b = row offset).  The
    64-token block holding the keep boundary k is split in two chunks: [t0, k) from the request rows
    (recomputed) and [k, t0 + 64) from the store page at row offset k mod P (inside one page since
    P is a multiple of 64), so no cached row goes through vlc_kv_relocate.  Store pages whose size is
    not a multiple of 64 (and T > P) fall back to relocating every cached row (relocated_ranges)."""
    spans = sorted(spec.images)
    out, cur = [], 0

    def text_run(a, b):
        for c in range(a, b, CHUNK):
            out.append([c, min(CHUNK, b - c), kvoff + c, -1])
    for m, (start, T) in sorted(enumerate(spec.images), key=lambda e: e[1][0]):
        text_run(cur, start)
        k = int(spec.keep[i, m])
        hit = bool(spec.kv_hit[m])
        P = int(spec.page_tokens)
        direct = hit and store_chunks_ok(T, P)
        ppl = np.asarray(spec.page_rows[m]).shape[1] if hit else 0
        # D = new start - cached start (the attention rotates its queries by -D for these chunks)
        dsh = (start - int(spec.origin[m] if spec.origin else start)) << 8 if direct else 0
        first_store = True
        for t0 in range(0, T, CHUNK):
            ln = min(CHUNK, T - t0)
            if direct and t0 >= k:
                store = [start + t0, ln | dsh, page_base[m] + i * ppl + t0 // P, t0 % P]
            elif direct and t0 < k < t0 + ln:          # the keep boundary splits this block
                out.append([start + t0, k - t0, kvoff + start + t0, -1])
                store = [start + k, (t0 + ln - k) | dsh, page_base[m] + i * ppl + k // P, k % P]
            else:
                out.append([start + t0, ln, kvoff + start + t0, -1])
                continue
            if first_store and len(out) % 2 and out[-1][3] >= 0 and (out[-1][1] >> 8) != (dsh >> 8):
                # a 128-key tile never pairs store chunks of two images (one query rotation per tile)
                last = out[-1]
                out.append([store[0], last[1] & ~0xFF, last[2], last[3]])
            first_store = False
            out.append(store)
        cur = start + T
    text_run(cur, spec.n)
    del spans
    return _pad_even(out)


def relocated_ranges(spec: RequestSpec, i: int):
    """Per image: the cached token range [k, T) of layer i that goes through vlc_kv_relocate into
    the request rows -- only when the page size does not allow direct store chunks (the chain's
    attention otherwise reads every cached row from its store page)."""
    out = []
    for m, (start, T) in enumerate(spec.images):
        if not spec.kv_hit[m]:
            continue
        k = int(spec.keep[i, m])
        if k >= T:
            continue
        if not store_chunks_ok(T, int(spec.page_tokens)):
            out.append((m, k, T))
    return out


def full_relocation(specs: list, L: int):
    """vlc_kv_relocate descriptors that move EVERY cached (layer, token) row of the batch into the
    request rows -- the unfused gather + re-rotation + scatter, used to measure that kernel against
    its own HBM roofline (bench.py); the prefill chain itself reads cached chunks from the store.
    Returns (descs int32 [d, 8], blocks int32 [b, 2], page_table, rows)."""
    n_req = [s.n for s in specs]
    kvoff = np.concatenate([[0], np.cumsum(n_req)[:-1]]).astype(np.int64)
    pages, base = [], {}
    for r, spec in enumerate(specs):
        for m in range(len(spec.images)):
            if spec.kv_hit[m]:
                base[(r, m)] = sum(len(p) for p in pages)
                pages.append(np.asarray(spec.page_rows[m], dtype=np.int32).reshape(-1))
    descs, blocks, rows = [], [], 0
    for i in range(L):
        for r, spec in enumerate(specs):
            for m, (start, T) in enumerate(spec.images):
                k = int(spec.keep[i, m])
                if not spec.kv_hit[m] or k >= T:
                    continue
                ppl = np.asarray(spec.page_rows[m]).shape[1]
                for off in range(0, T - k, RELOC_TOK):
                    blocks.append([len(descs), off])
                descs.append([i, base[(r, m)] + i * ppl, k, T - k, int(kvoff[r]) + start + k, start + k, 0, 0])
                rows += T - k
    return (np.array(descs, np.int32).reshape(-1, 8), np.array(blocks, np.int32).reshape(-1, 2),
            (np.concatenate(pages) if pages else np.zeros(1, np.int32)).astype(np.int32), rows)


def query_tiles(pos, tiles_of, rows: int = 128, unit_cost: int = 1):
    """Cut one request's position-sorted queries into tiles of <= `rows` rows minimising the key
    tiles the attention walks: a query tile scans every key up to its LAST query's position, so a
    fixed 128-row cut that straddles a gap between recomputed position clusters (the leading tokens
    of the next image) makes the whole tile scan that far.  Exact DP over the cut points
    (O(n * rows) host work, cached with the layout); `unit_cost` key tiles per extra query tile
    breaks ties towards fewer tiles.  C3 at 5%: 128 | 108 rows (18 + 35 key tiles per head) ->
    118 | 118 rows cut at the image-1 / image-2 gap (10 + 35).  Returns [(a, b)] row ranges."""
    n = len(pos)
    if n == 0:
        return []
    cost = np.array([int(tiles_of(int(pos[b - 1]))) for b in range(1, n + 1)], dtype=np.int64)
    best, arg = np.zeros(n + 1, dtype=np.int64), np.zeros(n + 1, dtype=np.int64)
    for b in range(1, n + 1):
        lo = max(0, b - rows)
        a = lo + int(np.argmin(best[lo:b]))       # first minimum: the longest tile among ties
        best[b], arg[b] = best[a] + cost[b - 1] + unit_cost, a
    out, b = [], n
    while b > 0:
        out.append((arg[b], b))
        b = arg[b]
    return out[::-1]


def attention_work(q_ranges, qpos, tiles_of, chunk0, heads, max_ctas: int = 148):
    """Work items of vlc_attn_paged: one CTA per (request, head, <= 128 position-sorted queries,
    range of 128-key tiles).  tiles_of(req, max query position) = 128-key tiles the query tile
    needs (causal); chunk0[req] = the request's chunk-list offset.  Tile ranges are split so that
    every CTA gets about the same number of tiles (late query tiles see more keys, so they get more
    splits); <= 8 splits per query tile, and at most max_ctas CTAs (co-resident: split groups merge
    in-kernel) whenever anything is split.

    Returns (items int32 [n, 8], number of split groups)."""
    units = []
    cuts = {req: query_tiles(qpos[q0:q0 + cnt], lambda p, r=req: tiles_of(r, p)) for req, q0, cnt in q_ranges}
    for h in range(heads):
        for req, q0, cnt in q_ranges:
            for a, b in cuts[req]:
                units.append((req, q0 + a, b - a, h, max(1, int(tiles_of(req, int(qpos[q0 + b - 1]))))))
    total = sum(u[4] for u in units)
    if len(units) >= max_ctas:
        ns = [1] * len(units)
    else:
        target = max(1, -(-total // max_ctas))
        while True:
            ns = [max(1, min(8, -(-u[4] // target))) for u in units]
            if sum(ns) <= max_ctas:
                break
            target += 1
    items, group = [], 0
    for (req, t0, nq, h, tiles), n in zip(units, ns):
        n = min(n, tiles)
        c0 = int(chunk0[req])
        if n == 1:
            items.append([t0, nq, h, c0, 0, tiles, -1, 1])
            continue
        bounds = [tiles * sidx // n for sidx in range(n)] + [tiles]
        for sidx in range(n):
            items.append([t0, nq, h, c0, bounds[sidx], bounds[sidx + 1], group, (sidx << 8) | n])
        group += 1
    return np.array(items, dtype=np.int32).reshape(-1, 8), group


def tiles_needed(chunks: np.ndarray, max_pos: int) -> int:
    """128-key tiles of a position-ordered chunk list that hold keys <= max_pos."""
    need = int(np.searchsorted(chunks[:, 0], max_pos, side="right"))
    return -(-need // 2)


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
    # store pages referenced by this batch: one flat page table (per-call data), per image a base
    pages, page_base = [], {}
    for r, spec in enumerate(specs):
        for m, (start, T) in enumerate(spec.images):
            if spec.kv_hit[m]:
                page_base[(r, m)] = sum(len(p) for p in pages)
                pages.append(np.asarray(spec.page_rows[m], dtype=np.int32).reshape(-1))
    q_ranges, attn_items, attn_chunks = [], [], []
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
        lists = [request_chunks(spec, i, int(kvoff[r]), {m: page_base[(r, m)] for m in range(len(spec.images))
                                                         if (r, m) in page_base})
                 for r, spec in enumerate(specs)]
        chunk0 = np.concatenate([[0], np.cumsum([len(x) for x in lists])[:-1]]).astype(np.int64)
        items, groups = attention_work(ranges, qpos[i], lambda r, p: tiles_needed(lists[r], p), chunk0, heads)
        attn_items.append(np.ascontiguousarray(items))
        attn_chunks.append(np.ascontiguousarray(np.concatenate(lists).astype(np.int32)))
        slots = max(slots, groups)

    # relocation descriptors (vlc_kv_relocate), grouped by layer: only the cached rows that share a
    # key chunk with recomputed ones (attention reads every other cached chunk from the store)
    descs, blocks, layer_blocks, ntok_total = [], [], [0], 0
    for i in range(L):
        for r, spec in enumerate(specs):
            for m, k, e in relocated_ranges(spec, i):
                start = spec.images[m][0]
                ntok = e - k
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
                  attn_chunks=attn_chunks, attn_items=attn_items, attn_slots=slots,
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
                     tuple(0 if p is None else np.asarray(p).shape[1] for p in s.page_rows), int(s.page_tokens),
                     tuple(int(o) for o in s.origin)))
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
