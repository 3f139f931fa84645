"""Reuse prefill on B200 behind the reference API (reference: engine.py:39-190).

`prefill_with_reuse(model, request, store)` keeps the reference's validation
order, error types, hit/miss/fallback semantics and result fields.  Compute runs
on the device: embed assembly, kv_relocate (cached K gathered from the paged
store, re-rotated to its new positions, V copied), then per layer RMSNorm ->
fused QKV GEMM (RoPE + KV scatter epilogue) -> mixed attention -> O GEMM +
residual -> RMSNorm -> gate/up GEMM (SwiGLU epilogue) -> down GEMM + residual,
then final norm + LM head for the last layer's rows.

Results are device-resident and materialise on access: `logits` and `kv.keys`
/`kv.values` are numpy like the reference; `device_logits`, `last_logits()` and
`kv.device_keys()` avoid the host copy.
"""
from __future__ import annotations

import threading
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .config import ModelConfig
from .exceptions import InputError
from .layout import SRC_SCRATCH, SRC_STORE, RequestSpec, build_layout, structure_of, with_data
from .model import KVTensors, ToyVLM
from .plans import ComputationMask, RecomputePlan, build_masks, layer_keep, mean_ratio, require_valid
from .sequence import TokenSequence, make_sequence
from .store import CacheStore, EncoderCacheEntry, ImageHash, KVCacheEntry, hash_image


# ---------------------------------------------------------------- analytic work (engine.py:39-85)

@dataclass(frozen=True)
class FlopsBreakdown:
    encoder: int
    attention: int
    mlp: int

    @property
    def total(self) -> int:
        return self.encoder + self.attention + self.mlp


def _attn_flops(computed: int, keys: int, cfg: ModelConfig) -> int:
    d, kv = cfg.model_dim, cfg.kv_dim
    return 2 * (3 * computed * d * kv + 2 * computed * keys * kv + computed * kv * d)


def _mlp_flops(computed: int, cfg: ModelConfig) -> int:
    return 6 * computed * cfg.model_dim * cfg.mlp_hidden


def encoder_flops(cfg: ModelConfig) -> int:
    t = cfg.tokens_per_image
    return 2 * t * cfg.patch_size ** 2 * cfg.model_dim + _attn_flops(t, t, cfg) + _mlp_flops(t, cfg)


def flops_from_masks(masks: ComputationMask, seq_len: int, cfg: ModelConfig,
                     images_encoded: int = 0) -> FlopsBreakdown:
    counts = masks.computed_counts
    return FlopsBreakdown(images_encoded * encoder_flops(cfg),
                          sum(_attn_flops(c, seq_len, cfg) for c in counts),
                          sum(_mlp_flops(c, cfg) for c in counts))


_FLOPS_CACHE: dict = {}


def _flops_from_counts(counts, n, cfg, encoded):
    """FlopsBreakdown of per-layer computed-row counts (memoised: pure in its arguments)."""
    key = (tuple(counts), n, encoded, cfg.num_layers, cfg.model_dim, cfg.kv_dim, cfg.mlp_hidden,
           cfg.tokens_per_image, cfg.patch_size)
    fb = _FLOPS_CACHE.get(key)
    if fb is None:
        fb = FlopsBreakdown(encoded * encoder_flops(cfg), sum(_attn_flops(c, n, cfg) for c in counts),
                            sum(_mlp_flops(c, cfg) for c in counts))
        if len(_FLOPS_CACHE) < 4096:
            _FLOPS_CACHE[key] = fb
    return fb   # frozen dataclass: safe to share


def count_flops(request, plan: RecomputePlan, config: ModelConfig, encoder_cached: bool = True) -> FlopsBreakdown:
    seq = getattr(request, "seq", request)
    require_valid(plan)
    masks = build_masks(plan, seq)
    return flops_from_masks(masks, len(seq), config, 0 if encoder_cached else len(seq.image_segments))


# ---------------------------------------------------------------- request / result types

@dataclass
class ReuseRequest:
    seq: TokenSequence
    image_hashes: list[ImageHash]
    plan: RecomputePlan
    images: list | None = None  # pixels, for the cache-miss fallback


class ReuseMetrics:
    """Reference fields (engine.py:100-108); compute_seconds is device time (CUDA events),
    resolved lazily so the prefill call itself never blocks the host."""

    def __init__(self, mean_ratio: float = 0.0):
        self.fallback_images = 0
        self.encoder_misses = 0
        self.computed_per_layer: list[int] = []
        self.flops: FlopsBreakdown | None = None
        self.resolve_seconds = 0.0
        self.mean_ratio = mean_ratio
        self._events = None
        self._compute = None

    @property
    def compute_seconds(self) -> float:
        if self._compute is None:
            if self._events is None:
                return 0.0
            self._events[1].synchronize()
            self._compute = self._events[0].elapsed_time(self._events[1]) / 1e3
        return self._compute

    @compute_seconds.setter
    def compute_seconds(self, v: float) -> None:
        self._compute = v


_PINNED: dict = {}   # numel -> pinned host staging row for last_logits()


def _locked(fn, lock):
    def call():
        with lock:
            return fn()
    return call


class ReuseResult:
    """positions (host), logits [len(positions), V] and merged pre-RoPE KV, device-backed."""

    def __init__(self, positions, dev_logits, kv: KVTensors, metrics: ReuseMetrics, lock=None):
        self.positions = positions
        self._dev_logits = dev_logits
        self._logits = None
        self.kv = kv
        self.metrics = metrics
        # the runner's lock: a host read must not interleave with a later call that detaches this
        # result (copies it out of the shared workspace) and reuses the workspace
        self._lock = lock if lock is not None else threading.RLock()
        if kv._loader is not None:
            kv._loader = _locked(kv._loader, self._lock)   # no reference back to self (no cycle)

    @property
    def device_logits(self):
        return self._dev_logits

    @property
    def logits(self) -> np.ndarray:
        if self._logits is None:
            with self._lock:
                self._logits = self._dev_logits.cpu().numpy()
        return self._logits

    def last_logits(self) -> np.ndarray:
        """Last row's logits (the next-token distribution) via a pinned staging buffer."""
        import torch
        with self._lock:
            row = self._dev_logits[-1]
            buf = _PINNED.get(row.numel())
            if buf is None:
                buf = _PINNED[row.numel()] = torch.empty(row.numel(), dtype=row.dtype, pin_memory=True)
            buf.copy_(row, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            return buf.numpy().copy()

    def _detach(self):
        """The runner is about to reuse its workspace: take private copies."""
        self._dev_logits = self._dev_logits.clone()
        if self.kv._dev is None and self.kv._keys is None:
            self.kv._device()
        if self.kv._dev is not None:
            self.kv._dev = tuple(t.clone() for t in self.kv._dev)
        self.kv._loader = None


# ---------------------------------------------------------------- runner cache

def _layout(runner, specs, L, heads):
    """Structural layouts are cached per runner; per-request data is patched in."""
    key = structure_of(specs, L, heads)
    lay = runner.layouts.get(key)
    if lay is None:
        lay = build_layout(specs, L, heads)
        if len(runner.layouts) >= 64:
            runner.layouts.pop(next(iter(runner.layouts)))
        runner.layouts[key] = lay
        return lay
    return with_data(lay, specs)


_RUNNER_LOCK = threading.Lock()


def _runner(model: ToyVLM):
    from .runtime import Runner
    r = getattr(model, "_runner", None)
    if r is None:
        with _RUNNER_LOCK:
            r = getattr(model, "_runner", None)
            if r is None:
                r = Runner(model.device)
                r.tp_group = model.tp_group
                model._runner = r
    return r


def encode_image(model: ToyVLM, pixels) -> np.ndarray:
    """GPU toy ViT (model.py:302-332); returns host fp32 [T, d] like the reference."""
    _check_pixels(model.config, pixels)
    runner = _runner(model)
    with runner.serial():
        return runner.encode([pixels]).cpu().numpy()


def encode_images_device(model: ToyVLM, pixels_list):
    for px in pixels_list:
        _check_pixels(model.config, px)
    runner = _runner(model)
    with runner.serial():
        return runner.encode(pixels_list).clone()     # the encoder workspace is reused by the next call


def _check_pixels(cfg: ModelConfig, pixels) -> None:
    px = np.asarray(pixels)
    if px.ndim != 2:
        raise InputError(f"expected a 2-d pixel grid, got shape {px.shape}")
    h, w = px.shape
    p = cfg.patch_size
    if h % p or w % p:
        raise InputError(f"image dims {px.shape} not divisible by patch size {p}")
    if (h // p) * (w // p) != cfg.tokens_per_image:
        raise InputError(f"image yields {(h // p) * (w // p)} patches, model expects {cfg.tokens_per_image}")
    if h != w:
        raise InputError("the device patchify expects square images")


# ---------------------------------------------------------------- the hot path

def _text_tokens(seq: TokenSequence, cfg: ModelConfig):
    pos, ids = [], []
    for seg in seq.segments:
        if seg.kind == "text":
            for p in range(seg.start, seg.start + seg.length):
                t = seq.ids[p]
                if t >= cfg.vocab_size:
                    raise InputError(f"token id {t} out of vocab")
                pos.append(p)            # a negative id embeds as a zero row (model.py:349-353)
                ids.append(t)
    return np.array(pos, dtype=np.int64), np.array(ids, dtype=np.int64)


class _Resolved:
    """Host result of the resolve phase of one request (engine.py:121-163)."""

    def __init__(self, spec, metrics, enc_pool, kv_pool, miss_px):
        self.spec, self.metrics, self.enc_pool, self.kv_pool, self.miss_px = spec, metrics, enc_pool, kv_pool, miss_px


def _resolve(model: ToyVLM, request: ReuseRequest, store: CacheStore, miss_base: int = 0) -> _Resolved:
    """Validation (reference order: PlanError, layer count, sequence/hash count), then per
    image: encoder-cache lookup, KV-cache lookup, miss / fallback bookkeeping."""
    cfg = model.config
    seq, plan = request.seq, request.plan
    require_valid(plan)
    if plan.num_layers != cfg.num_layers:
        raise InputError(f"plan has {plan.num_layers} layers, model has {cfg.num_layers}")
    seq.validate(cfg.tokens_per_image)
    segs = seq.image_segments
    if len(request.image_hashes) != len(segs):
        raise InputError("one hash per image segment required")
    metrics = ReuseMetrics(mean_ratio=mean_ratio(plan))
    T, L = cfg.tokens_per_image, cfg.num_layers
    keep = np.repeat(layer_keep(plan, T)[:, None], len(segs), axis=1).astype(np.int32)

    fp = model.fingerprint
    runner_kv = model.device.kv
    enc_src, kv_hit, page_rows, miss_px, origin = [], [], [], [], []
    enc_pool = kv_pool = None
    for m, seg in enumerate(segs):                               # engine.py:140-159
        h = request.image_hashes[m]
        enc = store.get_encoder(h, expected_fingerprint=fp)
        if enc is not None:
            if enc_pool is not None and enc._pool is not enc_pool:
                raise InputError("encoder entries of one model must share a pool")
            enc_pool = enc._pool
            enc_src.append((SRC_STORE, enc.slot * T))
        else:
            metrics.encoder_misses += 1
            if request.images is None or request.images[m] is None:
                raise InputError(f"encoder cache miss for image {m} and no pixels supplied")
            _check_pixels(cfg, request.images[m])
            enc_src.append((SRC_SCRATCH, (miss_base + len(miss_px)) * T))
            miss_px.append(request.images[m])
        entry = store.get_kv(h, expected_fingerprint=fp)
        if entry is not None:
            if entry.tokens != T or entry.layers != L:
                raise InputError("cached KV shape does not match the model")
            if entry.pool.width != runner_kv:
                raise InputError(f"cached KV width {entry.pool.width} does not match this model's K/V width "
                                 f"{runner_kv} (head-parallel stores hold each rank's head slice)")
            kv_pool = entry.pool
            # keep is non-increasing over layers: any layer that skips image tokens reads cached KV
            kv_hit.append(bool((keep[:, m] < T).any()))
            page_rows.append(entry.pages)
            origin.append(int(entry.origin_position))
            if kv_hit[-1]:
                _ensure_rotated(model, entry)
        else:
            kv_hit.append(False)
            page_rows.append(None)
            origin.append(0)
            if (keep[:, m] < T).any():                            # reuse requested, nothing to reuse
                metrics.fallback_images += 1
                keep[:, m] = T
    text_pos, text_ids = _text_tokens(seq, cfg)
    counts = (len(text_pos) + keep.sum(axis=1)).tolist()   # one numpy reduction, not one per layer
    metrics.computed_per_layer = counts
    metrics.flops = _flops_from_counts(counts, len(seq), cfg, metrics.encoder_misses)
    spec = RequestSpec(n=len(seq), text_pos=text_pos, text_ids=text_ids,
                       images=[(s.start, s.length) for s in segs], keep=keep, kv_hit=kv_hit,
                       enc_src=enc_src, page_rows=page_rows, page_tokens=kv_pool.P if kv_pool is not None else 64,
                       origin=origin)
    return _Resolved(spec, metrics, enc_pool, kv_pool, miss_px)


def _ensure_rotated(model: ToyVLM, entry) -> None:
    """The store entry's K rotated at the positions it was cached at (origin + t), into its pool's kr
    pages (same page ids): once per entry and RoPE configuration, on the caller's stream.  The attention
    reads these pages for reused rows and rotates its queries by -(new start - origin) instead of
    re-rotating every cached key (engine.py:180 algebra: R(s + t) k = R(s - o) R(o + t) k)."""
    cfg = model.config
    sig = (cfg.head_dim, float(cfg.rope_base))
    if getattr(entry, "rotated_for", None) == sig:
        return
    import torch
    from .layout import RELOC_TOK
    pool, P = entry.pool, entry.pool.P
    L, T = entry.layers, entry.tokens
    dw = model.device
    dw.ensure_positions(int(entry.origin_position) + T + 1)
    pages = np.asarray(entry.pages, dtype=np.int32)
    ppl = pages.shape[1]
    j = np.arange(ppl)
    ntok = np.minimum(P, T - j * P)
    descs = np.zeros((L, ppl, 8), dtype=np.int32)
    descs[:, :, 1] = np.arange(L * ppl).reshape(L, ppl)
    descs[:, :, 3] = ntok[None, :]
    descs[:, :, 4] = pages * P
    descs[:, :, 5] = int(entry.origin_position) + j[None, :] * P
    descs = descs.reshape(-1, 8)
    nt = descs[:, 3]
    nblk = -(-nt // RELOC_TOK)
    blocks = np.stack([np.repeat(np.arange(len(descs)), nblk),
                       np.concatenate([np.arange(k) * RELOC_TOK for k in nblk])], axis=1).astype(np.int32)
    pad = np.zeros((-pages.size) % 4, dtype=np.int32)          # blocks are read as int2: 8-byte aligned
    ints = torch.from_numpy(np.concatenate([pages.reshape(-1), pad, descs.reshape(-1), blocks.reshape(-1)])).cuda()
    o_d = pages.size + pad.size
    o_b = o_d + descs.size
    N.check(N.load().vlc_kv_relocate(pool.k.data_ptr(), None, P, ints.data_ptr(), pool.width, cfg.head_dim,
                                     pool.kr.data_ptr(), None, pool.kr.shape[0], ints[o_d:].data_ptr(),
                                     ints[o_b:].data_ptr(), len(blocks), dw.cos.data_ptr(), dw.sin.data_ptr(),
                                     cfg.head_dim // 2, torch.cuda.current_stream().cuda_stream), "vlc_kv_relocate")
    entry.rotated_for = sig


def prefill_with_reuse(model: ToyVLM, request: ReuseRequest, store: CacheStore) -> ReuseResult:
    return prefill_batch_with_reuse(model, [request], store)[0]


def prefill_batch_with_reuse(model: ToyVLM, requests: list, store: CacheStore) -> list:
    """Several independent reuse prefills in ONE device pass (BASELINE configs[4]): the
    computed rows of all requests are concatenated (varlen), so every layer's GEMMs stream
    the weights once for the whole batch; attention stays per request (own KV rows,
    causal by position).  Result i equals prefill_with_reuse(model, requests[i], store)."""
    if not requests:
        return []
    runner = _runner(model)
    with runner.serial():
        return _prefill_batch(model, requests, store, runner)


def _prefill_batch(model: ToyVLM, requests: list, store: CacheStore, runner) -> list:
    cfg = model.config
    L = cfg.num_layers
    t0 = time.perf_counter()
    resolved, miss_px = [], []
    for req in requests:
        r = _resolve(model, req, store, miss_base=len(miss_px))
        resolved.append(r)
        miss_px.extend(r.miss_px)
    enc_pools = {id(r.enc_pool): r.enc_pool for r in resolved if r.enc_pool is not None}
    kv_pools = {id(r.kv_pool): r.kv_pool for r in resolved if r.kv_pool is not None}
    if len(enc_pools) > 1 or len(kv_pools) > 1:
        raise InputError("requests of one batch must resolve to one encoder pool and one KV pool")
    enc_pool = next(iter(enc_pools.values()), None)
    kv_pool = next(iter(kv_pools.values()), None)
    scratch = runner.encode(miss_px) if miss_px else None
    dt = time.perf_counter() - t0
    for r in resolved:
        r.metrics.resolve_seconds = dt

    specs = [r.spec for r in resolved]
    lay = _layout(runner, specs, L, runner.dw.heads)
    import torch
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    text_ids = np.concatenate([s.text_ids for s in specs])
    out = runner.prefill(lay, text_ids, enc_pool.rows.view(-1, cfg.model_dim) if enc_pool else None,
                         scratch, kv_pool, events=ev)
    results = []
    for i, r in enumerate(resolved):
        r.metrics._events = ev
        start, cnt = lay.logit_ranges[i]
        kv = KVTensors(loader=_merged_kv_loader(out, lay, r.spec, kv_pool, cfg, req=i))
        res = ReuseResult(lay.positions[i], out["logits"][start:start + cnt], kv, r.metrics, runner.lock)
        runner.ws.live.add(res)
        results.append(res)
    return results


def _merged_kv_loader(out, lay, spec: RequestSpec, kv_pool, cfg: ModelConfig, req: int = 0):
    """Merged pre-RoPE KV [L, n, kv] of one request: computed rows from the QKV epilogue's
    pre-RoPE copy, reused rows from the store pages (engine.py:153-155, 177-178).
    Index construction is deferred to the first access."""
    kpre, vc, R = out["kpre"], out["vc"], out["R"]

    def load():
        import torch
        L, n, kvd = cfg.num_layers, spec.n, out["kc"].shape[2]   # this rank's heads under head-parallel
        kvoff = int(lay.kvoff[req])
        sel = np.flatnonzero(lay.row_req == req)
        pos = lay.row_pos[sel].astype(np.int64)
        kpre_idx, kpre_dst, pool_idx, pool_dst = [], [], [], []
        for i in range(L):
            live = sel < lay.c[i]
            kpre_idx.append(i * R + sel[live])
            kpre_dst.append(i * n + pos[live])
            for m, (start, T) in enumerate(spec.images):
                if not spec.kv_hit[m]:
                    continue
                t = np.arange(int(spec.keep[i, m]), T)
                if len(t):
                    pages = spec.page_rows[m]
                    pool_idx.append(pages[i, t // kv_pool.P].astype(np.int64) * kv_pool.P + t % kv_pool.P)
                    pool_dst.append(i * n + start + t)
        # one int32 upload of the row maps, then vlc_gather_rows: K rows from the QKV epilogue's pre-RoPE
        # copy (computed) and the store pages (reused); V rows from the request cache and the store
        KVR = vc.shape[1]
        v_src = (np.arange(L, dtype=np.int64)[:, None] * KVR + kvoff + np.arange(n)[None, :]).reshape(-1)
        v_dst = np.arange(L * n, dtype=np.int64)
        pk = [np.concatenate(kpre_idx), np.concatenate(kpre_dst), v_src, v_dst]
        if pool_idx:
            pk += [np.concatenate(pool_idx), np.concatenate(pool_dst)]
        sizes = [len(a) for a in pk]
        idx = torch.from_numpy(np.concatenate(pk).astype(np.int32)).cuda()
        offs = np.concatenate([[0], np.cumsum(sizes)])
        K = torch.zeros(L * n, kvd, dtype=torch.bfloat16, device="cuda")
        V = torch.zeros(L * n, kvd, dtype=torch.bfloat16, device="cuda")
        stream = torch.cuda.current_stream().cuda_stream

        def gather(dst, src, j):        # pairs (src rows pk[j], dst rows pk[j + 1])
            N.check(N.load().vlc_gather_rows(dst.data_ptr(), idx[offs[j + 1]:].data_ptr(), src.data_ptr(),
                                             idx[offs[j]:].data_ptr(), sizes[j], kvd * 2, stream), "vlc_gather_rows")
        gather(K, kpre, 0)
        gather(V, vc, 2)
        if pool_idx:
            # reused rows straight from the store pages (the attention reads them there too)
            gather(K, kv_pool.k, 4)
            gather(V, kv_pool.v, 4)
        K, V = K.view(L, n, kvd), V.view(L, n, kvd)
        return K.view(L, n, kvd), V
    return load


def prefill_full(model: ToyVLM, seq: TokenSequence, image_embeds) -> tuple[np.ndarray, KVTensors]:
    """Dense causal prefill (model.py:362-389) on device: plan = 1.0 through the same kernels."""
    import torch
    res = _prefill_embeds(model, seq, image_embeds)
    if not bool(torch.isfinite(res.device_logits).all()):      # model.py:387-388
        raise InputError("non-finite logits from prefill")
    # the result object is dropped here: give the returned KV its own device copy so that it stays
    # valid when the runner's output buffers are reused
    k, v = (t.clone() for t in res.kv._device())
    return res.logits, KVTensors(loader=lambda: (k, v))


def _prefill_embeds(model: ToyVLM, seq: TokenSequence, image_embeds, inject=None, capture=()) -> ReuseResult:
    """Full prefill with explicit image embeddings (host numpy or device rows)."""
    runner = _runner(model)
    with runner.serial():
        return _prefill_embeds_locked(model, seq, image_embeds, runner, inject, capture)


def _prefill_embeds_locked(model, seq, image_embeds, runner, inject, capture) -> ReuseResult:
    import torch
    cfg = model.config
    seq.validate(cfg.tokens_per_image)
    segs = seq.image_segments
    if len(segs) != len(image_embeds):
        raise InputError(f"sequence has {len(segs)} image segments but {len(image_embeds)} embedding blocks "
                         "were supplied")
    T, L, d = cfg.tokens_per_image, cfg.num_layers, cfg.model_dim
    if segs:
        blocks = []
        for e in image_embeds:
            t = e if isinstance(e, torch.Tensor) else torch.from_numpy(np.asarray(e, dtype=np.float32))
            if tuple(t.shape) != (T, d):
                raise InputError(f"embedding block shape {tuple(t.shape)} does not match model")
            blocks.append(t.to(device="cuda", dtype=torch.float32))
        scratch = torch.cat(blocks).contiguous()
    else:
        scratch = None
    text_pos, text_ids = _text_tokens(seq, cfg)
    keep = np.full((L, len(segs)), T, dtype=np.int32)
    spec = RequestSpec(n=len(seq), text_pos=text_pos, text_ids=text_ids,
                       images=[(s.start, s.length) for s in segs], keep=keep, kv_hit=[False] * len(segs),
                       enc_src=[(SRC_SCRATCH, m * T) for m in range(len(segs))], page_rows=[None] * len(segs))
    lay = _layout(runner, [spec], L, runner.dw.heads)
    metrics = ReuseMetrics(mean_ratio=1.0)
    metrics.computed_per_layer = [len(seq)] * L
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    out = runner.prefill(lay, text_ids, None, scratch, None, events=ev, inject=inject, capture=capture)
    metrics._events = ev
    start, cnt = lay.logit_ranges[0]
    res = ReuseResult(lay.positions[0], out["logits"][start:start + cnt],
                      KVTensors(loader=_merged_kv_loader(out, lay, spec, None, cfg)), metrics, runner.lock)
    res._scratch = scratch
    res._capture = out["capture"]
    runner.ws.live.add(res)
    return res


# ---------------------------------------------------------------- dense forward with injected KV (engine.py:239-292)

def forward_injected(model: ToyVLM, seq: TokenSequence, image_embeds, inject_keys=None, inject_values=None,
                     use_cached=None, capture_layers=()):
    """Teacher-forced dense forward with per-layer KV substitution (reference engine.py:239-283): at
    (layer i, position p) with use_cached[i, p], attention sees inject_keys/values[i, p] (pre-RoPE,
    rotated to p on the device) instead of the fresh projections; hidden states are still computed
    everywhere.  Returns (logits [n, V] numpy, {layer: attention block output [n, d]})."""
    import torch
    cfg = model.config
    L, n, kvd = cfg.num_layers, len(seq), cfg.kv_dim
    if use_cached is None:
        use_cached = np.zeros((L, n), dtype=bool)
    use_cached = np.asarray(use_cached, dtype=bool)
    if use_cached.shape != (L, n):
        raise InputError(f"use_cached must be [{L}, {n}]")
    if use_cached.any() and (inject_keys is None or inject_values is None):
        raise InputError("use_cached set but no injected KV supplied")
    # the reference captures layer i when i or i - L is listed (engine.py:277); nothing else
    caps = sorted({int(c) + L if int(c) < 0 else int(c) for c in capture_layers if -L <= int(c) < L})
    runner = _runner(model)
    if runner.tp_group is not None:
        raise NotImplementedError("forward_injected under head-parallel attention is not supported")
    inject = None
    if use_cached.any():
        def dev(a):
            t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a, np.float32))
            return t.to(device="cuda", dtype=torch.bfloat16).reshape(L * n, kvd).contiguous()
        descs, blocks, layer_blocks = [], [], [0]
        for i in range(L):
            row = use_cached[i]
            edges = np.flatnonzero(np.diff(np.concatenate([[0], row.astype(np.int8), [0]])))
            for s0, s1 in zip(edges[0::2], edges[1::2]):        # runs of injected positions
                for off in range(0, int(s1 - s0), 8):
                    blocks.append([len(descs), off])
                descs.append([i, i * n + int(s0), 0, int(s1 - s0), int(s0), int(s0), 0, 0])
            layer_blocks.append(len(blocks))
        inject = dict(k=dev(inject_keys), v=dev(inject_values), descs=np.array(descs, np.int32),
                      blocks=np.array(blocks, np.int32), layer_blocks=np.array(layer_blocks))
    res = _prefill_embeds(model, seq, image_embeds, inject=inject, capture=caps)
    captured = {i: res._capture[i][:n].cpu().numpy() for i in caps}
    return res.logits, captured


def plan_to_use_cached(plan: RecomputePlan, seq: TokenSequence) -> np.ndarray:
    """The injected-path mask equivalent to a plan: stale wherever the skip path reuses cached KV
    (engine.py:286-292)."""
    use_cached = ~build_masks(plan, seq).layers
    use_cached[:, ~seq.image_mask()] = False
    return use_cached


# ---------------------------------------------------------------- decode over merged KV (engine.py:195-232)

@dataclass
class DecodeResult:
    ids: list
    step_logits: np.ndarray   # distribution each generated id was taken from
    tail_logits: np.ndarray   # logits after each teacher-forced tail token


def decode_with_merged_kv(model: ToyVLM, merged_kv: KVTensors, tail_ids=(), max_new: int = 0,
                          initial_logits=None) -> DecodeResult:
    """Greedy decode attending over merged KV (reference engine.py:204-232): tail tokens are
    teacher-forced first, then generation continues from the last tail logits or from
    `initial_logits` (e.g. the reuse prefill's last row).  Every step runs on the device
    (runtime.DeviceDecoder); ids are chosen on the host (argmax of the returned row)."""
    import torch
    if max_new < 0:
        raise InputError("max_new must be >= 0")
    cfg = model.config
    V = cfg.vocab_size
    tail_logits = np.empty((len(tail_ids), V), dtype=np.float32)
    if not len(tail_ids) and max_new == 0:
        return DecodeResult([], np.empty((0, V), np.float32), tail_logits)
    if max_new > 0 and not len(tail_ids) and initial_logits is None:
        raise InputError("decoding needs a starting distribution: supply tail tokens or "
                         "initial_logits from the prefill")
    runner = _runner(model)
    if merged_kv._loader is not None or merged_kv._dev is not None:
        keys, values = merged_kv.device_keys(), merged_kv.device_values()
    else:
        keys = torch.from_numpy(np.ascontiguousarray(merged_kv.keys, np.float32)).cuda().to(torch.bfloat16)
        values = torch.from_numpy(np.ascontiguousarray(merged_kv.values, np.float32)).cuda().to(torch.bfloat16)
    state = runner.decoder(keys, values, capacity=len(tail_ids) + max_new)

    def step(tok):
        if not 0 <= tok < V:
            raise InputError(f"token id {tok} out of vocab")
        return state.step(tok)[0].cpu().numpy()

    cur = None if initial_logits is None else np.asarray(initial_logits, dtype=np.float32)
    for j, tok in enumerate(tail_ids):
        cur = step(int(tok))
        tail_logits[j] = cur
    ids, step_logits = [], np.empty((max_new, V), dtype=np.float32)
    for t in range(max_new):
        step_logits[t] = cur
        tok = int(np.argmax(cur))
        ids.append(tok)
        cur = step(tok)
    return DecodeResult(ids, step_logits, tail_logits)


def generate(model: ToyVLM, seq: TokenSequence, image_embeds, max_new: int):
    """Full prefill then greedy decoding (model.py:467-471): (ids, step_logits [max_new, V])."""
    logits, kv = prefill_full(model, seq, image_embeds)
    out = decode_with_merged_kv(model, kv, max_new=max_new, initial_logits=logits[-1])
    return out.ids, out.step_logits


def apply_rope(x, positions, head_dim: int, base: float):
    """Rotate [..., kv] vectors to `positions` (model.py:137-163), on the device in fp32 with the
    reference's fp32 angle / cos / sin tables.  A utility of the API surface; the hot path rotates
    inside the QKV epilogue and kv_relocate.  Returns numpy for numpy input, else a cuda tensor."""
    import torch
    from .model import rope_inv_freq
    host = not isinstance(x, torch.Tensor)
    t = torch.as_tensor(np.asarray(x, dtype=np.float32) if host else x).to("cuda", torch.float32)
    squeeze = t.dim() == 1
    if squeeze:
        t = t[None, :]
    pos = np.atleast_1d(np.asarray(positions))
    if pos.shape[0] == 1 and t.shape[-2] != 1:
        pos = np.broadcast_to(pos, (t.shape[-2],))
    ang = pos.astype(np.float32)[:, None] * rope_inv_freq(head_dim, base)[None, :]
    cos = torch.from_numpy(np.cos(ang, dtype=np.float32)).cuda()[:, None, :]
    sin = torch.from_numpy(np.sin(ang, dtype=np.float32)).cuda()[:, None, :]
    half = head_dim // 2
    sh = t.reshape(*t.shape[:-1], t.shape[-1] // head_dim, head_dim)
    a, b = sh[..., :half], sh[..., half:]
    out = torch.cat((a * cos - b * sin, b * cos + a * sin), dim=-1).reshape(t.shape)
    if squeeze:
        out = out[0]
    return out.cpu().numpy() if host else out


# ---------------------------------------------------------------- cache-miss fill (bench.py:82-104)

def fill_store_request(model: ToyVLM, store: CacheStore, seq: TokenSequence, images) -> list:
    """One full device prefill of the request, then one encoder entry and one per-layer
    pre-RoPE KV slice per image written into the store (device to device)."""
    embeds = encode_images_device(model, images) if images else None
    T = model.config.tokens_per_image
    blocks = [embeds[m * T:(m + 1) * T] for m in range(len(images))]
    res = _prefill_embeds(model, seq, blocks)
    K, V = res.kv.device_keys(), res.kv.device_values()
    fp = model.fingerprint
    for seg, px, emb in zip(seq.image_segments, images, blocks):
        h = hash_image(px)
        sl = slice(seg.start, seg.start + seg.length)
        store.put_encoder(EncoderCacheEntry(h, emb, fp))
        store.put_kv(KVCacheEntry(h, K[:, sl], V[:, sl], origin_position=seg.start, model_fingerprint=fp))
    return blocks


def fill_store(model: ToyVLM, store: CacheStore, images, prefix) -> None:
    cfg = model.config
    for px in images:
        fill_store_request(model, store, make_sequence(prefix, 1, cfg.tokens_per_image), [px])
