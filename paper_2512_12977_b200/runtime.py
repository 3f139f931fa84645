"""Device executor of the reuse prefill: workspaces and the per-layer launch chain.

All compute goes through libvlcache (include/vlcache.h); torch only allocates
HBM, provides the stream and does host<->device copies.
"""
from __future__ import annotations

import contextlib
import math
import threading
import weakref

import numpy as np

from . import _native as N
from .layout import Layout, attention_work, contiguous_chunks, tiles_needed
from .model import RMS_EPS, DeviceWeights

N_SMS = 148
_DEBUG_SYNC = bool(int(__import__("os").environ.get("VLC_DEBUG_SYNC", "0")))  # sync + log every launch


def _torch():
    import torch
    return torch


def _stream() -> int:
    return _torch().cuda.current_stream().cuda_stream


def pick_splits(n_pad: int, k_pad: int, m_tokens: int) -> int:
    """Split-K factor so a weight-streaming GEMM covers the 148 SMs."""
    m_tiles = n_pad // 128
    n_tile = 256 if m_tokens >= 256 else max(16, (m_tokens + 15) // 16 * 16)
    tiles = m_tiles * ((m_tokens + n_tile - 1) // n_tile)
    k_blocks = k_pad // 64
    if tiles >= N_SMS:
        return 1
    s = min(max(1, k_blocks // 4), max(1, round(N_SMS / tiles)))
    return max(1, s)


class Workspace:
    """Grow-only device buffers keyed by name."""

    def __init__(self):
        self.bufs: dict[str, object] = {}
        self.pinned: dict[str, tuple] = {}     # key -> (pinned host staging tensor, last copy event)
        self.live = weakref.WeakSet()

    def get(self, name: str, shape: tuple, dtype, zero: bool = True):
        torch = _torch()
        t = self.bufs.get(name)
        if t is None or t.dtype != dtype or t.dim() != len(shape) or any(a < b for a, b in zip(t.shape, shape)):
            if t is not None:
                shape = tuple(max(a, b) for a, b in zip(t.shape, shape)) if t.dim() == len(shape) else shape
            t = (torch.zeros if zero else torch.empty)(shape, dtype=dtype, device="cuda")
            self.bufs[name] = t
        return t

    def detach_live(self):
        for r in list(self.live):
            r._detach()
        self.live = weakref.WeakSet()


class IntPack:
    """Concatenate int32 arrays into one host buffer -> one H2D copy; views by name."""

    def __init__(self):
        self.parts, self.off, self.n = [], {}, 0

    def add(self, name, arr):
        a = np.ascontiguousarray(np.asarray(arr, dtype=np.int32).reshape(-1))
        self.off[name] = (self.n, a.size)
        self.parts.append(a)
        self.n += a.size + (-a.size) % 4   # keep 16-byte alignment of every view
        if (-a.size) % 4:
            self.parts.append(np.zeros((-a.size) % 4, np.int32))

    def _full_host(self):
        """The whole int32 buffer: the (shared, read-only) template with the per-call patches."""
        host = getattr(self, "host", None)
        if host is None:
            return np.concatenate(self.parts) if self.parts else np.zeros(4, np.int32)
        patches = getattr(self, "patches", None)
        if not patches:
            return host
        host = host.copy()
        for name, arr in patches.items():
            o, n = self.off[name]
            host[o:o + n] = arr
        return host

    def upload(self, ws: Workspace, key: str):
        """One async H2D copy through a persistent pinned staging buffer of the workspace (no
        per-call pinned allocation); the staging buffer is reused once its last copy completed."""
        torch = _torch()
        host = self._full_host()
        n = max(4, host.size)
        dev = ws.get(key, (n,), torch.int32, zero=False)
        pin, ev = ws.pinned.get(key, (None, None))
        if pin is None or pin.numel() < n:
            pin = torch.empty(max(n, 1 << 16), dtype=torch.int32, pin_memory=True)
            ev = None
        elif ev is not None:
            ev.synchronize()              # the previous copy out of this staging buffer is done
        pin.numpy()[:host.size] = host
        dev[:host.size].copy_(pin[:host.size], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        ws.pinned[key] = (pin, ev)
        ws.last_h2d_bytes = 4 * int(host.size)
        self.dev = dev
        return self

    def upload_segments(self, ws: Workspace, key: str, names):
        """Refresh only the named segments of an already uploaded pack of the same layout
        structure (per-call token ids / page ids); the structural arrays stay resident."""
        torch = _torch()
        pin, ev = ws.pinned[key]
        if ev is not None:
            ev.synchronize()
        dev = ws.bufs[key]
        views = ws.__dict__.setdefault("pinned_np", {})   # cached numpy view / pointers of the staging
        cached = views.get(key)
        if cached is None or cached[0] is not pin:
            cached = views[key] = (pin, pin.numpy(), pin.data_ptr())
        pn, pin_ptr = cached[1], cached[2]
        # the named segments as one contiguous span when they are adjacent (the pack puts the
        # per-call segments first): one H2D copy instead of one per segment
        spans = sorted(self.off[name] for name in names)
        lo, hi = spans[0][0], max(o + n for o, n in spans)
        if sum(n for _, n in spans) >= (hi - lo) * 3 // 4:
            spans = [(lo, hi - lo)]
        nbytes = 0
        patches = getattr(self, "patches", None) or {}
        lib, stream = N.load(), _stream()
        for o, n in spans:
            pn[o:o + n] = self.host[o:o + n]          # template (structural values)
            for name, arr in patches.items():          # per-call segments inside the span
                po, pn_ = self.off[name]
                if o <= po and po + pn_ <= o + n:
                    pn[po:po + pn_] = arr
            N.check(lib.vlc_copy_h2d_async(dev.data_ptr() + 4 * o, pin_ptr + 4 * o, 4 * n, stream),
                    "vlc_copy_h2d_async")
            nbytes += 4 * n
        ws.last_h2d_bytes = nbytes
        if ev is None:
            ev = torch.cuda.Event()
        ev.record()                      # one event per staging buffer, re-recorded each call
        ws.pinned[key] = (pin, ev)
        self.dev = dev
        return self

    def ptr(self, name) -> int:
        o, _ = self.off[name]
        return int(self.dev.data_ptr()) + 4 * o


def _epi(**kw) -> N.Epilogue:
    e = N.Epilogue()
    for k, v in kw.items():
        setattr(e, k, v)
    return e


class Runner:
    """Issues the kernel chain for one model on the current stream."""

    def __init__(self, dw: DeviceWeights):
        self.dw = dw
        self.cfg = dw.cfg
        # Two output/workspace sets used alternately: a result keeps pointing at its set (no copy)
        # and is only detached (copied out) if it is still alive when its set comes round again.
        self.sets = [Workspace(), Workspace()]
        self._cur = 0
        self.ws = self.sets[0]
        self.shared = Workspace()    # per-call scratch (split-K partials, counters, attention merge)
        self.enc_ws = Workspace()
        self.lib = N.load()
        # deterministic: split-K partials of the residual GEMMs reduced in a fixed order (bitwise
        # reproducible runs; per call through vlc_epilogue.deterministic) instead of red.add in
        # arrival order (faster).
        self.deterministic = False
        torch = _torch()
        self.splitk = self.shared.get("splitk", (64 << 20,), torch.float32, zero=False)
        self.counters = self.shared.get("counters", (1 << 16,), torch.int32)
        self.attn_counters = self.shared.get("attn_counters", (1 << 14,), torch.int32)
        self.launches = 0          # kernels issued by this runner (all entry points)
        self.graphs: dict = {}     # structure key -> captured CUDA graph of the prefill chain
        self.layouts: dict = {}    # structure key -> Layout (engine._layout)
        self.graph_launches: dict = {}
        self.tracer = None         # list -> (name, ev0, ev1, algo_bytes, algo_flops) per launch
        self.tp_group = None       # head-parallel process group (engine sets it from the model)
        # Concurrent callers: the workspaces, split-K scratch and counters belong to
        # the runner, so calls are serialised -- on the host by the lock, on the device by making
        # each call's stream wait for the previous call's completion event.
        self.lock = threading.RLock()
        self._done = None

    @contextlib.contextmanager
    def serial(self):
        """One call's exclusive use of this runner's device state (host lock + stream order)."""
        torch = _torch()
        with self.lock:
            cur = torch.cuda.current_stream()
            if self._done is not None:
                cur.wait_event(self._done)
            try:
                yield
            finally:
                if self._done is None:
                    self._done = torch.cuda.Event()
                self._done.record(cur)

    def _run(self, name, fn, nbytes=0, flops=0, kernels=1):
        """Issue one C-ABI call; optionally bracket it with CUDA events on the current stream."""
        if _DEBUG_SYNC:
            import sys
            import time
            sys.stderr.write(f"[vlc] {name} ...")
            sys.stderr.flush()
            t0 = time.perf_counter()
            fn()
            _torch().cuda.synchronize()
            sys.stderr.write(f" {1e3 * (time.perf_counter() - t0):.3f} ms\n")
            sys.stderr.flush()
        elif self.tracer is None:
            fn()
        else:
            torch = _torch()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            self.tracer.append((name, e0, e1, nbytes, flops))
        self.launches += kernels

    # ---------------------------------------------------------------- primitives
    def gemm(self, w, k_pad, x, m, epi: N.Epilogue, splits: int | None = None, name="gemm", k_valid=None):
        """w: PackedWeight; x: packed activations (row tile N.row_tile(m, w.n)), flat bf16 tensor."""
        if m <= 0:
            return
        if splits is None:
            splits = 0                       # stream-K over all SMs
        epi.m_tokens = m
        if epi.kind == N.EPI_RESID and self.deterministic:
            epi.deterministic = 1
        R = N.row_tile(m, w.n)
        kv_ = k_valid or k_pad
        nbytes = 2 * epi.n_valid * kv_ + 2 * m * kv_
        self._run(name, lambda: N.check(self.lib.vlc_gemm_bf16(
            w.data_ptr(), w.n, w.k, x.data_ptr(), -(-m // R) * R, m, epi, splits, self.splitk.data_ptr(),
            self.splitk.numel() * 4, self.counters.data_ptr(), _stream()), "vlc_gemm_bf16"),
            nbytes, 2 * m * epi.n_valid * kv_)

    def rmsnorm(self, x, gamma, out, rows, out_f32=False, row_map=0, pk=(0, 0)):
        """out: fp32 row-major [rows, ld] (out_f32) or flat packed bf16 with geometry pk=(R, KB)."""
        d = self.cfg.model_dim
        if rows <= 0:
            return
        ldo = out.shape[1] if out.dim() == 2 else d
        self._run("rmsnorm", lambda: N.check(self.lib.vlc_rmsnorm(
            x.data_ptr(), x.shape[1], gamma.data_ptr(), out.data_ptr(), ldo, int(out_f32), rows, d,
            row_map, RMS_EPS, pk[0], pk[1], _stream()), "vlc_rmsnorm"), rows * d * (4 + (4 if out_f32 else 2)))

    def attention(self, q, kc, vc, layer, chunks_ptr, items_ptr, n_items, qpos_ptr, rowof_ptr, out, slots,
                  nbytes=0, flops=0, pk=(0, 0), kv=None, heads=None, pool=None, page_table=0):
        """vlc_attn_paged over one layer.  pool: the store's _PagePool whose pages the chunk list
        references (None: every chunk is request rows).  kv / heads: this rank's K/V width and head
        count (default: the decoder's, head-split)."""
        torch = _torch()
        cfg, dw = self.cfg, self.dw
        hd = cfg.head_dim
        kv = kv or dw.kv
        heads = heads or dw.heads
        if pool is None and dw.cos is None:
            dw.ensure_positions(2)     # tables only read for store chunks; the pointer must be valid
        ws_o =self.shared.get("attn_ws_o", (max(1, slots) * 8 * 256 * hd,), torch.float32, zero=False)
        ws_ml = self.shared.get("attn_ws_ml", (max(1, slots) * 8 * 256 * 2,), torch.float32, zero=False)
        a = N.AttnPagedArgs(
            q=q.data_ptr(), q_rows_cap=q.shape[0], kc=kc.data_ptr(), vc=vc.data_ptr(), layers_cap=kc.shape[0],
            kv_rows_cap=kc.shape[1], layer=layer,
            pool_k=pool.kr.data_ptr() if pool is not None else None,
            pool_v=pool.v.data_ptr() if pool is not None else None,
            pool_rows=pool.k.shape[0] if pool is not None else 0, page_table=page_table or None,
            page_rows=pool.P if pool is not None else 0,
            cos_tab=dw.cos.data_ptr(), sin_tab=dw.sin.data_ptr(), tab_ld=hd // 2,
            kv=kv, heads=heads, head_dim=hd, chunks=chunks_ptr, items=items_ptr, n_items=n_items,
            qpos=qpos_ptr, rowof=rowof_ptr, out=out.data_ptr(), ldo=kv, pk_rows=pk[0], pk_kb=pk[1],
            ws_o=ws_o.data_ptr(), ws_ml=ws_ml.data_ptr(), ws_slots=slots, counters=self.attn_counters.data_ptr(),
            scale_log2=math.log2(math.e) / math.sqrt(hd))
        self._run("attention", lambda: N.check(self.lib.vlc_attn_paged(a, _stream()), "vlc_attn_paged"),
                  nbytes, flops)

    # ---------------------------------------------------------------- vision encoder (miss path)
    def encode(self, pixels_list) -> "object":
        """GPU toy ViT (model.py:302-332) for k images -> fp32 [k*T, d] (workspace scratch).
        GEMM inputs (patches, normed rows, attention output, SwiGLU output) are PACKED."""
        torch = _torch()
        cfg, dw, ws = self.cfg, self.dw, self.enc_ws
        T, d, kv, p = cfg.tokens_per_image, cfg.model_dim, cfg.kv_dim, cfg.patch_size
        k = len(pixels_list)
        M = k * T
        cap = -(-max(256, M) // 256) * 256
        E = dw.enc
        Rp = N.row_tile(T, E["patch_w"].n)
        rows_img = -(-T // Rp) * Rp
        patches = ws.get("patches", (k * rows_img * dw.kp,), torch.bfloat16)
        xe = ws.get("xe", (cap, d), torch.float32)
        xn = ws.get("xn", (cap * dw.kd,), torch.bfloat16)
        qe = ws.get("qe", (cap, kv), torch.bfloat16)
        ke = ws.get("ke", (1, cap, kv), torch.bfloat16)
        ve = ws.get("ve", (1, cap, kv), torch.bfloat16)
        att = ws.get("att", (cap * dw.kkv_enc,), torch.bfloat16)
        hb = ws.get("h", (cap * dw.kh,), torch.bfloat16)
        out = ws.get("out", (cap, d), torch.float32)
        side = cfg.image_side
        host = np.stack([np.asarray(px, dtype=np.float32).reshape(side, side) for px in pixels_list])
        dev_px = ws.get("pixels", (k, side, side), torch.float32, zero=False)
        dev_px[:k].copy_(torch.from_numpy(host).pin_memory(), non_blocking=True)
        for m in range(k):
            self._run("patchify", lambda m=m: N.check(self.lib.vlc_patchify(
                dev_px[m].data_ptr(), side, p, patches.data_ptr(), m * rows_img, Rp, dw.kp // 128, _stream()),
                "vlc_patchify"))
        for m in range(k):
            # per-image GEMM so the positional rows line up with token t
            self.gemm(E["patch_w"], dw.kp, patches[m * rows_img * dw.kp:], T,
                      _epi(kind=N.EPI_BIAS_ADD, n_valid=d, out=xe[m * T].data_ptr(), ldo=d,
                           bias=E["patch_b"].data_ptr(), add=E["pos"].data_ptr(), ld_add=d))
        # each GEMM input packed with that GEMM's row tile
        pkq = (N.row_tile(M, E["wqkv_plain"].n), dw.kd // 128)
        pkkv = (N.row_tile(M, E["wo"].n), dw.kkv_enc // 128)
        pkg = (N.row_tile(M, E["wgu"].n), dw.kd // 128)
        pkh = (N.row_tile(M, E["wd"].n), dw.kh // 128)
        self.rmsnorm(xe, E["attn_norm"], xn, M, pk=pkq)
        self.gemm(E["wqkv_plain"], dw.kd, xn, M,
                  _epi(kind=N.EPI_QKV_PLAIN, n_valid=3 * kv, out=qe.data_ptr(), ldo=kv, out2=ke.data_ptr(), ld2=kv,
                       out3=ve.data_ptr(), ld3=kv, seg=kv, hd=cfg.head_dim))
        # bidirectional (model.py:325): every query sees all T keys of its image (position T - 1)
        ranges = [(m, m * T, T) for m in range(k)]
        qpos = np.full(M, T - 1, dtype=np.int32)
        chunks = [contiguous_chunks(m * T, T) for m in range(k)]
        chunk0 = np.arange(k) * len(chunks[0])
        items, slots = attention_work(ranges, qpos, lambda r, p: tiles_needed(chunks[r], p), chunk0,
                                      cfg.num_heads)
        pack = IntPack()
        pack.add("items", items)
        pack.add("chunks", np.concatenate(chunks))
        pack.add("qpos", qpos)
        pack.add("rowof", np.arange(M))
        pack.upload(ws, "enc_ints")
        self.attention(qe, ke, ve, 0, pack.ptr("chunks"), pack.ptr("items"), len(items), pack.ptr("qpos"),
                       pack.ptr("rowof"), att, slots, pk=pkkv, kv=kv, heads=cfg.num_heads)
        self.gemm(E["wo"], dw.kkv_enc, att, M, _epi(kind=N.EPI_RESID, n_valid=d, out=xe.data_ptr(), ldo=d))
        self.rmsnorm(xe, E["mlp_norm"], xn, M, pk=pkg)
        self.gemm(E["wgu"], dw.kd, xn, M,
                  _epi(kind=N.EPI_SWIGLU, n_valid=2 * cfg.mlp_hidden, out=hb.data_ptr(), ldo=dw.kh,
                       pk_rows=pkh[0], pk_kb=pkh[1]))
        self.gemm(E["wd"], dw.kh, hb, M, _epi(kind=N.EPI_RESID, n_valid=d, out=xe.data_ptr(), ldo=d))
        self.rmsnorm(xe, E["out_norm"], out, M, out_f32=True)
        return out[:M]

    # ---------------------------------------------------------------- token-by-token decode
    def decoder(self, keys, values, capacity: int) -> "DeviceDecoder":
        """Decode state over merged pre-RoPE KV (device bf16 [L, n0, kv]), model.py:392-411."""
        return DeviceDecoder(self, keys, values, capacity)

    # ---------------------------------------------------------------- decoder
    def _pick_set(self) -> Workspace:
        """The output set for this call: one no live result points into (preferring the set not
        used last), else detach the results of the older set."""
        for k in (self._cur ^ 1, self._cur):
            if len(self.sets[k].live) == 0:
                self._cur = k
                break
        else:
            self._cur ^= 1
            self.sets[self._cur].detach_live()
        self.ws = self.sets[self._cur]
        return self.ws

    def prefill(self, lay: Layout, text_src: np.ndarray, enc_store_rows, enc_scratch_rows, kv_pool, events=None,
                use_graph: bool = True, inject=None, capture=()):
        """Run embed -> kv_relocate -> L layers -> final norm -> head for a built Layout.

        The launch chain depends only on the layout STRUCTURE (row counts, work lists) and
        on buffer addresses; per-request data (token ids, store pages) travels in one int32
        upload.  The chain is therefore captured once per structure into a CUDA graph and
        replayed: one launch instead of ~230.  Returns the device tensors of the result."""
        torch = _torch()
        cfg, dw = self.cfg, self.dw
        ws = self._pick_set()
        L, d, kv, V = cfg.num_layers, cfg.model_dim, dw.kv, cfg.vocab_size
        c = lay.c
        c0 = int(c[0])
        R = -(-max(256, c0) // 256) * 256          # row capacity (whole 256-row tiles)
        KVR = max(128, lay.kv_rows)
        dw.ensure_positions(max(lay.kv_rows, 1) + 1)
        buf = dict(
            x=ws.get("x", (R, d), torch.float32), xn=ws.get("xn", (R * dw.kd,), torch.bfloat16),
            q=ws.get("q", (R + 256, kv), torch.bfloat16), att=ws.get("att", (R * dw.kkv,), torch.bfloat16),
            h=ws.get("h", (R * dw.kh,), torch.bfloat16), kc=ws.get("kc", (L, KVR, kv), torch.bfloat16),
            vc=ws.get("vc", (L, KVR, kv), torch.bfloat16), kpre=ws.get("kpre", (L, R, kv), torch.bfloat16),
            logits=ws.get("logits", (max(int(c[L - 1]), 1), V), torch.float32, zero=False))
        if self.tp_group is not None:
            buf["y"] = ws.get("y", (R, d), torch.float32)      # this rank's O-projection partial
        hd = cfg.head_dim
        self.shared.get("attn_ws_o", (max(1, lay.attn_slots) * 8 * 256 * hd,), torch.float32, zero=False)
        self.shared.get("attn_ws_ml", (max(1, lay.attn_slots) * 8 * 256 * 2,), torch.float32, zero=False)

        pack = self._pack(lay)
        skey = getattr(lay, "_skey", None)
        if skey is None:
            skey = lay._skey = lay.structure_key()
        if getattr(ws, "ints_key", None) == skey:       # structure resident: only ids / pages change
            pack.upload_segments(ws, "ints", ("src", "pages"))
        else:
            pack.upload(ws, "ints")
            ws.ints_key = skey
        ptrs = (enc_store_rows.data_ptr() if enc_store_rows is not None else 0,
                enc_scratch_rows.data_ptr() if enc_scratch_rows is not None else 0,
                kv_pool.k.data_ptr() if kv_pool is not None else 0,
                kv_pool.v.data_ptr() if kv_pool is not None else 0, kv_pool.P if kv_pool is not None else 0,
                pack.dev.data_ptr(), dw.cos.data_ptr(), dw.cs.data_ptr(), self.splitk.data_ptr(),
                self.shared.bufs["attn_ws_o"].data_ptr(), self.shared.bufs["attn_ws_ml"].data_ptr()) + tuple(
                    t.data_ptr() for t in buf.values())
        buf["kv_pool"] = kv_pool                      # cached chunks are read from its pages
        if inject is not None or capture:
            # measurement path (forward_injected): per-layer KV substitution after the QKV GEMM and
            # captured attention-block outputs; eager launches
            use_graph = False
            buf["capture"] = {i: torch.zeros(max(c0, 1), d, dtype=torch.float32, device="cuda") for i in capture}
            if inject is not None:
                ipk = IntPack()
                ipk.add("descs", inject["descs"])
                ipk.add("blocks", inject["blocks"])
                ipk.add("pages", np.arange(inject["k"].shape[0], dtype=np.int32))
                ipk.upload(self.shared, "inj_ints")
                buf["inject"] = (inject, ipk)
        chain = lambda: self._chain(lay, pack, buf, ptrs)  # noqa: E731
        if events is not None:
            events[0].record()
        if use_graph and self.tracer is None and not _DEBUG_SYNC and self._graph_ok():
            skey = getattr(lay, "_skey", None)
            if skey is None:
                skey = lay._skey = lay.structure_key()
            key = (skey, ptrs, self.deterministic)
            g = self.graphs.get(key)
            if g is None:
                chain()                                   # eager run serves this call
                g = torch.cuda.CUDAGraph()
                cap = torch.cuda.Stream()           # captured off the caller's stream
                cap.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(cap):
                    with torch.cuda.graph(g, stream=cap):
                        launches = self.launches
                        chain()
                        self.graph_launches[key] = self.launches - launches
                        self.launches = launches
                torch.cuda.current_stream().wait_stream(cap)
                if len(self.graphs) >= 16:
                    self.graphs.pop(next(iter(self.graphs)))
                self.graphs[key] = g
            else:
                g.replay()
                self.launches += self.graph_launches[key]
        else:
            chain()
        if events is not None:
            events[1].record()
        return {"logits": buf["logits"], "kc": buf["kc"], "vc": buf["vc"], "kpre": buf["kpre"],
                "R": buf["kpre"].shape[1], "KVR": buf["kc"].shape[1], "pack": pack,
                "capture": buf.get("capture", {})}

    @staticmethod
    def _pack(lay: Layout) -> "IntPack":
        """int32 arrays of the launch chain in one host buffer.  The structural part is built
        once per layout and cached on it; only token ids and page ids change per call."""
        tpl = getattr(lay, "_pack_tpl", None)
        if tpl is None:
            pk = IntPack()
            pk.add("src", lay.row_src)            # per-call segments first and adjacent: one copy
            pk.add("pages", lay.page_table)
            pk.add("row_pos", lay.row_pos)
            pk.add("row_kv", lay.row_kv)
            for i in range(lay.L):
                pk.add(f"qdst{i}", lay.qdst[i])
                pk.add(f"qpos{i}", lay.qpos[i])
                pk.add(f"rowof{i}", lay.rowof[i])
                pk.add(f"items{i}", lay.attn_items[i])
                pk.add(f"chunks{i}", lay.attn_chunks[i])
            pk.add("descs", lay.reloc_descs if len(lay.reloc_descs) else np.zeros(8))
            pk.add("blocks", lay.reloc_blocks if len(lay.reloc_blocks) else np.zeros(2))
            pk.add("final", lay.final_rows)
            tpl = lay._pack_tpl = (np.concatenate(pk.parts), dict(pk.off))
        host, off = tpl
        pk = IntPack()
        # the template stays shared and unmodified; the per-call segments travel as patches (the
        # structure-resident path uploads only them, no copy of the whole ~0.5 MB template)
        pk.host, pk.off = host, off
        pk.patches = {"src": lay.row_src.reshape(-1).astype(np.int32, copy=False),
                      "pages": lay.page_table.reshape(-1).astype(np.int32, copy=False)}
        return pk

    def _allreduce(self, t):
        import torch.distributed as dist
        if self.tracer is None:
            dist.all_reduce(t, group=self.tp_group)
        else:
            torch = _torch()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dist.all_reduce(t, group=self.tp_group)
            e1.record()
            self.tracer.append(("allreduce", e0, e1, t.numel() * 4, 0))

    def _graph_ok(self) -> bool:
        """The chain is graph-captured unless it contains a non-capturable collective (gloo)."""
        if self.tp_group is None:
            return True
        import torch.distributed as dist
        return dist.get_backend(self.tp_group) == "nccl"

    def _chain(self, lay: Layout, pack: "IntPack", buf: dict, ptrs):
        cfg, dw = self.cfg, self.dw
        L, d, kv, V = cfg.num_layers, cfg.model_dim, dw.kv, cfg.vocab_size
        x, xn, q, att, hb = buf["x"], buf["xn"], buf["q"], buf["att"], buf["h"]
        kc, vc, kpre, logits = buf["kc"], buf["vc"], buf["kpre"], buf["logits"]
        c = lay.c
        c0, cL = int(c[0]), int(c[L - 1])
        enc_a, enc_b, kpool, vpool, P = ptrs[:5]
        kv_pool_obj = buf.get("kv_pool")
        s = _stream()
        kd = dw.kd // 128
        # layer-0 rows: text embeddings + cached / freshly encoded image rows
        self._run("embed", lambda: N.check(self.lib.vlc_embed_assemble(
            x.data_ptr(), d, dw.embed.data_ptr(), d, enc_a, enc_b, pack.ptr("src"), c0, s), "vlc_embed_assemble"),
            c0 * d * 6)
        # cached K/V rows that share a 64-key chunk with recomputed ones when the store's page size
        # does not allow reading them in place (attention reads every other cached chunk from the store)
        nb = len(lay.reloc_blocks)
        if nb:
            self._run("kv_relocate", lambda: N.check(self.lib.vlc_kv_relocate(
                kpool, vpool, P, pack.ptr("pages"), kv, cfg.head_dim, kc.data_ptr(), vc.data_ptr(), kc.shape[1],
                pack.ptr("descs"), pack.ptr("blocks"), nb, dw.cos.data_ptr(), dw.sin.data_ptr(),
                cfg.head_dim // 2, _stream()), "vlc_kv_relocate"), lay.reloc_tokens * kv * 2 * 4)

        for i in range(L):
            ci = int(c[i])
            W = dw.layers[i]
            # each GEMM input packed with that GEMM's row tile (one wide tile for 257..512 rows)
            Rq, Ro = N.row_tile(ci, W["wqkv"].n), N.row_tile(ci, W["wo"].n)
            Rg, Rd = N.row_tile(ci, W["wgu"].n), N.row_tile(ci, W["wd"].n)
            self.rmsnorm(x, W["attn_norm"], xn, ci, pk=(Rq, kd))
            self.gemm(W["wqkv"], dw.kd, xn, ci, _epi(
                kind=N.EPI_QKV_ROPE, n_valid=3 * kv, out=q.data_ptr(), ldo=kv,
                out2=kc[i].data_ptr(), ld2=kv, out3=vc[i].data_ptr(), ld3=kv, out4=kpre[i].data_ptr(), ld4=kv,
                map1=pack.ptr(f"qdst{i}"), map2=pack.ptr("row_kv"), pos=pack.ptr("row_pos"),
                cos_tab=dw.cos.data_ptr(), sin_tab=dw.sin.data_ptr(), tab_ld=cfg.head_dim // 2,
                cs_tab=dw.cs.data_ptr() if cfg.head_dim % 4 == 0 else None,
                hd=cfg.head_dim, seg=kv), name="gemm_qkv", k_valid=d)
            if "inject" in buf:
                inj, ipk = buf["inject"]
                lb = inj["layer_blocks"]
                if lb[i + 1] > lb[i]:    # injected pre-RoPE K (rotated to the row positions) / V overwrite
                    self._run("kv_inject", lambda i=i, lb=lb, inj=inj, ipk=ipk: N.check(self.lib.vlc_kv_relocate(
                        inj["k"].data_ptr(), inj["v"].data_ptr(), 1, ipk.ptr("pages"), kv, cfg.head_dim,
                        kc.data_ptr(), vc.data_ptr(), kc.shape[1], ipk.ptr("descs"),
                        ipk.ptr("blocks") + 8 * int(lb[i]), int(lb[i + 1] - lb[i]), dw.cos.data_ptr(),
                        dw.sin.data_ptr(), cfg.head_dim // 2, _stream()), "vlc_kv_relocate"))
            vis = int(lay.qpos[i, :ci].astype(np.int64).sum()) + ci
            self.attention(q, kc, vc, i, pack.ptr(f"chunks{i}"), pack.ptr(f"items{i}"), len(lay.attn_items[i]),
                           pack.ptr(f"qpos{i}"), pack.ptr(f"rowof{i}"), att, lay.attn_slots,
                           nbytes=lay.kv_rows * kv * 4 + ci * kv * 4, flops=4 * cfg.head_dim * dw.heads * vis,
                           pk=(Ro, dw.kkv // 128), pool=kv_pool_obj, page_table=pack.ptr("pages"))
            if i in buf.get("capture", {}):
                # captured attention block output (engine.py:273-275): O projection alone, then
                # x += it fused with the MLP norm
                cap = buf["capture"][i]
                self.gemm(W["wo"], dw.kkv, att, ci, _epi(kind=N.EPI_F32, n_valid=d, out=cap.data_ptr(), ldo=d),
                          name="gemm_o", k_valid=kv)
                self._run("rmsnorm", lambda cap=cap, W=W: N.check(self.lib.vlc_add_rmsnorm(
                    x.data_ptr(), d, cap.data_ptr(), d, W["mlp_norm"].data_ptr(), xn.data_ptr(), d, ci, d, RMS_EPS,
                    Rg, kd, _stream()), "vlc_add_rmsnorm"))
            elif self.tp_group is None:
                self.gemm(W["wo"], dw.kkv, att, ci, _epi(kind=N.EPI_RESID, n_valid=d, out=x.data_ptr(), ldo=d),
                          name="gemm_o", k_valid=kv)
                self.rmsnorm(x, W["mlp_norm"], xn, ci, pk=(Rg, kd))
            else:
                # head-parallel: row-parallel O projection of this rank's heads -> y, one all-reduce
                # of y over the group (NCCL / NVLink), then x += y fused into the MLP norm
                y = buf["y"]
                y[:ci].zero_()
                self.gemm(W["wo"], dw.kkv, att, ci, _epi(kind=N.EPI_RESID, n_valid=d, out=y.data_ptr(), ldo=d),
                          name="gemm_o", k_valid=kv)
                self._allreduce(y[:ci])
                self._run("rmsnorm", lambda: N.check(self.lib.vlc_add_rmsnorm(
                    x.data_ptr(), d, y.data_ptr(), d, W["mlp_norm"].data_ptr(), xn.data_ptr(), d, ci, d, RMS_EPS,
                    Rg, kd, _stream()), "vlc_add_rmsnorm"), ci * d * 14)
            self.gemm(W["wgu"], dw.kd, xn, ci,
                      _epi(kind=N.EPI_SWIGLU, n_valid=2 * cfg.mlp_hidden, out=hb.data_ptr(), ldo=dw.kh,
                           pk_rows=Rd, pk_kb=dw.kh // 128),
                      name="gemm_gate_up", k_valid=d)
            self.gemm(W["wd"], dw.kh, hb, ci, _epi(kind=N.EPI_RESID, n_valid=d, out=x.data_ptr(), ldo=d),
                      name="gemm_down", k_valid=cfg.mlp_hidden)
        self.rmsnorm(x, dw.final_norm, xn, cL, row_map=pack.ptr("final"), pk=(N.row_tile(cL, dw.head.n), kd))
        self.gemm(dw.head, dw.kd, xn, cL, _epi(kind=N.EPI_F32, n_valid=V, out=logits.data_ptr(), ldo=V),
                  name="gemm_head", k_valid=d)


class DeviceDecoder:
    """Growable request KV on the device for greedy decoding (reference DecoderState,
    model.py:392-439): keys held ROTATED at their positions, values as is; each step runs the
    layer chain for one token at the next position through the same kernels as the prefill
    (QKV GEMM with RoPE + KV-append epilogue, attention over all previous keys, O / MLP / head)."""

    def __init__(self, runner: Runner, keys, values, capacity: int):
        torch = _torch()
        if runner.tp_group is not None:
            raise NotImplementedError("decode under head-parallel attention is not supported")
        self.r, cfg, dw = runner, runner.cfg, runner.dw
        L, n0, kv = keys.shape
        self.n, self.cap = int(n0), int(n0 + capacity)
        d = cfg.model_dim
        dw.ensure_positions(self.cap + 1)
        self.kc = torch.zeros(L, self.cap, kv, dtype=torch.bfloat16, device="cuda")
        self.vc = torch.zeros_like(self.kc)
        R = N.row_tile(1)
        self.x = torch.zeros(R, d, dtype=torch.float32, device="cuda")
        self.xn = torch.zeros(N.packed_numel(R, d, R), dtype=torch.bfloat16, device="cuda")
        self.q = torch.zeros(R + 256, kv, dtype=torch.bfloat16, device="cuda")
        self.att = torch.zeros(N.packed_numel(R, dw.kkv, R), dtype=torch.bfloat16, device="cuda")
        self.h = torch.zeros(N.packed_numel(R, dw.kh, R), dtype=torch.bfloat16, device="cuda")
        self.logits = torch.zeros(1, cfg.vocab_size, dtype=torch.float32, device="cuda")
        if n0:
            # rotate every cached key to its position: kv_relocate with the merged KV as a pool of
            # one-token pages (page table = row index), destination rows = positions
            kf = keys.reshape(L * n0, kv).contiguous()
            vf = values.reshape(L * n0, kv).contiguous()
            pt = torch.arange(L * n0, dtype=torch.int32, device="cuda")
            descs = np.array([[i, i * n0, 0, n0, 0, 0, 0, 0] for i in range(L)], dtype=np.int32)
            blocks = np.array([[i, t] for i in range(L) for t in range(0, n0, 8)], dtype=np.int32)
            dd = torch.from_numpy(descs).cuda()
            bb = torch.from_numpy(blocks).cuda()
            N.call("vlc_kv_relocate", kf.data_ptr(), vf.data_ptr(), 1, pt.data_ptr(), kv, cfg.head_dim,
                   self.kc.data_ptr(), self.vc.data_ptr(), self.cap, dd.data_ptr(), bb.data_ptr(), len(blocks),
                   dw.cos.data_ptr(), dw.sin.data_ptr(), cfg.head_dim // 2, _stream())
            _torch().cuda.current_stream().synchronize()

    def step(self, token: int):
        """Append `token` at the next position; device logits row [1, V] (model.py:413-439)."""
        with self.r.serial():
            return self._step(token)

    def _step(self, token: int):
        torch = _torch()
        r, cfg, dw = self.r, self.r.cfg, self.r.dw
        if self.n >= self.cap:
            raise RuntimeError("decode capacity exhausted")
        L, d, kv, V = cfg.num_layers, cfg.model_dim, dw.kv, cfg.vocab_size
        pos = self.n
        R = N.row_tile(1)
        chunks = contiguous_chunks(0, pos + 1)
        items, groups = attention_work([(0, 0, 1)], np.array([pos], np.int32), lambda q, p: tiles_needed(chunks, p),
                                       [0], dw.heads)
        pack = IntPack()
        pack.add("src", np.array([[0, token]]))
        pack.add("pos", np.array([pos]))
        pack.add("zero", np.array([0]))
        pack.add("items", items)
        pack.add("chunks", chunks)
        pack.upload(r.shared, "dec_ints")
        s = _stream()
        r._run("embed", lambda: N.check(r.lib.vlc_embed_assemble(
            self.x.data_ptr(), d, dw.embed.data_ptr(), d, 0, 0, pack.ptr("src"), 1, s), "vlc_embed_assemble"))
        for i in range(L):
            W = dw.layers[i]
            r.rmsnorm(self.x, W["attn_norm"], self.xn, 1, pk=(R, dw.kd // 128))
            r.gemm(W["wqkv"], dw.kd, self.xn, 1, _epi(
                kind=N.EPI_QKV_ROPE, n_valid=3 * kv, out=self.q.data_ptr(), ldo=kv,
                out2=self.kc[i].data_ptr(), ld2=kv, out3=self.vc[i].data_ptr(), ld3=kv,
                map1=pack.ptr("zero"), map2=pack.ptr("pos"), pos=pack.ptr("pos"),
                cos_tab=dw.cos.data_ptr(), sin_tab=dw.sin.data_ptr(), tab_ld=cfg.head_dim // 2,
                cs_tab=dw.cs.data_ptr() if cfg.head_dim % 4 == 0 else None,
                hd=cfg.head_dim, seg=kv), name="gemm_qkv", k_valid=d)
            r.attention(self.q, self.kc, self.vc, i, pack.ptr("chunks"), pack.ptr("items"), len(items),
                        pack.ptr("pos"), pack.ptr("zero"), self.att, groups, pk=(R, dw.kkv // 128))
            r.gemm(W["wo"], dw.kkv, self.att, 1, _epi(kind=N.EPI_RESID, n_valid=d, out=self.x.data_ptr(), ldo=d),
                   name="gemm_o", k_valid=kv)
            r.rmsnorm(self.x, W["mlp_norm"], self.xn, 1, pk=(R, dw.kd // 128))
            r.gemm(W["wgu"], dw.kd, self.xn, 1,
                   _epi(kind=N.EPI_SWIGLU, n_valid=2 * cfg.mlp_hidden, out=self.h.data_ptr(), ldo=dw.kh,
                        pk_rows=R, pk_kb=dw.kh // 128), name="gemm_gate_up", k_valid=d)
            r.gemm(W["wd"], dw.kh, self.h, 1, _epi(kind=N.EPI_RESID, n_valid=d, out=self.x.data_ptr(), ldo=d),
                   name="gemm_down", k_valid=cfg.mlp_hidden)
        r.rmsnorm(self.x, dw.final_norm, self.xn, 1, pk=(R, dw.kd // 128))
        r.gemm(dw.head, dw.kd, self.xn, 1, _epi(kind=N.EPI_F32, n_valid=V, out=self.logits.data_ptr(), ldo=V),
               name="gemm_head", k_valid=d)
        self.n += 1
        return self.logits
