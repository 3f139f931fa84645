"""Content-addressed encoder / KV cache store, resident in B200 HBM.

Same contract as the reference store (store.py:29-241): sha256 keys over raw
pixel bytes, lock-free gets, locked puts, per-fingerprint shape discipline,
StaleCacheError on a fingerprint mismatch, a miss is `None`.  Storage differs:
  * KV entries live in a PAGED bf16 pool per KV width: a page holds
    `page_tokens` token rows of one layer, an entry owns L * ceil(T/P) pages
    listed in its page table (int32 [L, ceil(T/P)]).  kv_relocate gathers
    straight from these pages into the request cache.
  * encoder entries occupy one fp32 slot [T, d] of a slot pool.
  * entry objects returned by gets are device-backed views; their `keys`,
    `values`, `embeddings` attributes materialise fp32 numpy on access.
Persistence uses the reference on-disk format (manifest.json + sha256-named
little-endian fp32 blobs, store.py:159-241).
"""
from __future__ import annotations

import hashlib
import json
import os
import threading
import time
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .exceptions import InputError, IntegrityError, StaleCacheError

DIGEST_ALGO = "sha256"
MANIFEST_NAME = "manifest.json"
STORE_FORMAT = "kvreuse-store-v1"


@dataclass(frozen=True)
class ImageHash:
    """Lowercase 64-hex sha256 digest."""

    hex: str

    def __post_init__(self):
        if len(self.hex) != 64 or self.hex != self.hex.lower():
            raise InputError(f"not a lowercase 64-char hex digest: {self.hex!r}")

    def __str__(self) -> str:
        return self.hex


def _raw_bytes(pixels) -> bytes:
    buf = np.ascontiguousarray(pixels)
    if buf.size == 0:
        raise InputError("cannot hash an empty pixel buffer")
    return buf.tobytes()


def hash_image(pixels) -> ImageHash:
    """sha256 over the image's raw C-order bytes, caller's dtype (store.py:43-51)."""
    return ImageHash(hashlib.sha256(_raw_bytes(pixels)).hexdigest())


def hash_request(images) -> ImageHash:
    """sha256 over the concatenated raw bytes of all images, in order (store.py:54-61)."""
    if not images:
        raise InputError("cannot hash an empty image list")
    h = hashlib.sha256()
    for px in images:
        h.update(_raw_bytes(px))
    return ImageHash(h.hexdigest())


@dataclass
class EncoderCacheEntry:
    hash: ImageHash
    embeddings: object        # [T, d] float32 (numpy, or a cuda tensor)
    model_fingerprint: int


@dataclass
class KVCacheEntry:
    hash: ImageHash
    keys: object              # [L, T, kv] pre-RoPE (numpy fp32, or cuda tensor)
    values: object
    origin_position: int
    model_fingerprint: int


# ---------------------------------------------------------------- device pools

def _torch():
    import torch
    from . import _native
    if not torch.cuda.is_available():
        raise _native.NativeError("CacheStore needs a CUDA device (no CPU fallback)")
    _native.load()
    return torch


class _PagePool:
    """bf16 [capacity * page_tokens, width] rows; page p = rows [p*P, (p+1)*P).  k holds pre-RoPE K
    (the reference's stored form, store.py:140-147); kr the same keys rotated at the position they were
    cached at (filled per entry by engine._ensure_rotated), which the attention reads."""

    def __init__(self, width: int, page_tokens: int, pages: int):
        torch = _torch()
        self.width, self.P = width, page_tokens
        self.k = torch.zeros(pages * page_tokens, width, dtype=torch.bfloat16, device="cuda")
        self.v = torch.zeros_like(self.k)
        self.kr = torch.zeros_like(self.k)
        self.free = list(range(pages - 1, -1, -1))

    @property
    def capacity(self) -> int:
        return self.k.shape[0] // self.P

    def alloc(self, n: int) -> np.ndarray:
        if n > len(self.free):
            self._grow(max(2 * self.capacity, self.capacity + n))
        return np.array([self.free.pop() for _ in range(n)], dtype=np.int32)

    def release(self, pages) -> None:
        self.free.extend(int(p) for p in pages)

    def _grow(self, pages: int) -> None:
        torch = _torch()
        old = self.capacity
        k = torch.zeros(pages * self.P, self.width, dtype=torch.bfloat16, device="cuda")
        v, kr = torch.zeros_like(k), torch.zeros_like(k)
        k[:self.k.shape[0]] = self.k
        v[:self.v.shape[0]] = self.v
        kr[:self.kr.shape[0]] = self.kr
        self.k, self.v, self.kr = k, v, kr
        self.free = list(range(pages - 1, old - 1, -1)) + self.free


class _SlotPool:
    """fp32 [slots, T, d] encoder-output slots."""

    def __init__(self, tokens: int, width: int, slots: int):
        torch = _torch()
        self.rows = torch.zeros(slots, tokens, width, dtype=torch.float32, device="cuda")
        self.free = list(range(slots - 1, -1, -1))

    def alloc(self) -> int:
        if not self.free:
            torch = _torch()
            old = self.rows.shape[0]
            new = torch.zeros(2 * old, *self.rows.shape[1:], dtype=torch.float32, device="cuda")
            new[:old] = self.rows
            self.rows = new
            self.free = list(range(2 * old - 1, old - 1, -1))
        return self.free.pop()

    def release(self, slot: int) -> None:
        self.free.append(int(slot))


class StoredEncoder:
    """Device-backed encoder entry (attributes as EncoderCacheEntry)."""

    def __init__(self, h: ImageHash, pool: _SlotPool, slot: int, fp: int):
        self.hash, self._pool, self.slot, self.model_fingerprint = h, pool, slot, fp
        self._host = None

    def device_embeddings(self):
        return self._pool.rows[self.slot]

    @property
    def embeddings(self) -> np.ndarray:
        if self._host is None:
            self._host = self.device_embeddings().cpu().numpy()
        return self._host


class StoredKV:
    """Device-backed KV entry (attributes as KVCacheEntry)."""

    def __init__(self, h: ImageHash, pool: _PagePool, pages: np.ndarray, layers: int, tokens: int,
                 origin: int, fp: int):
        self.hash, self.pool, self.pages = h, pool, pages  # pages int32 [L, ceil(T/P)]
        self.layers, self.tokens = layers, tokens
        self.origin_position, self.model_fingerprint = origin, fp
        self._host_k = self._host_v = None
        self.rotated_for = None     # (head_dim, rope_base) whose rotation pool.kr holds for these pages

    def _rows(self):
        torch = _torch()
        t = np.arange(self.tokens)
        rows = self.pages[:, t // self.pool.P].astype(np.int64) * self.pool.P + (t % self.pool.P)
        return torch.from_numpy(rows.reshape(-1)).cuda()

    def device_keys(self):
        return self.pool.k[self._rows()].view(self.layers, self.tokens, -1)

    def device_values(self):
        return self.pool.v[self._rows()].view(self.layers, self.tokens, -1)

    @property
    def keys(self) -> np.ndarray:
        if self._host_k is None:
            self._host_k = self.device_keys().float().cpu().numpy()
        return self._host_k

    @property
    def values(self) -> np.ndarray:
        if self._host_v is None:
            self._host_v = self.device_values().float().cpu().numpy()
        return self._host_v


def _finite_f32(name: str, arr):
    """Host numpy -> contiguous fp32 (checked); cuda tensor -> checked, kept on device."""
    if hasattr(arr, "is_cuda") and arr.is_cuda:
        torch = _torch()
        if not bool(torch.isfinite(arr).all()):
            raise InputError(f"{name} contains non-finite values")
        return arr
    a = np.ascontiguousarray(arr, dtype=np.float32)
    if not np.isfinite(a).all():
        raise InputError(f"{name} contains non-finite values")
    return a


def _shape(a) -> tuple:
    return tuple(int(s) for s in a.shape)


class CacheStore:
    """HBM-resident content-addressed store (see module doc)."""

    def __init__(self, page_tokens: int = 64):
        if page_tokens <= 0:
            raise InputError("page_tokens must be positive")
        self.page_tokens = page_tokens
        self._enc: dict[str, StoredEncoder] = {}
        self._kv: dict[str, StoredKV] = {}
        self._shapes: dict[int, dict[str, tuple]] = {}
        self._kv_pools: dict[int, _PagePool] = {}
        self._enc_pools: dict[tuple, _SlotPool] = {}
        self._write_lock = threading.Lock()
        self.version = 0

    def __len__(self) -> int:
        return len(self._enc) + len(self._kv)

    def _check_shape(self, fp: int, kind: str, shape: tuple) -> None:
        known = self._shapes.setdefault(fp, {})
        if kind in known and known[kind] != shape:
            raise InputError(f"{kind} entry shape {shape} disagrees with previously stored "
                             f"{known[kind]} for model {fp:#x}")
        known[kind] = shape

    @staticmethod
    def _check_fingerprint(entry, expected: int | None, key: str) -> None:
        if expected is not None and entry.model_fingerprint != expected:
            raise StaleCacheError(f"{key}: cached by model {entry.model_fingerprint:#x}, "
                                  f"requested for {expected:#x}")

    # -- puts / gets
    def put_encoder(self, entry: EncoderCacheEntry) -> None:
        emb = _finite_f32("embeddings", entry.embeddings)
        shape = _shape(emb)
        if len(shape) != 2:
            raise InputError(f"embeddings must be [T, d], got {shape}")
        torch = _torch()
        with self._write_lock:
            self._check_shape(entry.model_fingerprint, "encoder", shape)
            pool = self._enc_pools.get(shape)
            if pool is None:
                pool = self._enc_pools[shape] = _SlotPool(shape[0], shape[1], 8)
            slot = pool.alloc()
            src = emb if isinstance(emb, torch.Tensor) else torch.from_numpy(emb)
            pool.rows[slot].copy_(src.to(device="cuda", dtype=torch.float32), non_blocking=False)
            old = self._enc.get(entry.hash.hex)
            self._enc[entry.hash.hex] = StoredEncoder(entry.hash, pool, slot, entry.model_fingerprint)
            if old is not None:
                old._pool.release(old.slot)
            self.version += 1

    def get_encoder(self, h: ImageHash, expected_fingerprint: int | None = None):
        entry = self._enc.get(h.hex)
        if entry is None:
            return None
        self._check_fingerprint(entry, expected_fingerprint, f"encoder/{h.hex}")
        return entry

    def put_kv(self, entry: KVCacheEntry) -> None:
        from . import _native
        keys = _finite_f32("keys", entry.keys)
        values = _finite_f32("values", entry.values)
        if _shape(keys) != _shape(values):
            raise InputError("key/value shapes differ")
        shape = _shape(keys)
        if len(shape) != 3:
            raise InputError(f"KV entries must be [L, T, kv], got {shape}")
        L, T, kv = shape
        if kv % 8:
            raise InputError("kv_dim must be a multiple of 8 for the device pool")
        torch = _torch()
        P = min(self.page_tokens, T)
        ppl = (T + P - 1) // P
        with self._write_lock:
            self._check_shape(entry.model_fingerprint, "kv", shape)
            key = (kv, P)
            pool = self._kv_pools.get(key)
            if pool is None:
                pool = self._kv_pools[key] = _PagePool(kv, P, max(64, 4 * L * ppl))
            pages = pool.alloc(L * ppl).reshape(L, ppl)
            ptab = torch.from_numpy(pages.reshape(-1).copy()).cuda()
            stream = torch.cuda.current_stream().cuda_stream
            for src, dst in ((keys, pool.k), (values, pool.v)):
                if isinstance(src, torch.Tensor):
                    s = src.contiguous()
                    is_f32 = int(s.dtype == torch.float32)
                    if s.dtype not in (torch.float32, torch.bfloat16):
                        s, is_f32 = s.float(), 1
                else:
                    s, is_f32 = torch.from_numpy(src).cuda(), 1
                _native.call("vlc_store_write_pages", s.data_ptr(), is_f32, L, T, kv, ptab.data_ptr(), ppl,
                             dst.data_ptr(), P, stream)
            torch.cuda.current_stream().synchronize()
            old = self._kv.get(entry.hash.hex)
            self._kv[entry.hash.hex] = StoredKV(entry.hash, pool, pages, L, T, int(entry.origin_position),
                                                entry.model_fingerprint)
            if old is not None:
                old.pool.release(old.pages.reshape(-1))
            self.version += 1

    def get_kv(self, h: ImageHash, expected_fingerprint: int | None = None):
        entry = self._kv.get(h.hex)
        if entry is None:
            return None
        self._check_fingerprint(entry, expected_fingerprint, f"kv/{h.hex}")
        return entry

    def kv_pool_for(self, entry: StoredKV) -> _PagePool:
        return entry.pool

    # -- persistence (reference format, store.py:159-241)
    def persist(self, directory: str | Path) -> None:
        directory = Path(directory)
        (directory / "blobs").mkdir(parents=True, exist_ok=True)
        with self._write_lock, _dir_lock(directory):
            entries = {}
            for hx, enc in sorted(self._enc.items()):
                arr = np.ascontiguousarray(enc.embeddings, dtype="<f4")
                entries[f"encoder/{hx}"] = _write_blob(directory, arr, {
                    "kind": "encoder", "image_hash": hx, "shape": list(arr.shape),
                    "model_fingerprint": enc.model_fingerprint})
            for hx, kv in sorted(self._kv.items()):
                stacked = np.stack([kv.keys, kv.values])
                entries[f"kv/{hx}"] = _write_blob(directory, stacked, {
                    "kind": "kv", "image_hash": hx, "shape": list(stacked.shape),
                    "origin_position": kv.origin_position, "model_fingerprint": kv.model_fingerprint})
            (directory / MANIFEST_NAME).write_text(json.dumps(
                {"format": STORE_FORMAT, "digest_algo": DIGEST_ALGO, "entries": entries}, indent=1, sort_keys=True))

    @classmethod
    def load(cls, directory: str | Path, page_tokens: int = 64) -> "CacheStore":
        directory = Path(directory)
        mpath = directory / MANIFEST_NAME
        if not mpath.exists():
            raise IntegrityError(f"no manifest at {mpath}")
        try:
            manifest = json.loads(mpath.read_text())
        except json.JSONDecodeError as exc:
            raise IntegrityError(f"corrupt manifest {mpath}: {exc}") from None
        if manifest.get("format") != STORE_FORMAT:
            raise IntegrityError(f"unknown store format {manifest.get('format')!r}")
        store = cls(page_tokens)
        for key, meta in sorted(manifest.get("entries", {}).items()):
            arr = _read_blob(directory, key, meta)
            h, fp = ImageHash(meta["image_hash"]), int(meta["model_fingerprint"])
            if meta["kind"] == "encoder":
                store.put_encoder(EncoderCacheEntry(h, arr, fp))
            elif meta["kind"] == "kv":
                store.put_kv(KVCacheEntry(h, arr[0], arr[1], int(meta["origin_position"]), fp))
            else:
                raise IntegrityError(f"{key}: unknown entry kind {meta['kind']!r}")
        return store


def _write_blob(directory: Path, arr: np.ndarray, meta: dict) -> dict:
    raw = np.ascontiguousarray(arr, dtype="<f4").tobytes()
    digest = hashlib.sha256(raw).hexdigest()
    rel = f"blobs/{digest}.bin"
    if not (directory / rel).exists():
        (directory / rel).write_bytes(raw)
    return dict(meta, blob=rel, sha256=digest, bytes=len(raw))


def _read_blob(directory: Path, key: str, meta: dict) -> np.ndarray:
    path = directory / meta["blob"]
    if not path.exists():
        raise IntegrityError(f"{key}: missing blob {meta['blob']}")
    raw = path.read_bytes()
    if len(raw) != meta["bytes"]:
        raise IntegrityError(f"{key}: blob is {len(raw)} bytes, manifest says {meta['bytes']}")
    if hashlib.sha256(raw).hexdigest() != meta["sha256"]:
        raise IntegrityError(f"{key}: blob checksum mismatch")
    return np.frombuffer(raw, dtype="<f4").reshape(meta["shape"]).copy()


class _dir_lock:
    """O_EXCL lockfile for one store directory (store.py:244-269)."""

    def __init__(self, directory: Path, timeout: float = 10.0):
        self.path, self.timeout = directory / ".lock", timeout

    def __enter__(self):
        deadline = time.monotonic() + self.timeout
        while True:
            try:
                os.close(os.open(self.path, os.O_CREAT | os.O_EXCL | os.O_WRONLY))
                return self
            except FileExistsError:
                if time.monotonic() > deadline:
                    raise IntegrityError(f"store directory {self.path.parent} is locked") from None
                time.sleep(0.05)

    def __exit__(self, *exc):
        try:
            os.unlink(self.path)
        except FileNotFoundError:
            pass
        return False
