"""ctypes binding of libvlcache.so (include/vlcache.h).

The library is the only compute path: if it is missing, or no CUDA device is
present, every device entry point raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

from .exceptions import InputError, KVReuseError

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libvlcache.so")

VLC_OK, VLC_ERR_INVALID, VLC_ERR_UNSUPPORTED, VLC_ERR_CUDA = 0, 1, 2, 3
EPI_F32, EPI_RESID, EPI_BF16, EPI_BIAS_ADD, EPI_SWIGLU, EPI_QKV_PLAIN, EPI_QKV_ROPE = range(7)

EXPORTS = ("vlc_last_error", "vlc_version", "vlc_embed_assemble", "vlc_rmsnorm",
           "vlc_add_rmsnorm", "vlc_kv_relocate", "vlc_store_write_pages", "vlc_gemm_bf16", "vlc_gemm_row_tile",
           "vlc_pack_operand", "vlc_attn_paged", "vlc_gather_rows",
           "vlc_patchify", "vlc_set_tuning", "vlc_set_debug_buffer", "vlc_copy_h2d_async")


class NativeError(KVReuseError):
    """A CUDA-side failure reported by libvlcache (status VLC_ERR_CUDA / UNSUPPORTED)."""


class Epilogue(C.Structure):
    _fields_ = [("kind", C.c_int), ("n_valid", C.c_int), ("m_tokens", C.c_int),
                ("out", C.c_void_p), ("ldo", C.c_int), ("out2", C.c_void_p), ("ld2", C.c_int),
                ("out3", C.c_void_p), ("ld3", C.c_int), ("out4", C.c_void_p), ("ld4", C.c_int),
                ("map1", C.c_void_p), ("map2", C.c_void_p), ("pos", C.c_void_p),
                ("cos_tab", C.c_void_p), ("sin_tab", C.c_void_p), ("tab_ld", C.c_int),
                ("hd", C.c_int), ("seg", C.c_int), ("bias", C.c_void_p), ("add", C.c_void_p),
                ("ld_add", C.c_int), ("pk_rows", C.c_int), ("pk_kb", C.c_int),
                ("deterministic", C.c_int), ("cs_tab", C.c_void_p)]


class AttnPagedArgs(C.Structure):
    """include/vlcache.h vlc_attn_paged_args."""
    _fields_ = [("q", C.c_void_p), ("q_rows_cap", C.c_int), ("kc", C.c_void_p), ("vc", C.c_void_p),
                ("layers_cap", C.c_int), ("kv_rows_cap", C.c_int), ("layer", C.c_int),
                ("pool_k", C.c_void_p), ("pool_v", C.c_void_p), ("pool_rows", C.c_int),
                ("page_table", C.c_void_p), ("page_rows", C.c_int),
                ("cos_tab", C.c_void_p), ("sin_tab", C.c_void_p), ("tab_ld", C.c_int),
                ("kv", C.c_int), ("heads", C.c_int), ("head_dim", C.c_int),
                ("chunks", C.c_void_p), ("items", C.c_void_p), ("n_items", C.c_int),
                ("qpos", C.c_void_p), ("rowof", C.c_void_p), ("out", C.c_void_p), ("ldo", C.c_int),
                ("pk_rows", C.c_int), ("pk_kb", C.c_int),
                ("ws_o", C.c_void_p), ("ws_ml", C.c_void_p), ("ws_slots", C.c_int),
                ("counters", C.c_void_p), ("scale_log2", C.c_float), ("trace", C.c_void_p)]


_lib = None


def load():
    """Load (not build) the library; raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        vp, i, f = C.c_void_p, C.c_int, C.c_float
        lib.vlc_last_error.restype = C.c_char_p
        lib.vlc_version.restype = i
        lib.vlc_embed_assemble.argtypes = [vp, i, vp, i, vp, vp, vp, i, vp]
        lib.vlc_rmsnorm.argtypes = [vp, i, vp, vp, i, i, i, i, vp, f, i, i, vp]
        lib.vlc_add_rmsnorm.argtypes = [vp, i, vp, i, vp, vp, i, i, i, f, i, i, vp]
        lib.vlc_kv_relocate.argtypes = [vp, vp, i, vp, i, i, vp, vp, i, vp, vp, i, vp, vp, i, vp]
        lib.vlc_store_write_pages.argtypes = [vp, i, i, i, i, vp, i, vp, i, vp]
        lib.vlc_gemm_bf16.argtypes = [vp, i, i, vp, i, i, C.POINTER(Epilogue), i, vp, C.c_size_t, vp, vp]
        lib.vlc_gemm_row_tile.argtypes = [i, i]
        lib.vlc_pack_operand.argtypes = [vp, i, i, i, vp, i, i, vp]
        lib.vlc_attn_paged.argtypes = [C.POINTER(AttnPagedArgs), vp]
        lib.vlc_patchify.argtypes = [vp, i, i, vp, i, i, i, vp]
        lib.vlc_gather_rows.argtypes = [vp, vp, vp, vp, i, i, vp]
        lib.vlc_set_tuning.argtypes = [i, i]
        lib.vlc_copy_h2d_async.argtypes = [vp, vp, C.c_size_t, vp]
        lib.vlc_set_debug_buffer.argtypes = [vp]
        for name in EXPORTS:
            getattr(lib, name).restype = C.c_char_p if name == "vlc_last_error" else i
        _lib = lib
    return _lib


def check(status: int, what: str) -> None:
    if status == VLC_OK:
        return
    msg = load().vlc_last_error().decode(errors="replace")
    if status == VLC_ERR_INVALID:
        raise InputError(f"{what}: {msg}")
    raise NativeError(f"{what}: {msg} (status {status})")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def ptr(t) -> int:
    """Device pointer of a torch tensor (None -> NULL)."""
    return 0 if t is None else int(t.data_ptr())


_ROW_TILES: dict = {}


def row_tile(m_tokens: int, n_pad: int | None = None) -> int:
    """Row tile R of the packed activations consumed by a GEMM of n_pad weight rows over m_tokens rows
    (vlc_gemm_row_tile: <= 256, except 257..512 tokens stay one wide tile in a one-wave GEMM).  Without
    n_pad: the <= 256 rule (kernels other than the GEMM's activation input)."""
    if n_pad is None or m_tokens <= 256 or m_tokens > 512:
        return 256 if m_tokens >= 256 else max(16, (m_tokens + 15) // 16 * 16)
    key = (int(n_pad), int(m_tokens))
    r = _ROW_TILES.get(key)
    if r is None:
        r = _ROW_TILES[key] = int(load().vlc_gemm_row_tile(int(n_pad), int(m_tokens)))
    return r


def packed_numel(rows: int, K: int, R: int) -> int:
    return -(-rows // R) * R * -(-K // 128) * 128


def pack(t, R: int, K: int | None = None, rows_cap: int | None = None):
    """Row-major bf16 cuda tensor [rows, cols] -> flat packed buffer (include/vlcache.h)."""
    import torch
    rows, cols = t.shape
    K = K or cols
    KB = -(-K // 128)
    rcap = max(rows, rows_cap or 0)
    out = torch.zeros(packed_numel(rcap, K, R), dtype=torch.bfloat16, device=t.device)
    src = t.contiguous()
    call("vlc_pack_operand", src.data_ptr(), rows, cols, src.shape[1], out.data_ptr(), R, KB,
         torch.cuda.current_stream().cuda_stream)
    return out


def unpack(p, rows: int, cols: int, R: int, K: int | None = None):
    """Inverse of pack() (torch indexing; test / result helper)."""
    import torch
    K = K or cols
    KB = -(-K // 128)
    row = torch.arange(rows, device=p.device).view(-1, 1)
    k = torch.arange(cols, device=p.device).view(1, -1)
    rt, r = row // R, row % R
    off = ((((rt * KB + (k >> 7)) * 2 + ((k >> 6) & 1)) * R + r) * 64 + ((((k >> 3) & 7) ^ (r & 7)) << 3) + (k & 7))
    return p.view(-1)[off]
