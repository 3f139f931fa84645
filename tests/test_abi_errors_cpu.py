"""C-ABI argument validation (include/vlcache.h): every entry point rejects bad arguments with a status
code and a thread-local message before touching the device -- so these run without a GPU -- and the
Python binding maps INVALID to InputError (the reference's exception for caller errors) and UNSUPPORTED
to NativeError."""
import ctypes as C

import pytest

from paper_2512_12977_b200 import _native as N
from paper_2512_12977_b200.exceptions import InputError

P = 1 << 12            # a non-null, 16-byte aligned dummy address: validation never dereferences it


@pytest.fixture(scope="module")
def lib():
    return N.load()


def _err(lib):
    return lib.vlc_last_error().decode()


def _epi(**kw):
    e = N.Epilogue()
    for k, v in kw.items():
        setattr(e, k, v)
    return e


def _attn(**kw):
    a = N.AttnPagedArgs(q=P, kc=P, vc=P, items=P, chunks=P, qpos=P, rowof=P, out=P, kv=256, heads=2, head_dim=128,
                        tab_ld=64)
    for k, v in kw.items():
        setattr(a, k, v)
    return a


CASES = [
    ("embed_assemble", lambda L: L.vlc_embed_assemble(P, 256, P, 256, None, None, P, -1, None),
     N.VLC_ERR_INVALID, "embed_assemble: bad args"),
    ("rmsnorm null", lambda L: L.vlc_rmsnorm(None, 256, P, P, 256, 0, 4, 256, None, 1e-6, 0, 0, None),
     N.VLC_ERR_INVALID, "rmsnorm: bad args"),
    ("rmsnorm packed f32", lambda L: L.vlc_rmsnorm(P, 256, P, P, 256, 1, 4, 256, None, 1e-6, 16, 2, None),
     N.VLC_ERR_INVALID, "packed output needs bf16"),
    ("add_rmsnorm", lambda L: L.vlc_add_rmsnorm(P, 256, None, 256, P, P, 256, 4, 256, 1e-6, 0, 0, None),
     N.VLC_ERR_INVALID, "add_rmsnorm: bad args"),
    ("kv_relocate head_dim", lambda L: L.vlc_kv_relocate(P, P, 64, P, 240, 12, P, P, 8, P, P, 1, P, P, 6, None),
     N.VLC_ERR_UNSUPPORTED, "head_dim must be a multiple of 16"),
    ("kv_relocate tab_ld", lambda L: L.vlc_kv_relocate(P, P, 64, P, 256, 128, P, P, 8, P, P, 1, P, P, 128, None),
     N.VLC_ERR_INVALID, "tab_ld must be head_dim/2"),
    ("kv_relocate V without pool", lambda L: L.vlc_kv_relocate(P, None, 64, P, 256, 128, P, P, 8, P, P, 1, P, P,
                                                                64, None),
     N.VLC_ERR_INVALID, "kv_relocate: null pointer"),
    ("store_write_pages", lambda L: L.vlc_store_write_pages(P, 1, 0, 64, 256, P, 1, P, 64, None),
     N.VLC_ERR_INVALID, "store_write_pages: bad args"),
    ("pack_operand", lambda L: L.vlc_pack_operand(P, 10, 256, 256, P, 12, 2, None),
     N.VLC_ERR_INVALID, "pack_operand: bad args"),
    ("gemm null", lambda L: L.vlc_gemm_bf16(None, 256, 256, P, 256, 16, C.byref(_epi(m_tokens=16)), 0, None, 0,
                                            None, None),
     N.VLC_ERR_INVALID, "gemm: null pointer"),
    ("gemm shape", lambda L: L.vlc_gemm_bf16(P, 200, 256, P, 256, 16, C.byref(_epi(m_tokens=16)), 0, None, 0,
                                             None, None),
     N.VLC_ERR_UNSUPPORTED, "multiples of 128"),
    ("attn null", lambda L: L.vlc_attn_paged(C.byref(_attn(q=None)), None),
     N.VLC_ERR_INVALID, "attn_paged: null pointer"),
    ("attn head_dim", lambda L: L.vlc_attn_paged(C.byref(_attn(head_dim=48, kv=96)), None),
     N.VLC_ERR_UNSUPPORTED, "head_dim must be 16/32/64/128"),
    ("attn kv", lambda L: L.vlc_attn_paged(C.byref(_attn(kv=512)), None),
     N.VLC_ERR_INVALID, "kv != heads*head_dim"),
    ("attn store chunks", lambda L: L.vlc_attn_paged(C.byref(_attn(pool_k=P)), None),
     N.VLC_ERR_INVALID, "store chunks need pools"),
    ("attn co-residency", lambda L: L.vlc_attn_paged(C.byref(_attn(ws_slots=1, counters=P, ws_o=P, ws_ml=P,
                                                                   n_items=149)), None),
     N.VLC_ERR_INVALID, "<= 148 items"),
    ("gather_rows", lambda L: L.vlc_gather_rows(P, P, P, P, 4, 10, None),
     N.VLC_ERR_INVALID, "gather_rows: bad args"),
    ("patchify", lambda L: L.vlc_patchify(P, 30, 4, P, 0, 16, 1, None),
     N.VLC_ERR_INVALID, "patchify: bad args"),
    ("set_tuning", lambda L: L.vlc_set_tuning(12345, 1),
     N.VLC_ERR_INVALID, "unknown key"),
    ("copy_h2d", lambda L: L.vlc_copy_h2d_async(None, P, 16, None),
     N.VLC_ERR_INVALID, "copy_h2d: null pointer"),
]


@pytest.mark.parametrize("name,call,status,msg", CASES, ids=[c[0] for c in CASES])
def test_entry_point_rejects_bad_arguments(lib, name, call, status, msg):
    st = call(lib)
    assert st == status, (name, st, _err(lib))
    assert msg in _err(lib)


def test_binding_maps_status_to_reference_exceptions(lib):
    with pytest.raises(InputError, match="pack_operand"):
        N.check(lib.vlc_pack_operand(P, 10, 256, 256, P, 12, 2, None), "pack")
    with pytest.raises(N.NativeError, match="multiples of 128"):
        N.check(lib.vlc_gemm_bf16(P, 200, 256, P, 256, 16, C.byref(_epi(m_tokens=16)), 0, None, 0, None, None),
                "gemm")
    N.check(0, "ok")                                   # VLC_OK passes through
