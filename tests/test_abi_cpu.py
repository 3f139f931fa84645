"""The C-ABI library loads without a GPU and exports every entry point include/vlcache.h
declares; the product path refuses to run without CUDA (no CPU fallback)."""
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "vlcache.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vlc_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2512_12977_b200 import _build, _native
    _build.build()
    return _native.load()


def test_header_declares_the_minimum_set():
    names = _declared()
    for n in ("vlc_last_error", "vlc_embed_assemble", "vlc_gather_rows", "vlc_kv_relocate", "vlc_rmsnorm", "vlc_gemm_bf16",
              "vlc_attn_paged", "vlc_store_write_pages"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2512_12977_b200 import _native
    names = _declared()
    for n in names:
        assert hasattr(lib, n), n
    assert set(_native.EXPORTS) <= set(names)
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (vlc_[a-z0-9_]+)", out))
    assert set(names) <= exported, set(names) - exported


def test_library_is_sm100a_cubin(lib):
    from paper_2512_12977_b200 import _native
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_error_without_device(lib):
    assert lib.vlc_version() > 0
    assert isinstance(lib.vlc_last_error(), bytes)


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    import paper_2512_12977_b200 as P
    from paper_2512_12977_b200._native import NativeError
    import numpy as np
    k = np.zeros((1, 4, 8), np.float32)
    with pytest.raises(NativeError):
        P.CacheStore().put_kv(P.KVCacheEntry(P.hash_image(k), k, k, 0, 0))
    cfg = P.ModelConfig(num_layers=1, num_heads=2, model_dim=16, kv_dim=16, vocab_size=11, patch_size=2,
                        tokens_per_image=4)
    with pytest.raises(NativeError):
        P.init_model(cfg).device
