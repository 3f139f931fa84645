"""Store persistence interop (store.py:159-241) on CPU: the reference's on-disk format
(tests/golden/ref_store, written by the real reference, make_ref_store.py) and the integrity checks
that fire before any entry reaches the device (test_store.py:131-193)."""
import json
import os
import shutil

import pytest

import paper_2512_12977_b200 as P
from conftest import GOLDEN
from paper_2512_12977_b200 import store as S

REF_STORE = os.path.join(GOLDEN, "ref_store")


@pytest.fixture
def copy(tmp_path):
    d = tmp_path / "store"
    shutil.copytree(REF_STORE, d)
    return d


def _enc_blob(d):
    m = json.loads((d / "manifest.json").read_text())
    key = next(k for k in m["entries"] if k.startswith("encoder/"))
    return d / m["entries"][key]["blob"]


def test_reference_manifest_matches_our_format():
    m = json.loads(open(os.path.join(REF_STORE, S.MANIFEST_NAME)).read())
    assert m["format"] == S.STORE_FORMAT and m["digest_algo"] == S.DIGEST_ALGO
    kinds = sorted(v["kind"] for v in m["entries"].values())
    assert kinds == ["encoder", "kv"]
    for key, meta in m["entries"].items():
        assert meta["blob"] == f"blobs/{meta['sha256']}.bin"
        arr = S._read_blob(__import__("pathlib").Path(REF_STORE), key, meta)     # checksum + size verified
        assert list(arr.shape) == meta["shape"]


def test_truncated_blob(copy):
    b = _enc_blob(copy)
    b.write_bytes(b.read_bytes()[:-4])
    with pytest.raises(P.IntegrityError, match="bytes"):
        P.CacheStore.load(copy)


def test_flipped_byte(copy):
    b = _enc_blob(copy)
    raw = bytearray(b.read_bytes())
    raw[7] ^= 0x40
    b.write_bytes(bytes(raw))
    with pytest.raises(P.IntegrityError, match="checksum"):
        P.CacheStore.load(copy)


def test_missing_blob_and_manifest(copy):
    _enc_blob(copy).unlink()
    with pytest.raises(P.IntegrityError, match="missing blob"):
        P.CacheStore.load(copy)
    (copy / "manifest.json").write_text("{not json")
    with pytest.raises(P.IntegrityError, match="corrupt manifest"):
        P.CacheStore.load(copy)
    (copy / "manifest.json").unlink()
    with pytest.raises(P.IntegrityError, match="no manifest"):
        P.CacheStore.load(copy)


def test_unknown_format(copy):
    m = json.loads((copy / "manifest.json").read_text())
    m["format"] = "something-else"
    (copy / "manifest.json").write_text(json.dumps(m))
    with pytest.raises(P.IntegrityError, match="unknown store format"):
        P.CacheStore.load(copy)
