"""Persist a small store with the REAL reference (kvreuse 0.1.0) -> tests/golden/ref_store/.

Run in the build container only:  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_ref_store.py

The fixture pins store-persistence interop (store.py:159-241): the drop-in's CacheStore.load must
read the reference's on-disk format (manifest.json + sha256-named little-endian fp32 blobs).
Scene: SMALL_CFG (pkg/tests/conftest.py:7-12), one 16x16 image (make_image(16, 3)) cached under
the 6-token prefix prompt_ids(97, 6, 1) (the small scene of make_golden.py).
"""
import os
import shutil
import sys

REF = os.environ.get("VLC_REF_PATH", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from kvreuse import ModelConfig, init_model  # noqa: E402
from kvreuse.bench import fill_store  # noqa: E402
from kvreuse.store import CacheStore  # noqa: E402
from kvreuse.toydata import make_image, prompt_ids  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_store")

if __name__ == "__main__":
    cfg = ModelConfig(num_layers=4, num_heads=2, model_dim=32, kv_dim=32, vocab_size=97, patch_size=4,
                      tokens_per_image=16, seed=7)
    model = init_model(cfg)
    store = CacheStore()
    fill_store(model, store, [make_image(16, 3)], prompt_ids(97, 6, 1))
    shutil.rmtree(OUT, ignore_errors=True)
    store.persist(OUT)
    print("wrote", OUT, sorted(os.listdir(os.path.join(OUT, "blobs"))))
