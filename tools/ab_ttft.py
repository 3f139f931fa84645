"""A/B of chain variants on the C3 bench request (same process, same weights / store): p50 device
TTFT per variant, alternating rounds.  Variants are Runner attributes: defer_norm (deferred RMSNorm)
and env-free schedule toggles passed as NAME=attr:value,... on the command line.

  python tools/ab_ttft.py base= nonorm=defer_norm:0
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2512_12977_b200 as P  # noqa: E402
from paper_2512_12977_b200 import _native as N  # noqa: E402
if os.environ.get("VLC_LIB_VARIANT"):          # experiment builds (tools/build_variant.py)
    N.LIB_PATH = os.environ["VLC_LIB_VARIANT"]
for kv in filter(None, os.environ.get("VLC_TUNING", "").split(",")):   # e.g. VLC_TUNING=17:1,10:0
    N.load().vlc_set_tuning(*(int(x) for x in kv.split(":")))
from paper_2512_12977_b200.engine import _runner, prefill_with_reuse  # noqa: E402
from paper_2512_12977_b200.toydata import make_images, prompt_ids  # noqa: E402

wl = bench.WORKLOADS[os.environ.get("WL", "C3")]
cfg = P.ModelConfig(**bench.CONFIGS[wl["cfg"]], seed=0)
T, V, L = cfg.tokens_per_image, cfg.vocab_size, cfg.num_layers
model = P.ToyVLM.device_random(cfg, seed=0)
runner = _runner(model)
store = P.CacheStore()
images = make_images(wl["images"], cfg.image_side, 1)
P.fill_store(model, store, images, prompt_ids(V, 8, 11))
text = prompt_ids(V, 32, 12)
seq = P.make_sequence(text[:16], wl["images"], T, text[16:])
hashes = [P.hash_image(px) for px in images]
ratio = float(os.environ.get("RATIO", wl["ratio"]))
req = P.ReuseRequest(seq, hashes, P.plan_static(ratio, L))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

variants = {}
for a in sys.argv[1:]:
    name, _, spec = a.partition("=")
    variants[name] = [(k, int(v)) for k, v in (kv.split(":") for kv in spec.split(",") if kv)]
if not variants:
    variants = {"base": []}
# NAME=attr:value sets a Runner attribute; NAME=@key:value a vlc_set_tuning key (default from TUNE_DEFAULTS)
TUNE_DEFAULTS = {16: 1, 17: 2, 18: 1, 9: 64, 10: 160, 7: 1}
defaults = {k: (TUNE_DEFAULTS[int(k[1:])] if k.startswith("@") else getattr(runner, k))
            for v in variants.values() for k, _ in v}


def apply(v):
    from paper_2512_12977_b200 import _native as N
    for k, val in list(defaults.items()) + list(v):
        if k.startswith("@"):
            N.load().vlc_set_tuning(int(k[1:]), int(val))
        else:
            setattr(runner, k, bool(val) if isinstance(defaults[k], bool) else val)
    runner.graphs.clear()              # launch configurations are captured with the graph


res = {n: [] for n in variants}
last = {}
for rnd in range(4):
    for n, v in variants.items():
        apply(v)
        for _ in range(3):
            prefill_with_reuse(model, req, store)
        torch.cuda.synchronize()
        for _ in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = prefill_with_reuse(model, req, store)
            e1.record()
            e1.synchronize()
            res[n].append(e0.elapsed_time(e1))
        last[n] = r.last_logits().copy()
base = next(iter(variants))
for n in variants:
    d = float(abs(last[n] - last[base]).max())
    print(f"{n:12s} p50 {statistics.median(res[n]):.4f} ms  min {min(res[n]):.4f}  "
          f"max|last - {base}| {d:.3e}", flush=True)
