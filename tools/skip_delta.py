"""In-graph cost of each kernel kind of the C3 chain: TTFT with that kind left out of the captured graph
(wrong results; timing only), by monkeypatching the Runner's launch methods in this process only.
  python tools/skip_delta.py"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2512_12977_b200 as P  # noqa: E402
from paper_2512_12977_b200 import runtime as RT  # noqa: E402
from paper_2512_12977_b200.engine import _runner, prefill_with_reuse  # noqa: E402
from paper_2512_12977_b200.toydata import make_images, prompt_ids  # noqa: E402

wl = bench.WORKLOADS["C3"]
cfg = P.ModelConfig(**bench.CONFIGS["C3"], seed=0)
L = cfg.num_layers
model = P.ToyVLM.device_random(cfg, seed=0)
runner = _runner(model)
store = P.CacheStore()
images = make_images(4, cfg.image_side, 1)
P.fill_store(model, store, images, prompt_ids(cfg.vocab_size, 8, 11))
text = prompt_ids(cfg.vocab_size, 32, 12)
seq = P.make_sequence(text[:16], 4, cfg.tokens_per_image, text[16:])
req = P.ReuseRequest(seq, [P.hash_image(p) for p in images], P.plan_static(0.05, L))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
orig_gemm, orig_norm, orig_attn = RT.Runner.gemm, RT.Runner.rmsnorm, RT.Runner.attention


def ttft(n=15):
    runner.graphs.clear()
    for _ in range(3):
        prefill_with_reuse(model, req, store)
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        prefill_with_reuse(model, req, store)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def skip_gemm(name):
    def g(self, *a, **k):
        if k.get("name") == name:
            return None
        return orig_gemm(self, *a, **k)
    return g


variants = [("none", {}), ("rmsnorm (57x)", {"rmsnorm": lambda self, *a, **k: None}),
            ("attention (28x)", {"attention": lambda self, *a, **k: None})]
variants += [(f"{nm} (x{28 if nm != 'gemm_head' else 1})", {"gemm": skip_gemm(nm)})
             for nm in ("gemm_qkv", "gemm_o", "gemm_gate_up", "gemm_down", "gemm_head")]
base = None
for rnd in range(2):
    for label, patch in variants:
        RT.Runner.gemm, RT.Runner.rmsnorm, RT.Runner.attention = orig_gemm, orig_norm, orig_attn
        for k, f in patch.items():
            setattr(RT.Runner, k, f)
        t = ttft()
        if label == "none":
            base = t
        if rnd == 1:
            print(f"{label:22s} TTFT {t:.3f} ms   in-graph cost {base - t:+.3f} ms", flush=True)
RT.Runner.gemm, RT.Runner.rmsnorm, RT.Runner.attention = orig_gemm, orig_norm, orig_attn
