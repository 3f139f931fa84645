#!/usr/bin/env python
"""TTFT benchmark of the B200 VLCache reuse prefill (BASELINE.json metric).

Default workload (config.workload): the Qwen2.5-VL-7B-shape reuse prefill of
BASELINE configs[2] in reference semantics -- 28 layers, d = kv = 3584, 28
heads, V = 152064; 4 cached images x 1024 tokens reused at SHIFTED positions
(cached under an 8-token prefix, reused after a 16-token prefix) + 32 text
tokens; static 5% recompute.  A "step" is one `prefill_with_reuse` of that
request.  Weights are random-init on the device (same distributions as the
reference); images/prompts come from the reference's seeded generators.

  value      p50 device TTFT (ms) with inputs resident in HBM, L2 flushed
             between steps; max over ranks.
  e2e        same call through the public API with host inputs: wall time from
             prefill_with_reuse() entry to the last-row logits on the host.
  roofline   dominant kernel from a CUDA-event-traced pass.
  cpu_baseline  the CPU oracle (numpy restatement of the reference) on a bounded
             sample: 2 of the 28 layers timed per layer, extrapolated.

`--impl reference` prints the CPU arm only (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "p50 TTFT ms (reuse@2-5% vs full prefill) at 1/2/4/8 B200; logit err vs CPU"
CONFIGS = {
    "C1": dict(num_layers=4, num_heads=8, model_dim=256, kv_dim=256, vocab_size=4096, patch_size=4,
               tokens_per_image=256),
    "C2": dict(num_layers=28, num_heads=12, model_dim=1536, kv_dim=1536, vocab_size=151936, patch_size=4,
               tokens_per_image=1024),
    "C3": dict(num_layers=28, num_heads=28, model_dim=3584, kv_dim=3584, vocab_size=152064, patch_size=4,
               tokens_per_image=1024),
}
WORKLOADS = {
    "C3": dict(cfg="C3", images=4, ratio=0.05,
               desc="Qwen2.5-VL-7B shape (ref semantics L28 d=kv=3584 H28 h7168 V152064), 4x1024 cached image "
                    "tokens reused at shifted positions + 32 text, static 5% recompute"),
    "C2": dict(cfg="C2", images=1, ratio=0.03,
               desc="Qwen2-VL-2B shape (ref semantics L28 d=kv=1536 H12 h3072 V151936), 1024 image tokens, 3%"),
    "C1": dict(cfg="C1", images=1, ratio=0.05, desc="tiny L4 d256 H8, 256 image + 32 text, 5%"),
    "C5": dict(cfg="C2", images=2, ratio=0.03, requests=64, pool=8, micro=8,
               desc="64 concurrent requests sharing 8 cached images (Qwen2-VL-2B shape, ref semantics), each "
                    "16 text + 2 seeded images x 1024 tokens + 16 text, 3% recompute; requests sharded "
                    "round-robin over ranks, micro-batches of 8 requests per device pass"),
}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", p["bf16_tflops"])), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.lines, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- CPU arm (oracle port)

class CpuSample:
    """Bounded sample of the reference algorithm on host cores: the oracle's reuse prefill
    over `sample_layers` of the layers (same d/kv/H/V/T, sequence and plan) with random
    weights / cached KV of the workload shape; per-layer time extrapolated to full depth."""

    def __init__(self, cfg_kw: dict, images: int, ratio: float, sample_layers: int = 2, seed: int = 0):
        from oracle import kvreuse_oracle as O
        self.O, self.L, self.ratio, self.sl = O, cfg_kw["num_layers"], ratio, sample_layers
        self.c = c = O.Cfg(**{**cfg_kw, "num_layers": sample_layers, "seed": seed})
        g = np.random.default_rng(seed)
        d, kv, h, V, T = c.model_dim, c.kv_dim, c.hidden, c.vocab_size, c.tokens_per_image

        def rnd(*shape, scale=1.0):   # uniform, variance-matched: timing does not depend on values
            a = g.random(shape, dtype=np.float32)
            a -= np.float32(0.5)
            a *= np.float32(scale * 3.4641016)
            return a

        w = {"embed": rnd(V, d), "head": rnd(d, V, scale=d ** -0.5), "final_norm": np.ones(d, np.float32)}
        for i in range(sample_layers):
            w.update({f"l{i}_attn_norm": np.ones(d, np.float32), f"l{i}_mlp_norm": np.ones(d, np.float32),
                      f"l{i}_wq": rnd(d, kv, scale=d ** -0.5), f"l{i}_wk": rnd(d, kv, scale=d ** -0.5),
                      f"l{i}_wv": rnd(d, kv, scale=d ** -0.5), f"l{i}_wo": rnd(kv, d, scale=kv ** -0.5),
                      f"l{i}_w_gate": rnd(d, h, scale=d ** -0.5), f"l{i}_w_up": rnd(d, h, scale=d ** -0.5),
                      f"l{i}_w_down": rnd(h, d, scale=h ** -0.5)})
        text = O.prompt(V, 32, 12)
        self.ids, self.segs = O.layout(text[:16], images, T, text[16:])
        self.enc, self.kvs, self.hashes = {}, {}, []
        for m in range(images):
            key = f"{m:064x}"
            self.hashes.append(key)
            self.enc[key] = rnd(T, d)
            self.kvs[key] = O.KVEntry(rnd(sample_layers, T, kv), rnd(sample_layers, T, kv), 8)
        self.w = w

    def run(self):
        tm = {}
        self.O.reuse_prefill(self.c, self.w, self.ids, self.segs, self.hashes, (self.ratio,) * self.sl,
                             self.enc, self.kvs, timings=tm)
        per_layer = statistics.mean(tm["layers"])
        ttft = tm["resolve"] * self.L / self.sl + tm["embed"] + per_layer * self.L + tm["head"]
        return ttft * 1e3, {"sample_layers": self.sl, "per_layer_s": per_layer, "resolve_s": tm["resolve"],
                            "head_s": tm["head"]}


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args, wl):
    cfg_kw = CONFIGS[wl["cfg"]]
    times = []
    # one sampled layer per step (the per-layer time x L extrapolation) keeps a default run of the
    # arm within a few minutes on the host cores
    sample = CpuSample(cfg_kw, wl["images"], wl["ratio"], sample_layers=1)
    for step in range(args.warmup + args.steps):
        ms, det = sample.run()
        if step >= args.warmup:
            times.append(ms)
    v = statistics.median(times)
    cores = cpu_cores()
    sample = (f"oracle (numpy restatement of kvreuse.prefill_with_reuse) over {det['sample_layers']} of "
              f"{cfg_kw['num_layers']} layers per step, per-layer time x {cfg_kw['num_layers']} + resolve/head; "
              f"BLAS threads = all {cores} cores")
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "ms", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(statistics.mean(times), 3),
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded prompts, random weights/KV of the workload shape)",
            "config": {"workload": wl["desc"], "recompute": wl["ratio"], "image_tokens": wl["images"] * 1024,
                       "text_tokens": 32},
            "cpu_baseline": {"value": round(v, 3), "unit": "ms", "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": round(v, 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm

def _flush_l2(buf):
    buf.add_(1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C3", choices=list(WORKLOADS),
                    help="C3: the BASELINE metric (TTFT); C5: aggregate tokens/s of batched requests")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--parallel", default="replicas", choices=["replicas", "heads"],
                    help="N>1: independent requests per rank (default) or head-parallel attention on one "
                         "request (one NCCL all-reduce per layer)")
    ap.add_argument("--trace", default="", help="write per-kernel trace json here")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    wl = WORKLOADS[args.workload]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        if rank == 0:
            run_reference(args, wl)
        return

    import torch
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2512_12977_b200 as P
    from paper_2512_12977_b200.engine import _runner, prefill_with_reuse
    from paper_2512_12977_b200 import runtime as RT
    if args.workload == "C5":
        run_c5(args, wl, P, rank, world, local, dist)
        return

    cfg = P.ModelConfig(**CONFIGS[wl["cfg"]], seed=0)
    T, V, L = cfg.tokens_per_image, cfg.vocab_size, cfg.num_layers
    head_par = args.parallel == "heads" and world > 1
    model = P.ToyVLM.device_random(cfg, seed=0, tp_group=dist.group.WORLD if head_par else None)
    runner = _runner(model)
    store = P.CacheStore()
    from paper_2512_12977_b200.toydata import make_images, prompt_ids
    images = make_images(wl["images"], cfg.image_side, 1 if head_par else 1 + rank)
    P.fill_store(model, store, images, prompt_ids(V, 8, 11))          # device miss path
    text = prompt_ids(V, 32, 12)
    seq = P.make_sequence(text[:16], wl["images"], T, text[16:])
    hashes = [P.hash_image(px) for px in images]
    plan = P.plan_static(wl["ratio"], L)
    req = P.ReuseRequest(seq, hashes, plan)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def timed(request, st, steps, warmup):
        for _ in range(warmup):
            prefill_with_reuse(model, request, st)
        torch.cuda.synchronize()
        out = []
        for _ in range(steps):
            _flush_l2(flush)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            prefill_with_reuse(model, request, st)
            e1.record()
            e1.synchronize()
            out.append(e0.elapsed_time(e1))
        return out

    # ---- warmup + timed region (device TTFT, inputs resident)
    for _ in range(args.warmup):
        prefill_with_reuse(model, req, store)
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = runner.launches
    t_wall0 = time.perf_counter()
    step_ms = []
    for _ in range(args.steps):
        _flush_l2(flush)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        prefill_with_reuse(model, req, store)
        e1.record()
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    region_s = time.perf_counter() - t_wall0
    launches = runner.launches - launches0
    p50 = statistics.median(step_ms)
    mean = statistics.mean(step_ms)
    # ---- e2e through the public API (host inputs, last-row logits to host)
    e2e = []
    bytes_h2d = 0
    for _ in range(args.steps):
        _flush_l2(flush)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = prefill_with_reuse(model, req, store)
        last = res.last_logits()
        e2e.append((time.perf_counter() - t0) * 1e3)
        bytes_h2d = int(getattr(runner.ws, "last_h2d_bytes", runner.ws.bufs["ints"].numel() * 4))
    clocks = sampler.stop()
    if dist:
        t = torch.tensor([p50, mean, statistics.median(e2e)], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        p50, mean, e2e_p50 = (float(v) for v in t.tolist())
    else:
        e2e_p50 = statistics.median(e2e)

    # ---- baselines on the same GPU: full recompute (no_vit) and origin (GPU ViT + full)
    full_ms = statistics.median(timed(P.ReuseRequest(seq, hashes, P.plan_static(1.0, L)), store, 5, 2))
    origin_ms = statistics.median(timed(P.ReuseRequest(seq, hashes, P.plan_static(1.0, L), images=images),
                                        P.CacheStore(), 3, 1))
    c4 = layer_aware_vs_uniform(P, model, seq, hashes, store, L, timed) if args.workload == "C3" else None
    sweep = {}
    for r in (0.02, 0.03, 0.04, 0.05):
        sweep[str(r)] = round(statistics.median(timed(P.ReuseRequest(seq, hashes, P.plan_static(r, L)), store,
                                                      7, 2)), 4)

    # ---- per-kernel trace (separate pass, events around each launch)
    hbm, tf_burst, tf_sust, peak_src = _peaks()
    runner.tracer = []
    ntrace = 5
    for _ in range(ntrace):
        _flush_l2(flush)
        prefill_with_reuse(model, req, store)
    torch.cuda.synchronize()
    agg = {}
    for name, e0, e1, nb, fl in runner.tracer:
        a = agg.setdefault(name, [0.0, 0, 0, 0])
        a[0] += e0.elapsed_time(e1)
        a[1] += 1
        a[2] += nb
        a[3] += fl
    runner.tracer = None
    total_k = sum(v[0] for v in agg.values())
    kernels = []
    for name, (ms, cnt, nb, fl) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        s = ms / 1e3
        kernels.append({"name": name, "ms_per_step": round(ms / ntrace, 4), "launches_per_step": cnt // ntrace,
                        "share": round(ms / total_k, 4), "GBps": round(nb / s / 1e9, 1) if nb else None,
                        "TFps": round(fl / s / 1e12, 2) if fl else None})
    dom = kernels[0]
    dname = dom["name"]
    try:   # DRAM bytes per launch from the committed ncu --set full capture (tools/ncu_traffic.py)
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            traffic = json.load(fh)
    except (OSError, ValueError):
        traffic = {}
    ms_d, cnt_d, nb_d, fl_d = agg[dname]
    if dname.startswith("gemm") or dname in ("kv_relocate", "rmsnorm", "embed"):
        ach = nb_d / (ms_d / 1e3) / 1e9
        roof = {"kernel": dname, "bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(ach / hbm, 4), "traffic": traffic.get(dname, {}).get("dram_bytes"),
                "algorithmic": f"{nb_d / cnt_d / 1e6:.2f} MB per launch (bf16 weights + activations)",
                "peak_source": f"{peak_src} hbm_gbs"}
    else:
        ach = fl_d / (ms_d / 1e3) / 1e12
        roof = {"kernel": dname, "bound": "tensor", "achieved": round(ach, 2), "peak": tf_burst, "unit": "TFLOP/s",
                "frac": round(ach / tf_burst, 4), "traffic": traffic.get(dname, {}).get("dram_bytes"),
                "peak_source": f"{peak_src} bf16_tflops"}
    others = {}
    for k in ("kv_relocate", "attention"):
        if k in agg:
            ms_k, c_k, nb_k, fl_k = agg[k]
            if k == "kv_relocate":
                a = nb_k / (ms_k / 1e3) / 1e9
                others[k] = {"bound": "hbm", "achieved": round(a, 1), "peak": hbm, "unit": "GB/s",
                             "frac": round(a / hbm, 4)}
            else:
                a = fl_k / (ms_k / 1e3) / 1e12
                others[k] = {"bound": "tensor", "achieved": round(a, 2), "peak": tf_burst, "unit": "TFLOP/s",
                             "frac": round(a / tf_burst, 4), "note": "causal-effective FLOPs"}
    # kv_relocate against its own roofline: the production chain runs it per layer on a low-priority
    # side stream as wide CTAs that only fill idle SMs (its event times above include that
    # sharing); here the same relocation runs as ONE launch of the full-rate kernel, alone.
    try:
        runner.tracer, runner.overlap_reloc = [], False
        runner.lib.vlc_set_tuning(14, 0)
        for _ in range(3):
            _flush_l2(flush)
            prefill_with_reuse(model, req, store)
        torch.cuda.synchronize()
        rl = [(e0.elapsed_time(e1), nb) for name, e0, e1, nb, fl in runner.tracer if name == "kv_relocate"]
        if rl:
            ms_r, nb_r = statistics.median(x[0] for x in rl), rl[0][1]
            a = nb_r / (ms_r / 1e3) / 1e9
            others["kv_relocate_single_launch"] = {
                "bound": "hbm", "achieved": round(a, 1), "peak": hbm, "unit": "GB/s", "frac": round(a / hbm, 4),
                "us": round(ms_r * 1e3, 1), "algorithmic": f"{nb_r / 1e6:.1f} MB (all layers; K+V read + write)"}
    finally:
        runner.tracer, runner.overlap_reloc = None, RT._OVERLAP_RELOC
        runner.lib.vlc_set_tuning(14, int(os.environ.get("VLC_RELOC_WIDE", "100000")))
    if args.trace:
        with open(args.trace, "w") as fh:
            json.dump({"kernels": kernels, "agg": {k: v for k, v in agg.items()}}, fh, indent=1)

    # ---- parity vs CPU oracle on configs[0] (C1), bf16-rounded weights
    parity = None
    if rank == 0:
        try:
            parity = parity_c1(P)
        except Exception as exc:  # never hide it: report in the line
            parity = {"error": repr(exc)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cs = CpuSample(CONFIGS[wl["cfg"]], wl["images"], wl["ratio"])
        cs.run()
        ms_cpu, det = cs.run()
        cores = cpu_cores()
        cpu = {"value": round(ms_cpu, 2), "unit": "ms", "cores": cores, "kind": "port",
               "sample": f"oracle reuse prefill over {det['sample_layers']}/{L} layers, per-layer x {L} "
                         f"(+resolve, head); numpy/OpenBLAS on {cores} threads"}

    n_tok = len(seq)
    c = prefill_with_reuse(model, req, store).metrics.computed_per_layer
    if rank == 0:
        line = {"metric": METRIC, "value": round(p50, 4), "unit": "ms", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(mean, 4), "higher_is_better": False,
                "scaling": "strong" if head_par else "weak", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic: device random-init weights (reference distributions), seeded toydata images "
                        "and prompts; store filled by the device miss path",
                "config": {"workload": wl["desc"], "recompute": wl["ratio"], "image_tokens": wl["images"] * T,
                           "text_tokens": 32, "seq_len": n_tok, "computed_rows_layer0": c[0],
                           "l2": "flushed between steps (512 MiB write); weights 9.6 GB >> L2",
                           "parallelism": (f"head-parallel attention over {world} GPUs (one NCCL all-reduce "
                                           f"per layer)" if head_par else
                                           f"replica per GPU x{world} (independent requests, no collective)")},
                "e2e": {"value": round(e2e_p50, 4), "unit": "ms", "h2d_bytes_per_step": bytes_h2d,
                        "d2h_bytes_per_step": V * 4,
                        "note": "wall clock: prefill_with_reuse() entry -> last-row logits on host"},
                "roofline": roof, "roofline_other": others, "kernels": kernels,
                "cpu_baseline": cpu, "gpu_launches": launches, "clocks": clocks,
                "full_prefill_ms": round(full_ms, 3), "origin_ms": round(origin_ms, 3),
                "speedup_vs_full_prefill": round(full_ms / p50, 2), "speedup_vs_origin": round(origin_ms / p50, 2),
                "sweep_p50_ms": sweep, "layer_aware_vs_uniform": c4, "parity_vs_cpu": parity,
                "prefill_tokens_per_s": round((1 if head_par else world) * n_tok / (p50 / 1e3), 1),
                "timed_region_s": round(region_s, 3)}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_c5(args, wl, P, rank, world, local, dist):
    """BASELINE configs[4]: independent requests sharded over ranks (no collective on the data
    path), each rank serving its shard in batched device passes (prefill_batch_with_reuse)."""
    import torch
    from paper_2512_12977_b200.sharding import shard_indices
    from paper_2512_12977_b200.toydata import make_images, prompt_ids
    cfg = P.ModelConfig(**CONFIGS[wl["cfg"]], seed=0)
    T, V, L = cfg.tokens_per_image, cfg.vocab_size, cfg.num_layers
    model = P.ToyVLM.device_random(cfg, seed=0)
    store = P.CacheStore()
    pool = make_images(wl["pool"], cfg.image_side, 1)
    P.fill_store(model, store, pool, prompt_ids(V, 8, 11))
    hashes = [P.hash_image(px) for px in pool]
    rng = np.random.default_rng(5)
    reqs, n_tok = [], []
    plan = P.plan_static(wl["ratio"], L)
    for i in range(wl["requests"]):
        pick = rng.choice(wl["pool"], wl["images"], replace=False)
        text = prompt_ids(V, 32, 100 + i)
        seq = P.make_sequence(text[:16], wl["images"], T, text[16:])
        reqs.append(P.ReuseRequest(seq, [hashes[k] for k in pick], plan))
        n_tok.append(len(seq))
    mine = shard_indices(len(reqs), rank, world)
    batches = [[reqs[i] for i in mine[b:b + wl["micro"]]] for b in range(0, len(mine), wl["micro"])]

    def step():
        last = None
        for b in batches:
            last = P.prefill_batch_with_reuse(model, b, store)
        return last

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ms = []
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step()
        e1.record()
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    clocks = sampler.stop()
    p50 = statistics.median(ms)
    if dist:
        t = torch.tensor([p50], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        p50 = float(t.item())
    total_tok = sum(n_tok)
    computed = sum(len(r.seq) - sum(s.length for s in r.seq.image_segments) +
                   len(r.seq.image_segments) * P.recompute_count(wl["ratio"], T) for r in reqs)
    if rank == 0:
        print(json.dumps({
            "metric": "aggregate prefill tokens/s (BASELINE configs[4])", "value": round(total_tok / (p50 / 1e3), 1),
            "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(p50, 3), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (device random weights, seeded toydata images/prompts)",
            "config": {"workload": wl["desc"], "requests": len(reqs), "prompt_tokens": total_tok,
                       "computed_tokens_per_layer": computed, "micro_batch": wl["micro"],
                       "parallelism": f"request sharding over {world} rank(s), no collective"},
            "computed_tokens_per_s": round(computed / (p50 / 1e3), 1), "clocks": clocks}), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def layer_aware_vs_uniform(P, model, seq, hashes, store, L, timed):
    """BASELINE configs[3]: the greedy layer-wise allocation (plan_greedy) vs uniform 5% at the
    same budget (P = 0.05 * L): TTFT and last-row logit deviation from full prefill on the same
    GPU.  The sensitivity table is synthetic and pinned (the reference's CPU profiling costs
    L*|grid|+1 dense passes per sample at this size): layer i's score decays with the ratio as
    w_i * exp(-r / 0.04), w_i = 1 / (1 + i / 4) -- shallow layers more sensitive (sec. 3)."""
    source = "synthetic"
    try:       # device-profiled table for this model (tools/profile_table.py), if committed
        with open(os.path.join(ROOT, "profiles", "c3_sensitivity_table.json")) as fh:
            prof = json.load(fh)
        if int(prof["model_fingerprint"]) != model.fingerprint:
            raise ValueError("table profiled for another model")
        table = P.SensitivityTable(np.asarray(prof["scores"]), tuple(prof["grid"]), float(prof["baseline"]),
                                   int(prof["samples"]), model.fingerprint)
        source = f"device-profiled ({prof['samples']} proxy samples, profiles/c3_sensitivity_table.json)"
    except (OSError, ValueError, KeyError):
        grid = tuple(round(0.002 * k, 3) for k in range(1, 151))
        w = 1.0 / (1.0 + np.arange(L) / 4.0)
        scores = w[:, None] * np.exp(-np.asarray(grid)[None, :] / 0.04)
        table = P.SensitivityTable(scores, grid, float(w.max()), 1, model.fingerprint)
    plans = {"uniform": P.plan_static(0.05, L), "layer_aware": P.plan_greedy(table, P.BudgetSpec(0.05 * L))}
    full = prefill_last(P, model, P.ReuseRequest(seq, hashes, P.plan_static(1.0, L)), store)
    out = {"table": source}
    for name, plan in plans.items():
        req = P.ReuseRequest(seq, hashes, plan)
        last = prefill_last(P, model, req, store)
        out[name] = {"mean_ratio": round(P.mean_ratio(plan), 4), "ratios_first_last": [plan.ratios[0], plan.ratios[-1]],
                     "p50_ms": round(statistics.median(timed(req, store, 7, 2)), 4),
                     "last_row_mse_vs_full": float(np.mean((last.astype(np.float64) - full) ** 2)),
                     "last_row_max_abs_vs_full": float(np.abs(last - full).max()),
                     "top1_equal_full": bool(np.argmax(last) == np.argmax(full))}
    return out


def prefill_last(P, model, req, store):
    return P.prefill_with_reuse(model, req, store).last_logits().astype(np.float64)


def parity_c1(P):
    """configs[0] on the GPU vs the CPU oracle, both on the same bf16-rounded weights."""
    from oracle import kvreuse_oracle as O
    kw = dict(CONFIGS["C1"], seed=0)
    oc = O.Cfg(**kw)
    w = {k: O.bf16_round(v) for k, v in O.make_weights(oc).items()}
    model = P.ToyVLM(P.ModelConfig(**kw), w)
    V, T = oc.vocab_size, oc.tokens_per_image
    imgs = O.images(1, oc.side, 1)
    enc, kv = {}, {}
    ids0, segs0 = O.layout(O.prompt(V, 8, 11), 1, T)
    O.fill_one(oc, w, ids0, segs0, imgs, enc, kv)
    store = P.CacheStore()
    h = O.sha256_hex(imgs[0])
    store.put_encoder(P.EncoderCacheEntry(P.ImageHash(h), enc[h], model.fingerprint))
    store.put_kv(P.KVCacheEntry(P.ImageHash(h), kv[h].keys, kv[h].values, 8, model.fingerprint))
    text = O.prompt(V, 32, 12)
    ids, segs = O.layout(text[:16], 1, T, text[16:])
    ref = O.reuse_prefill(oc, w, ids, segs, [h], (0.05,) * 4, enc, kv)
    res = P.prefill_with_reuse(model, P.ReuseRequest(P.make_sequence(text[:16], 1, T, text[16:]),
                                                     [P.ImageHash(h)], P.plan_static(0.05, 4)), store)
    lg = res.logits
    return {"config": "C1 (configs[0])", "rel_err": O.rel_err(lg, ref.logits),
            "max_abs": float(np.abs(lg - ref.logits).max()),
            "top1_last_row_equal": bool(np.argmax(lg[-1]) == np.argmax(ref.logits[-1])),
            "rows_bit_exact": bool(np.array_equal(res.positions, ref.rows)),
            "counts_bit_exact": res.metrics.computed_per_layer == ref.counts, "tolerance": "rel_err <= 2e-2"}


if __name__ == "__main__":
    main()
