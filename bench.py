#!/usr/bin/env python
"""TTFT benchmark of the B200 VLCache reuse prefill (BASELINE.json metric).

Default workload (config.workload): the Qwen2.5-VL-7B-shape reuse prefill of
BASELINE configs[2] in reference semantics -- 28 layers, d = kv = 3584, 28
heads, V = 152064; 4 cached images x 1024 tokens reused at SHIFTED positions
(cached under an 8-token prefix, reused after a 16-token prefix) + 32 text
tokens; static 5% recompute.  A "step" is one `prefill_with_reuse` of that
request.  Weights are random-init on the device (same distributions as the
reference); images/prompts come from the reference's seeded generators.
`--workload C2` is configs[1] (2B shape, one image, dynamic layer-wise 3% budget
from plan_greedy); `--workload C5` is configs[4] (64 requests, aggregate tokens/s).

  value         p50 device TTFT (ms) with inputs resident in HBM, L2 flushed
                between steps; max over ranks.
  e2e           same call through the public API with host inputs: wall time from
                prefill_with_reuse() entry to the last-row logits on the host.
  roofline      dominant kernel from a CUDA-event-traced pass.
  cpu_baseline  the reference's own kvreuse.prefill_with_reuse (installed in
                baseline/_ref; the oracle port if absent) at FULL depth on the same
                weights and the same stored KV as the device run, all host cores.
  parity_vs_cpu the device result of the benchmarked request against that CPU run.

`--impl reference` runs the reference arm only (rank 0): the unmodified reference
package at full depth on the workload's shape, one request per step.
`--gpus N` without a torch.distributed environment re-launches itself under
torch.distributed.run with N ranks (127.0.0.1 rendezvous).
"""
from __future__ import annotations

import argparse
import json
import os

if "reference" in __import__("sys").argv and "WORLD_SIZE" in os.environ:
    # rank 0 of a torchrun launch runs the CPU arm: torchrun sets OMP_NUM_THREADS=1 per rank, so give
    # OpenBLAS (read at numpy import, and ahead of OMP_NUM_THREADS) every host core explicitly
    os.environ["OPENBLAS_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
import socket
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
    "C3": dict(cfg="C3", images=4, ratio=0.05, plan="static",
               desc="Qwen2.5-VL-7B shape (ref semantics L28 d=kv=3584 H28 h7168 V152064), 4x1024 cached image "
                    "tokens reused at shifted positions + 32 text, static 5% recompute"),
    "C2": dict(cfg="C2", images=1, ratio=0.03, plan="greedy",
               desc="Qwen2-VL-2B shape (ref semantics L28 d=kv=1536 H12 h3072 V151936), 1024 image tokens reused "
                    "at a shifted position + 32 text, dynamic layer-wise budget 3% (plan_greedy, P = 0.03 L)"),
    "C1": dict(cfg="C1", images=1, ratio=0.05, plan="static", desc="tiny L4 d256 H8, 256 image + 32 text, 5%"),
    "C5": dict(cfg="C2", images=2, ratio=0.03, requests=64, pool=8, micro=8,
               desc="64 concurrent requests sharing 8 cached images (Qwen2-VL-2B shape, ref semantics), each "
                    "16 text + 2 seeded images x 1024 tokens + 16 text, 3% recompute; requests sharded "
                    "round-robin over ranks, micro-batches of 8 requests per device pass"),
}


def workload_plan(P, wl, L):
    """The workload's plan: plan_static(r), or for the dynamic budget plan_greedy at P = r * L
    (cli.py:222-228) over a diminishing sensitivity table whose shallow layers gain more
    (section 3) -- the same table tests/test_fullscale_parity_gpu.py checks on device
    against the oracle."""
    if wl.get("plan") != "greedy":
        return P.plan_static(wl["ratio"], L)
    grid = tuple(round(0.002 * k, 3) for k in range(1, 51))
    w = np.linspace(2.0, 0.25, L)[:, None]
    gains = w * np.exp(-np.asarray(grid)[None, :] / 0.03) * 0.002
    scores = np.maximum(1.0 - np.cumsum(gains, axis=1), 0.0)
    return P.plan_greedy(P.SensitivityTable(scores, grid, 1.0, 1, 0), P.BudgetSpec(wl["ratio"] * L))


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


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ---------------------------------------------------------------- the reference on the host cores

def reference_package():
    """The UNMODIFIED reference package `kvreuse`, pip-installed into baseline/_ref.
    None when it is not there (the CPU legs then run the oracle port)."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "kvreuse")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    import kvreuse
    return kvreuse


class HostReuse:
    """One reuse prefill of the workload on the host cores, through the reference's public API
    (kvreuse.prefill_with_reuse, engine.py:119-190) or, without it, the oracle restatement.

    kw: ModelConfig fields; w: reference-named fp32 weights; enc / kv: hash hex -> [T, d] rows /
    (keys [L, T, kv], values, origin); text: the 32 live text tokens; ratios: the plan."""

    def __init__(self, kw, w, text, hashes, enc, kv, ratios, fingerprint=1):
        self.K = reference_package()
        self.kind = "reference" if self.K is not None else "port"
        self.ratios = tuple(float(r) for r in ratios)
        T, n_img = kw["tokens_per_image"], len(hashes)
        if self.K is not None:
            K = self.K
            self.model = K.ToyVLM(K.ModelConfig(**kw), w)
            # the fingerprint is a lazily computed, cached property of the immutable model
            # (model.py:221-227): fixing it up front skips hashing 19 GB of weights at setup only
            self.model._fingerprint = int(fingerprint)
            self.store = K.CacheStore()
            for h in hashes:
                ih = K.ImageHash(h)
                self.store.put_encoder(K.EncoderCacheEntry(ih, enc[h], self.model.fingerprint))
                k, v, origin = kv[h]
                self.store.put_kv(K.KVCacheEntry(ih, k, v, int(origin), self.model.fingerprint))
            seq = K.make_sequence(list(text[:16]), n_img, T, suffix=list(text[16:]))
            self.req = K.ReuseRequest(seq, [K.ImageHash(h) for h in hashes], K.RecomputePlan(self.ratios))
        else:
            from oracle import kvreuse_oracle as O
            self.O = O
            self.oc = O.Cfg(**kw)
            self.w, self.keys = w, list(hashes)
            self.enc = enc
            self.kv = {h: O.KVEntry(*kv[h]) for h in hashes}
            self.ids, self.segs = O.layout(list(text[:16]), n_img, T, list(text[16:]))

    def run(self):
        """(seconds, dict of rows / logits / keys / values / counts / misses / fallbacks)."""
        t0 = time.perf_counter()
        if self.K is not None:
            r = self.K.prefill_with_reuse(self.model, self.req, self.store)
            dt = time.perf_counter() - t0
            return dt, dict(rows=np.asarray(r.positions), logits=r.logits, keys=r.kv.keys, values=r.kv.values,
                            counts=list(r.metrics.computed_per_layer), misses=r.metrics.encoder_misses,
                            fallbacks=r.metrics.fallback_images, resolve_s=r.metrics.resolve_seconds)
        r = self.O.reuse_prefill(self.oc, self.w, self.ids, self.segs, self.keys, self.ratios, self.enc, self.kv)
        dt = time.perf_counter() - t0
        return dt, dict(rows=r.rows, logits=r.logits, keys=r.keys, values=r.values, counts=r.counts,
                        misses=r.encoder_misses, fallbacks=r.fallback_images)


def run_reference(args, wl):
    """--impl reference: the reference's prefill_with_reuse at FULL depth on the workload's shape,
    one request per step, on all host cores.  Weights: each layer's matrices share one random
    block per shape (the per-layer arithmetic and memory traffic are those of distinct weights --
    a layer's 0.5 GB far exceeds the CPU caches -- at 1/28 of the host RAM); the store holds random
    pre-RoPE K/V for each image (the resolve copy is the reference's own)."""
    kw = dict(CONFIGS[wl["cfg"]], seed=0)
    L, d, kv, V, T = kw["num_layers"], kw["model_dim"], kw["kv_dim"], kw["vocab_size"], kw["tokens_per_image"]
    h = 2 * d
    g = np.random.default_rng(0)

    def rnd(*shape, scale=1.0):      # uniform, variance-matched: the timing does not depend on values
        a = g.random(shape, dtype=np.float32)
        a -= np.float32(0.5)
        a *= np.float32(scale * 3.4641016)
        return a
    blk = {"attn_norm": np.ones(d, np.float32), "mlp_norm": np.ones(d, np.float32),
           "wq": rnd(d, kv, scale=d ** -0.5), "wk": rnd(d, kv, scale=d ** -0.5), "wv": rnd(d, kv, scale=d ** -0.5),
           "wo": rnd(kv, d, scale=kv ** -0.5), "w_gate": rnd(d, h, scale=d ** -0.5),
           "w_up": rnd(d, h, scale=d ** -0.5), "w_down": rnd(h, d, scale=h ** -0.5)}
    w = {"embed": rnd(V, d), "head": rnd(d, V, scale=d ** -0.5), "final_norm": np.ones(d, np.float32)}
    for i in range(L):
        w.update({f"l{i}_{k}": v for k, v in blk.items()})
    from paper_2512_12977_b200.toydata import prompt_ids
    text = prompt_ids(V, 32, 12)
    hashes = [f"{m + 1:064x}" for m in range(wl["images"])]
    enc = {hh: rnd(T, d) for hh in hashes}
    kvs = {hh: (rnd(L, T, kv), rnd(L, T, kv), 8) for hh in hashes}
    import paper_2512_12977_b200 as P        # host-side planner only (no device work)
    ratios = workload_plan(P, wl, L).ratios
    host = HostReuse(kw, w, text, hashes, enc, kvs, ratios)
    times = []
    for step in range(args.warmup + args.steps):
        dt, _ = host.run()
        if step >= args.warmup:
            times.append(dt * 1e3)
    v = statistics.median(times)
    cores = cpu_cores()
    sample = (f"{'kvreuse 0.1.0 (baseline/_ref)' if host.kind == 'reference' else 'oracle port'} "
              f"prefill_with_reuse, full depth ({L}/{L} layers), one {wl['cfg']} request per step "
              f"(resolve + compute), numpy/OpenBLAS on all {cores} host cores")
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "ms", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(statistics.mean(times), 3),
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded prompts; random weights and cached KV of the workload shape)",
            "config": {"workload": wl["desc"], "recompute": wl["ratio"], "image_tokens": wl["images"] * T,
                       "text_tokens": 32, "plan_ratios_first_last": [ratios[0], ratios[-1]]},
            "cpu_baseline": {"value": round(v, 3), "unit": "ms", "cores": cores, "kind": host.kind,
                             "sample": sample},
            "e2e": {"value": round(v, 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- launcher

def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_relaunch(args) -> bool:
    """`--gpus N` (N > 1) outside torch.distributed: re-run this command as N ranks."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def dry_run(args):
    """Launcher check without a GPU: every rank joins a gloo group; rank 0 prints the world."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.ones(1)
        dist.all_reduce(t)
        n = int(t.item())
        dist.barrier()
        dist.destroy_process_group()
    else:
        n = 1
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks_joined": n, "gpus_flag": args.gpus}), flush=True)


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
                    help="C3: the BASELINE metric (TTFT); C2: configs[1]; C5: aggregate tokens/s of batched requests")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline / parity leg")
    ap.add_argument("--cpu-reps", type=int, default=2, help="reference runs in the cpu_baseline leg")
    ap.add_argument("--parallel", default="replicas", choices=["replicas", "heads"],
                    help="N>1: independent requests per rank (default) or head-parallel attention on one "
                         "request (one NCCL all-reduce per layer)")
    ap.add_argument("--trace", default="", help="write per-kernel trace json here")
    ap.add_argument("--dry-run", action="store_true", help="launcher check only (no GPU work)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    wl = WORKLOADS[args.workload]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        if rank == 0:
            run_reference(args, wl)
        return
    maybe_relaunch(args)
    if args.dry_run:
        dry_run(args)
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
    if args.workload == "C5":
        run_c5(args, wl, P, rank, world, local, dist)
        return

    cfg = P.ModelConfig(**CONFIGS[wl["cfg"]], seed=0)
    T, V, L = cfg.tokens_per_image, cfg.vocab_size, cfg.num_layers
    head_par = args.parallel == "heads" and world > 1
    cpu_leg = rank == 0 and world == 1 and not args.no_cpu
    export = {} if cpu_leg else None          # host copy of the device weights for the CPU leg
    t_setup = time.perf_counter()
    model = P.ToyVLM.device_random(cfg, seed=0, tp_group=dist.group.WORLD if head_par else None, export=export)
    runner = _runner(model)
    store = P.CacheStore()
    from paper_2512_12977_b200.toydata import make_images, prompt_ids
    images = make_images(wl["images"], cfg.image_side, 1 if head_par else 1 + rank)
    P.fill_store(model, store, images, prompt_ids(V, 8, 11))          # device miss path
    text = prompt_ids(V, 32, 12)
    seq = P.make_sequence(text[:16], wl["images"], T, text[16:])
    hashes = [P.hash_image(px) for px in images]
    plan = workload_plan(P, wl, L)
    req = P.ReuseRequest(seq, hashes, plan)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    setup_s = time.perf_counter() - t_setup

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
        res.last_logits()
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
    # algorithmic FLOPs of the dense prefill (all n rows at every layer, causal attention, head over n rows)
    n_all, d_, kv_, h_, hd_ = len(seq), cfg.model_dim, cfg.kv_dim, cfg.mlp_hidden, cfg.head_dim
    full_tf = (L * (2 * n_all * (3 * d_ * kv_ + kv_ * d_ + 3 * d_ * h_) + 4 * hd_ * cfg.num_heads * n_all * (n_all + 1) / 2)
               + 2 * n_all * d_ * V) / 1e12
    _, _, tf_sust0, _ = _peaks()
    full_roof = {"tflop": round(full_tf, 2), "achieved_tflops": round(full_tf / (full_ms / 1e3), 1),
                 "frac_of_sustained_bf16": round(full_tf / (full_ms / 1e3) / tf_sust0, 3)}
    # ReuseResult.kv (merged pre-RoPE K / V [L, n, kv], off the TTFT path, assembled on first access by
    # vlc_gather_rows): wall time of the access, and its algorithmic bytes (read + write K and V)
    kv_ms = []
    for _ in range(3):
        r_ = prefill_with_reuse(model, req, store)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r_.kv.device_keys()
        torch.cuda.synchronize()
        kv_ms.append((time.perf_counter() - t0) * 1e3)
        del r_
    kv_bytes = L * len(seq) * runner.dw.kv * 2 * 2 * 2
    merged_kv = {"ms": round(min(kv_ms), 3), "algorithmic_bytes": kv_bytes,
                 "GBps": round(kv_bytes / (min(kv_ms) / 1e3) / 1e9, 1),
                 "note": "first access of ReuseResult.kv: host row maps + vlc_gather_rows (not in TTFT)"}
    origin_ms = statistics.median(timed(P.ReuseRequest(seq, hashes, P.plan_static(1.0, L), images=images),
                                        P.CacheStore(), 3, 1))
    c4 = layer_aware_vs_uniform(P, model, seq, hashes, store, L, timed) if args.workload == "C3" else None
    sweep = {}
    if args.workload == "C3":
        # BASELINE's 2-5% sweep, then past it (6-10%: 257..512 recomputed rows stay one wide GEMM token tile)
        for r in (0.02, 0.03, 0.04, 0.05, 0.06, 0.08, 0.1):
            sweep[str(r)] = round(statistics.median(timed(P.ReuseRequest(seq, hashes, P.plan_static(r, L)), store,
                                                          7, 2)), 4)

    # ---- per-kernel trace (separate pass, events around each launch)
    hbm, tf_burst, tf_sust, peak_src = _peaks()
    runner.tracer = []
    ntrace = 5
    for _ in range(ntrace):
        _flush_l2(flush)
        # hold the stream on a device-side spin while the host issues the ~230 eager launches and
        # their events: the kernels then run back to back and each event pair brackets only its
        # kernel, not the host's ctypes launch latency (events still break PDL overlap, so these
        # are per-kernel durations alone, cold pipeline)
        torch.cuda._sleep(int(40e6))
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
    traffic = {}
    if args.workload == "C3":   # DRAM bytes per launch from the committed ncu --set full capture of the C3
        try:                    # layer (tools/ncu_traffic.py); other workloads: no capture, traffic null
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
    # kv_relocate against its own roofline: the prefill chain reads cached chunks straight from the
    # store (the gather + re-rotation fused into the attention) and relocates only the rows sharing
    # a chunk with recomputed ones; here the UNFUSED kernel moves every cached row of the request
    # (read K, V from the store + write rotated K, V into request rows) as one launch, alone.
    others["kv_relocate_single_launch"] = relocate_standalone(P, model, req, store, runner, flush, hbm)
    # attention against HBM as well (its K/V bytes per launch; the tensor fraction above is capped at ~0.37
    # by its 94 F/B arithmetic intensity) and the whole request against HBM: every launch's algorithmic
    # bytes (weights + activations + K/V) at the measured copy bandwidth vs the p50 TTFT
    if "attention" in agg:
        ms_k, c_k, nb_k, fl_k = agg["attention"]
        a = nb_k / (ms_k / 1e3) / 1e9
        others["attention_hbm"] = {"bound": "hbm", "achieved": round(a, 1), "peak": hbm, "unit": "GB/s",
                                   "frac": round(a / hbm, 4),
                                   "algorithmic": f"{nb_k / c_k / 1e6:.2f} MB per launch (K/V read once)"}
    req_bytes = sum(v[2] for v in agg.values()) / ntrace
    t_hbm_ms = req_bytes / (hbm * 1e9) * 1e3
    others["request_hbm"] = {"bound": "hbm", "algorithmic_gb": round(req_bytes / 1e9, 3),
                             "t_hbm_ms": round(t_hbm_ms, 3), "ttft_ms": round(p50, 4),
                             "frac": round(t_hbm_ms / p50, 4), "peak": hbm, "unit": "GB/s"}
    if args.trace:
        with open(args.trace, "w") as fh:
            json.dump({"kernels": kernels, "agg": {k: v for k, v in agg.items()}}, fh, indent=1)

    # ---- CPU leg: the reference at full depth on the SAME weights and stored KV, and parity of the
    # benchmarked request against it
    parity = cpu = None
    if cpu_leg:
        try:
            parity, cpu = cpu_leg_run(P, model, store, hashes, text, wl, plan, req, export, args.cpu_reps)
        except Exception as exc:  # never hide it: report in the line
            parity = {"error": repr(exc)}
    del export

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
                           "plan_ratios_first_last": [plan.ratios[0], plan.ratios[-1]],
                           "mean_ratio": round(P.mean_ratio(plan), 4),
                           "l2": "flushed between steps (512 MiB write); weights >> L2",
                           "parallelism": (f"head-parallel attention over {world} GPUs (one NCCL all-reduce "
                                           f"per layer)" if head_par else
                                           f"replica per GPU x{world} (independent requests, no collective)")},
                "e2e": {"value": round(e2e_p50, 4), "unit": "ms", "h2d_bytes_per_step": bytes_h2d,
                        "d2h_bytes_per_step": V * 4,
                        "note": "wall clock: prefill_with_reuse() entry -> last-row logits on host"},
                "roofline": roof, "roofline_other": others, "kernels": kernels,
                "cpu_baseline": cpu, "gpu_launches": launches, "clocks": clocks,
                "full_prefill_ms": round(full_ms, 3), "full_prefill_roofline": full_roof, "merged_kv": merged_kv,
                "origin_ms": round(origin_ms, 3),
                "speedup_vs_full_prefill": round(full_ms / p50, 2), "speedup_vs_origin": round(origin_ms / p50, 2),
                "sweep_p50_ms": sweep, "layer_aware_vs_uniform": c4, "parity_vs_cpu": parity,
                "prefill_tokens_per_s": round((1 if head_par else world) * n_tok / (p50 / 1e3), 1),
                "timed_region_s": round(region_s, 3), "setup_s": round(setup_s, 1)}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def relocate_standalone(P, model, req, store, runner, flush, hbm, reps=5):
    """vlc_kv_relocate of every cached (layer, token) row of the request, timed alone (CUDA events,
    L2 flushed before each launch); algorithmic bytes = rows x kv x 2 B x 4 (K, V read + written)."""
    import torch
    from paper_2512_12977_b200 import _native as N
    from paper_2512_12977_b200.engine import _resolve
    from paper_2512_12977_b200.layout import full_relocation
    cfg, dw = model.config, model.device
    res = _resolve(model, req, store)
    descs, blocks, ptab, rows = full_relocation([res.spec], cfg.num_layers)
    if not rows:
        return None
    pool = res.kv_pool
    dd, bb, pt = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (descs, blocks, ptab))
    n, kv = res.spec.n, dw.kv
    kc = torch.empty(cfg.num_layers, n, kv, dtype=torch.bfloat16, device="cuda")
    vc = torch.empty_like(kc)
    dw.ensure_positions(n + 1)
    times = []
    for _ in range(reps + 1):
        _flush_l2(flush)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        N.call("vlc_kv_relocate", pool.k.data_ptr(), pool.v.data_ptr(), pool.P, pt.data_ptr(), kv, cfg.head_dim,
               kc.data_ptr(), vc.data_ptr(), n, dd.data_ptr(), bb.data_ptr(), len(blocks), dw.cos.data_ptr(),
               dw.sin.data_ptr(), cfg.head_dim // 2, torch.cuda.current_stream().cuda_stream)
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = statistics.median(times[1:])
    nb = rows * kv * 2 * 4
    a = nb / (ms / 1e3) / 1e9
    return {"bound": "hbm", "achieved": round(a, 1), "peak": hbm, "unit": "GB/s", "frac": round(a / hbm, 4),
            "us": round(ms * 1e3, 1), "algorithmic": f"{nb / 1e6:.1f} MB (all layers; K+V read + write)",
            "note": "unfused kernel, measured alone; the chain reads these rows in the attention instead"}


def cpu_leg_run(P, model, store, hashes, text, wl, plan, req, export, reps):
    """cpu_baseline + parity_vs_cpu: the reference's prefill_with_reuse (baseline/_ref; the oracle
    port without it) at full depth on the device's own weights (bf16 values) and stored KV, timed
    on all host cores; the device result of the same request compared with it (north_star bars)."""
    cfg = model.config
    kw = dict(CONFIGS[wl["cfg"]], seed=0)
    enc, kv = {}, {}
    for h in hashes:
        e, k = store.get_encoder(h), store.get_kv(h)
        enc[h.hex] = np.ascontiguousarray(e.embeddings, dtype=np.float32)
        kv[h.hex] = (k.keys, k.values, k.origin_position)
    host = HostReuse(kw, export, text, [h.hex for h in hashes], enc, kv, plan.ratios, fingerprint=model.fingerprint)
    times, out = [], None
    for _ in range(max(1, reps)):
        dt, out = host.run()
        times.append(dt * 1e3)
    res = P.prefill_with_reuse(model, req, store)
    lg = res.logits
    num = den = 0.0
    keys, vals = res.kv.keys, res.kv.values
    for i in range(cfg.num_layers):     # rel_err over [L, n, kv], a layer at a time
        for a, e in ((keys[i], out["keys"][i]), (vals[i], out["values"][i])):
            num = max(num, float(np.max(np.abs(a.astype(np.float64) - e))))
            den = max(den, float(np.max(np.abs(e))))
    kv_err = num / max(den, 1e-6)
    ref_lg = out["logits"]
    parity = {"config": f"{wl['cfg']} (the benchmarked request: full depth, plan {plan.ratios[0]}..{plan.ratios[-1]})",
              "cpu_impl": host.kind,
              "rel_err": float(np.max(np.abs(lg.astype(np.float64) - ref_lg)) / max(1e-6, float(np.max(np.abs(ref_lg))))),
              "max_abs": float(np.max(np.abs(lg - ref_lg))), "kv_rel_err": kv_err,
              "top1_last_row_equal": bool(np.argmax(lg[-1]) == np.argmax(ref_lg[-1])),
              "rows_bit_exact": bool(np.array_equal(res.positions, out["rows"])),
              "counts_bit_exact": list(res.metrics.computed_per_layer) == list(out["counts"]),
              "hit_miss_equal": (res.metrics.encoder_misses, res.metrics.fallback_images) ==
                                (out["misses"], out["fallbacks"]),
              "tolerance": "rel_err <= 2e-2 (logits and merged K/V), top-1 equal, rows/counts bit-exact"}
    parity["pass"] = bool(parity["rel_err"] <= 2e-2 and kv_err <= 2e-2 and parity["top1_last_row_equal"]
                          and parity["rows_bit_exact"] and parity["counts_bit_exact"] and parity["hit_miss_equal"])
    cores = cpu_cores()
    cpu = {"value": round(statistics.median(times), 2), "unit": "ms", "cores": cores, "kind": host.kind,
           "sample": f"{'kvreuse.prefill_with_reuse (baseline/_ref)' if host.kind == 'reference' else 'oracle port'}"
                     f" of the benchmarked request at full depth ({cfg.num_layers}/{cfg.num_layers} layers) on the "
                     f"device's weights and stored KV; median of {len(times)}; numpy/OpenBLAS on {cores} threads",
           "reps_ms": [round(t, 1) for t in times]}
    return parity, cpu


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


def monotone_fit(table, P):
    """Denoised copy of a sensitivity table: per layer S_i(r) = S_i(0) - A_i (1 - exp(-r / tau)), A_i >= 1e-9
    by least squares on the profiled cells (one tau for all layers, picked from a small grid).  Gains are
    then strictly positive, so the greedy allocator (planner.py:61-102) spends the whole budget and ranks
    the layers by their fitted sensitivity."""
    grid = np.asarray(table.grid)
    d = table.baseline - np.asarray(table.scores)                     # [L, G] measured gains
    best = None
    for tau in (0.01, 0.02, 0.05, 0.1, 0.2):
        f = 1.0 - np.exp(-grid / tau)
        A = np.maximum((d * f).sum(1) / (f * f).sum(), 1e-9)
        err = float(((d - A[:, None] * f) ** 2).sum())
        if best is None or err < best[0]:
            best = (err, tau, A)
    _, tau, A = best
    scores = table.baseline - A[:, None] * (1.0 - np.exp(-grid / tau))[None, :]
    return P.SensitivityTable(np.maximum(scores, 0.0), table.grid, table.baseline, table.sample_count,
                              table.model_fingerprint), tau


def layer_aware_vs_uniform(P, model, seq, hashes, store, L, timed):
    """BASELINE configs[3]: the greedy layer-wise allocation (plan_greedy, planner.py:61-102) vs uniform
    5% at the same budget (P = 0.05 * L, cli.py:222-228): TTFT and last-row logit deviation from full
    prefill on the same GPU.  The table is profiled on the device with the reference protocol
    (sensitivity.py:88-178, tools/profile_table.py -> profiles/c3_sensitivity_table.json) for this model;
    its per-sample copies give each layer's gain standard error.  On random-init weights the gains are
    at the sample-noise level and the reference greedy stops where a raise's gain is <= 0, i.e. under-spends;
    the comparison at EQUAL budget therefore also runs the greedy on the table's monotone fit
    (monotone_fit)."""
    try:
        with open(os.path.join(ROOT, "profiles", "c3_sensitivity_table.json")) as fh:
            prof = json.load(fh)
        if int(prof["model_fingerprint"]) != model.fingerprint:
            raise ValueError("table profiled for another model")
    except (OSError, ValueError, KeyError) as exc:
        return {"error": f"no device-profiled table for this model: {exc}"}
    table = P.SensitivityTable(np.asarray(prof["scores"]), tuple(prof["grid"]), float(prof["baseline"]),
                               int(prof["samples"]), model.fingerprint)
    fit, tau = monotone_fit(table, P)
    budget = P.BudgetSpec(0.05 * L)
    plans = {"uniform": P.plan_static(0.05, L), "layer_aware": P.plan_greedy(table, budget),
             "layer_aware_fit": P.plan_greedy(fit, budget)}
    full = prefill_last(P, model, P.ReuseRequest(seq, hashes, P.plan_static(1.0, L)), store)
    out = {"table": f"device-profiled, reference protocol ({prof['samples']} proxy samples, grid {prof['grid']})",
           "layers_gain_above_2se": prof.get("layers_gain_above_2se"), "fit_tau": tau}
    for name, plan in plans.items():
        req = P.ReuseRequest(seq, hashes, plan)
        last = prefill_last(P, model, req, store)
        try:
            obj = round(P.objective(table, plan), 6)
        except P.InputError:                   # a ratio off the profiled grid (uniform 5%)
            obj = None
        out[name] = {"mean_ratio": round(P.mean_ratio(plan), 4), "ratios": list(plan.ratios),
                     "objective": obj, "objective_fit": round(P.objective(fit, plan), 6) if obj is not None else None,
                     "p50_ms": round(statistics.median(timed(req, store, 7, 2)), 4),
                     "last_row_mse_vs_full": float(np.mean((last.astype(np.float64) - full) ** 2)),
                     "last_row_max_abs_vs_full": float(np.abs(last - full).max()),
                     "top1_equal_full": bool(np.argmax(last) == np.argmax(full))}
    return out


def prefill_last(P, model, req, store):
    return P.prefill_with_reuse(model, req, store).last_logits().astype(np.float64)


if __name__ == "__main__":
    main()
