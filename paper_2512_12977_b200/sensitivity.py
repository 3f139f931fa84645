"""Layer sensitivity table consumed by the allocator (reference: sensitivity.py:42-81).

Only the table type and its lookup are on the hot path; the offline profiling
protocol (sensitivity.py:88-178) is out of scope for this drop-in.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .exceptions import InputError
from .plans import GRID_MAX, GRID_STEP


@dataclass
class SensitivityTable:
    scores: np.ndarray        # [L, len(grid)] mean logit MSE per (layer, ratio)
    grid: tuple[float, ...]
    baseline: float           # score with no recomputation anywhere
    sample_count: int
    model_fingerprint: int

    def __post_init__(self):
        self.scores = np.asarray(self.scores, dtype=np.float64)
        if self.scores.ndim != 2 or self.scores.shape[1] != len(self.grid):
            raise InputError("scores shape does not match grid")
        if (self.scores < 0).any() or self.baseline < 0:
            raise InputError("sensitivity scores must be non-negative")
        if list(self.grid) != sorted(set(self.grid)):
            raise InputError("grid must be strictly increasing")
        top = round(GRID_MAX / GRID_STEP)
        for r in self.grid:
            k = round(r / GRID_STEP)
            if not (1 <= k <= top and abs(r - k * GRID_STEP) <= 1e-9):
                raise InputError(f"grid ratio {r} off the planner grid")

    @property
    def num_layers(self) -> int:
        return int(self.scores.shape[0])

    def score(self, layer: int, ratio: float) -> float:
        """S(layer, ratio); ratio 0 is the no-recompute baseline."""
        if ratio == 0.0:
            return float(self.baseline)
        for j, g in enumerate(self.grid):
            if abs(g - ratio) <= 1e-9:
                return float(self.scores[layer, j])
        raise InputError(f"ratio {ratio} was not measured (grid {self.grid})")

    def check_fingerprint(self, model) -> str | None:
        if self.model_fingerprint != model.fingerprint:
            return (f"table was profiled with model {self.model_fingerprint:#x}, "
                    f"live model is {model.fingerprint:#x}")
        return None


# ---------------------------------------------------------------- profiling on the device
# (sensitivity.py:20-35, 88-178): every forward / decode runs through the GPU chain; the
# per-cell work is L * |grid| + 1 teacher-forced dense passes per sample.

@dataclass
class ProxySample:
    image: np.ndarray
    original_prompt: list
    neutral_prompt: list

    def validate(self, require_distinct: bool = False) -> None:
        if not len(self.original_prompt) or not len(self.neutral_prompt):
            raise InputError("prompts must be non-empty")
        if require_distinct and list(self.original_prompt) == list(self.neutral_prompt):
            raise InputError("neutral prompt must differ from the original")


def build_mismatched_kv(model, sample: ProxySample):
    """Full prefill with the neutral prompt; the image's pre-RoPE KV (sensitivity.py:88-99)."""
    from .engine import encode_images_device, prefill_full
    from .sequence import make_sequence
    from .store import KVCacheEntry, hash_image
    sample.validate()
    cfg = model.config
    emb = encode_images_device(model, [sample.image])
    seq = make_sequence(list(sample.neutral_prompt), 1, cfg.tokens_per_image)
    _, kv = prefill_full(model, seq, [emb])
    seg = seq.image_segments[0]
    sl = slice(seg.start, seg.start + seg.length)
    return KVCacheEntry(hash_image(sample.image), kv.device_keys()[:, sl].clone(),
                        kv.device_values()[:, sl].clone(), origin_position=seg.start,
                        model_fingerprint=model.fingerprint)


def baseline_decode(model, sample: ProxySample, max_new: int):
    """Greedy continuation with same-context KV (sensitivity.py:102-114): (logits [max_new, V], ids)."""
    from .engine import decode_with_merged_kv, encode_images_device, prefill_full
    from .sequence import make_sequence
    if max_new < 1:
        raise InputError("max_new must be >= 1")
    cfg = model.config
    emb = encode_images_device(model, [sample.image])
    seq = make_sequence(list(sample.original_prompt), 1, cfg.tokens_per_image)
    logits, kv = prefill_full(model, seq, [emb])
    dec = decode_with_merged_kv(model, kv, max_new=max_new, initial_logits=logits[-1])
    return dec.step_logits, dec.ids


def reuse_logits(model, sample: ProxySample, mismatched, layer: int, ratio: float, baseline_ids) -> np.ndarray:
    """Teacher-forced logits with the mismatched KV injected at every layer except the first
    floor(r*T) image tokens of the probed layer (sensitivity.py:117-147)."""
    import torch
    from .engine import encode_images_device, forward_injected
    from .plans import recompute_count
    from .sequence import make_sequence
    cfg = model.config
    if not 0 <= layer < cfg.num_layers:
        raise InputError(f"layer {layer} out of range")
    if not 0.0 <= ratio <= 1.0:
        raise InputError("ratio must lie in [0, 1]")
    emb = encode_images_device(model, [sample.image])
    seq = make_sequence(list(sample.original_prompt), 1, cfg.tokens_per_image, suffix=list(baseline_ids))
    seg = seq.image_segments[0]
    n, L = len(seq), cfg.num_layers
    ik = torch.zeros(L, n, cfg.kv_dim, dtype=torch.bfloat16, device="cuda")
    iv = torch.zeros_like(ik)
    sl = slice(seg.start, seg.start + seg.length)
    keys = mismatched.keys if isinstance(mismatched.keys, torch.Tensor) else torch.from_numpy(mismatched.keys)
    vals = mismatched.values if isinstance(mismatched.values, torch.Tensor) else torch.from_numpy(mismatched.values)
    ik[:, sl], iv[:, sl] = keys.to("cuda", torch.bfloat16), vals.to("cuda", torch.bfloat16)
    use_cached = np.zeros((L, n), dtype=bool)
    use_cached[:, sl] = True
    use_cached[layer, seg.start:seg.start + recompute_count(ratio, seg.length)] = False
    logits, _ = forward_injected(model, seq, [emb], ik, iv, use_cached)
    first = seg.start + seg.length - 1
    return logits[first:first + len(baseline_ids)]


def logit_mse(a, b) -> float:
    if np.shape(a) != np.shape(b):
        raise InputError(f"logit shapes differ: {np.shape(a)} vs {np.shape(b)}")
    return float(np.mean(np.square(np.asarray(a, np.float64) - np.asarray(b, np.float64))))


def profile(model, dataset, grid, max_new: int = 8) -> SensitivityTable:
    """Mean logit MSE over the dataset for every (layer, grid ratio) cell (sensitivity.py:156-178)."""
    if not dataset:
        raise InputError("dataset must contain at least one sample")
    grid = tuple(sorted(float(g) for g in grid))
    L = model.config.num_layers
    totals = np.zeros((L, len(grid)), dtype=np.float64)
    base = 0.0
    for sample in dataset:
        sample.validate()
        mismatched = build_mismatched_kv(model, sample)
        z_orig, ids = baseline_decode(model, sample, max_new)
        base += logit_mse(z_orig, reuse_logits(model, sample, mismatched, 0, 0.0, ids))
        for i in range(L):
            for j, r in enumerate(grid):
                totals[i, j] += logit_mse(z_orig, reuse_logits(model, sample, mismatched, i, r, ids))
    return SensitivityTable(totals / len(dataset), grid, base / len(dataset), len(dataset), model.fingerprint)
