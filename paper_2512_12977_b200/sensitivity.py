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
