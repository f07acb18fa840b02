"""Result types: mirror of IterationRecord / SqpResult (sqp.py:81-108) and BatchResult
(batch.py:78-89)."""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass
class IterationRecord:
    """One SQP iteration; ``alpha`` is None only on the record of a tolerance exit."""

    iteration: int
    merit: float
    constraint_l1: float
    alpha: float | None
    rho: float
    pcg_iterations: int
    accepted: bool
    step_inf_norm: float


@dataclass
class SqpResult:
    X: np.ndarray
    U: np.ndarray
    trace: list[IterationRecord]
    converged: bool

    @property
    def final_merit(self) -> float:
        return self.trace[-1].merit if self.trace else math.nan

    @property
    def iterations(self) -> int:
        return len(self.trace)


@dataclass
class BatchResult:
    """Per-problem results in input order; ``results[i]`` is None exactly when ``errors[i]``
    holds the failure message of that slot.  ``solve_times`` cannot be separated per solve on
    a GPU: every entry is device_time / M (device time measured with CUDA events)."""

    results: list[SqpResult | None]
    errors: list[str | None]
    wall_time: float
    solve_times: list[float]
    device_time: float = 0.0

    @property
    def ok(self) -> bool:
        return all(e is None for e in self.errors)
