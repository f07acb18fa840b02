"""Host helpers of the MPC caller around the batched solve: warm-start shift, nested rho grid,
disturbance hypotheses, best-of-batch selection (reference mpc.py:61-147, 283-298).  These are the
steps immediately before and after `batch_solve` in `_MpcEngine.advance` (mpc.py:240-330); the
solve itself and the device-side shift (`BatchEngine.shift_warm_start`) live behind the C ABI."""

from __future__ import annotations

import math

import numpy as np

from .problem import ExternalForce
from .results import SqpResult


def rho_grid(M: int, lo: float = 1e-8, hi: float = 1e1) -> np.ndarray:
    """First M values of the nested log-spaced refinement of [lo, hi] (mpc.py:61-78): midpoint,
    endpoints, then odd dyadic fractions level by level, so grids for growing M are prefixes."""
    if M < 1:
        raise ValueError("M must be >= 1")
    fractions = [0.5, 0.0, 1.0]
    level = 4
    while len(fractions) < M:
        fractions.extend(i / level for i in range(1, level, 2))
        level *= 2
    lo_e, hi_e = math.log10(lo), math.log10(hi)
    return 10.0 ** (lo_e + (hi_e - lo_e) * np.asarray(fractions[:M]))


def shift_warm_start(prev: SqpResult) -> tuple[np.ndarray, np.ndarray]:
    """Shift the previous solution left one knot, duplicating the tail (mpc.py:85-89)."""
    return (np.concatenate([prev.X[1:], prev.X[-1:]], axis=0),
            np.concatenate([prev.U[1:], prev.U[-1:]], axis=0))


def sample_hypotheses(center, sigma: float, M: int, seed: int) -> list[ExternalForce]:
    """Center plus M-1 candidates at Euclidean distance sigma, directions uniform on the sphere,
    deterministic in the seed (mpc.py:110-127)."""
    from .workloads import sample_force_hypotheses
    if M < 1:
        raise ValueError("M must be >= 1")
    if sigma < 0:
        raise ValueError("sigma must be >= 0")
    center = center.value if isinstance(center, ExternalForce) else np.asarray(center, dtype=float)
    return [ExternalForce.constant(f) for f in sample_force_hypotheses(center, sigma, M, seed)]


def best_of_batch(results) -> int:
    """Index of the solve with the lowest final merit, first minimum on ties, failed slots
    skipped (mpc.py:283-298)."""
    best, best_merit = -1, math.inf
    for i, res in enumerate(results):
        if res is None:
            continue
        if best < 0 or res.final_merit < best_merit:
            best, best_merit = i, res.final_merit
    if best < 0:
        raise ValueError("every solve of the batch failed")
    return best
