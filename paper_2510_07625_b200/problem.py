"""Problem description types: host-side mirror of the reference's ExternalForce
(dynamics.py:33-69), CostSpec (qpform.py:45-78) and ProblemSpec (qpform.py:82-140).

Validation happens eagerly at construction, with the reference's exception types and
conditions, so a malformed problem never reaches the device.  Nothing here evaluates
dynamics: rollouts and defects are device work.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from .errors import DimensionError


@dataclass(frozen=True)
class ExternalForce:
    """A force in a model's generalized-force channel (dynamics.py:33-69): constant
    ``value``, or ``profile(t)`` with ``value`` fixing the dimension."""

    value: np.ndarray
    profile: Callable[[float], np.ndarray] | None = None

    @classmethod
    def constant(cls, value) -> "ExternalForce":
        return cls(np.atleast_1d(np.asarray(value, dtype=float)))

    @classmethod
    def zero(cls, dim: int) -> "ExternalForce":
        return cls(np.zeros(dim))

    @classmethod
    def time_varying(cls, profile, dim: int) -> "ExternalForce":
        return cls(np.zeros(dim), profile)

    @property
    def dim(self) -> int:
        return self.value.shape[0]

    @property
    def is_constant(self) -> bool:
        return self.profile is None

    def at(self, t: float) -> np.ndarray:
        if self.profile is None:
            return self.value
        return np.asarray(self.profile(t), dtype=float)


def _require_symmetric(mat: np.ndarray, label: str):
    if mat.ndim != 2 or mat.shape[0] != mat.shape[1]:
        raise DimensionError(f"{label} must be square, got {mat.shape}")
    if not np.allclose(mat, mat.T, atol=1e-10):
        raise ValueError(f"{label} must be symmetric")


@dataclass
class CostSpec:
    """Quadratic tracking cost (qpform.py:45-78): dense symmetric Q, R, QN and a goal that is
    one state (n,) or a reference sequence (N+1, n)."""

    Q: np.ndarray
    R: np.ndarray
    QN: np.ndarray
    goal: np.ndarray

    def __post_init__(self):
        self.Q = np.asarray(self.Q, dtype=float)
        self.R = np.asarray(self.R, dtype=float)
        self.QN = np.asarray(self.QN, dtype=float)
        self.goal = np.asarray(self.goal, dtype=float)
        _require_symmetric(self.Q, "Q")
        _require_symmetric(self.R, "R")
        _require_symmetric(self.QN, "QN")

    def goal_at(self, k: int) -> np.ndarray:
        return self.goal if self.goal.ndim == 1 else self.goal[k]


@dataclass
class ProblemSpec:
    """One trajectory-optimisation problem over an N-step horizon (qpform.py:82-123)."""

    model: object
    cost: CostSpec
    horizon: int
    timestep: float
    x_start: np.ndarray
    force: ExternalForce | None = None

    def __post_init__(self):
        if self.horizon < 1:
            raise ValueError("horizon must be >= 1")
        if self.timestep <= 0:
            raise ValueError("timestep must be positive")
        self.x_start = np.asarray(self.x_start, dtype=float)
        n, m = self.model.state_dim, self.model.control_dim
        if self.x_start.shape != (n,):
            raise DimensionError(f"x_start shape {self.x_start.shape} != ({n},)")
        if self.cost.Q.shape != (n, n) or self.cost.QN.shape != (n, n):
            raise DimensionError("cost state weights do not match the model dimension")
        if self.cost.R.shape != (m, m):
            raise DimensionError("cost control weight does not match the model")
        if self.cost.goal.ndim == 2 and self.cost.goal.shape != (self.horizon + 1, n):
            raise DimensionError(f"per-knot goal must have shape ({self.horizon + 1}, {n})")
        if self.force is None:
            self.force = ExternalForce.zero(self.model.force_dim)

    def force_at_knot(self, k: int) -> np.ndarray:
        return self.force.at(k * self.timestep)

    def force_matrix(self) -> np.ndarray:
        """Assumed force at the start time k*h of every stage knot, (N, force_dim)
        (qpform.py:113-123)."""
        if self.force.is_constant:
            return np.broadcast_to(self.force.value, (self.horizon, self.force.dim))
        return np.stack([self.force_at_knot(k) for k in range(self.horizon)])
