"""Solver settings: mirror of PcgSettings (blocktri.py:62-81), LineSearchSettings
(sqp.py:32-52) and SolverSettings (sqp.py:56-77), same defaults and validation."""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class PcgSettings:
    tolerance: float = 1e-8
    max_iterations: int | None = None

    def __post_init__(self):
        if self.tolerance < 0:
            raise ValueError("tolerance must be >= 0")
        if self.max_iterations is not None and self.max_iterations < 1:
            raise ValueError("max_iterations must be >= 1")

    def iteration_cap(self, system_size: int) -> int:
        return self.max_iterations if self.max_iterations is not None else 10 * system_size


@dataclass(frozen=True)
class LineSearchSettings:
    mu: float = 10.0
    beta: float = 2.0
    num_shrinks: int = 8

    def __post_init__(self):
        if self.mu <= 0:
            raise ValueError("mu must be positive")
        if self.beta <= 1:
            raise ValueError("beta must be > 1")
        if self.num_shrinks < 1:
            raise ValueError("num_shrinks must be >= 1")

    def candidates(self) -> np.ndarray:
        return self.beta ** -np.arange(self.num_shrinks + 1, dtype=float)


@dataclass(frozen=True)
class SolverSettings:
    max_sqp_iterations: int = 50
    pcg: PcgSettings = field(default_factory=lambda: PcgSettings(tolerance=1e-8))
    line_search: LineSearchSettings = field(default_factory=LineSearchSettings)
    rho_init: float = 1e-4
    rho_min: float = 1e-8
    rho_max: float = 1e1
    rho_factor: float = 5.0
    step_tolerance: float | None = 1e-6      # None: run the whole iteration budget
    feasibility_tolerance: float = 1e-6
    regularize_r: bool = True
    pcg_retry_limit: int = 3

    def __post_init__(self):
        if not (self.rho_min <= self.rho_init <= self.rho_max):
            raise ValueError("rho_init must lie in [rho_min, rho_max]")
        if self.rho_factor <= 1:
            raise ValueError("rho_factor must be > 1")
        if self.max_sqp_iterations < 1:
            raise ValueError("max_sqp_iterations must be >= 1")
