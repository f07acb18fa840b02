"""Synthetic iiwa14 problem generators: the single source of truth for bench.py, the parity
tests and the CPU baseline.

Draws are consumed in solve order from ``np.random.default_rng(20251007)`` so any batch is a
prefix of a larger one.  Costs are shared across the batch:
Q = diag(10 x7, 0.1 x7), R = 1e-3 I, QN = diag(100 x7, 1 x7).
"""

from __future__ import annotations

import numpy as np

from .batch import BatchSpec
from .engine import PackedBatch
from .models import Iiwa14
from .problem import CostSpec, ExternalForce, ProblemSpec
from .settings import LineSearchSettings, PcgSettings, SolverSettings

SEED = 20251007


def iiwa14_cost_weights():
    Q = np.diag(np.concatenate([np.full(7, 10.0), np.full(7, 0.1)]))
    R = 1e-3 * np.eye(7)
    QN = np.diag(np.concatenate([np.full(7, 100.0), np.full(7, 1.0)]))
    return Q, R, QN


def fixed_budget_settings(iterations: int, pcg_tolerance: float = 1e-6, pcg_max_iterations: int | None = 200):
    """Timing mode: run exactly ``iterations`` SQP iterations (step_tolerance=None, sqp.py:65-66)."""
    return SolverSettings(max_sqp_iterations=iterations,
                          pcg=PcgSettings(tolerance=pcg_tolerance, max_iterations=pcg_max_iterations),
                          line_search=LineSearchSettings(), step_tolerance=None)


def sample_force_hypotheses(center, sigma: float, M: int, seed: int) -> np.ndarray:
    """Center plus M-1 candidates at radius sigma, directions uniform on the sphere
    (mpc.sample_hypotheses, mpc.py:110-127) -> (M, dim)."""
    center = np.asarray(center, dtype=float)
    rng = np.random.default_rng(seed)
    out = [center.copy()]
    for _ in range(M - 1):
        d = rng.standard_normal(center.shape[0])
        nrm = np.linalg.norm(d)
        while nrm < 1e-12:
            d = rng.standard_normal(center.shape[0])
            nrm = np.linalg.norm(d)
        out.append(center + sigma * d / nrm)
    return np.stack(out)


def iiwa14_reach_arrays(M: int, N: int, rho_init: float = 1e-4, seed: int = SEED) -> PackedBatch:
    """Reach: q0 ~ U(-0.6, 0.6)^7 at rest, single goal state q_goal ~ U(-1, 1)^7 at rest,
    X0 = tile(x_start), U0 = 0, no external force."""
    rng = np.random.default_rng(seed)
    Q, R, QN = iiwa14_cost_weights()
    x_start = np.zeros((M, 14))
    goal = np.zeros((M, N + 1, 14))
    for b in range(M):
        x_start[b, :7] = rng.uniform(-0.6, 0.6, size=7)
        goal[b, :, :7] = rng.uniform(-1.0, 1.0, size=7)
    return PackedBatch(
        x_start=x_start, goal=goal,
        Q=np.broadcast_to(Q, (M, 14, 14)).copy(), R=np.broadcast_to(R, (M, 7, 7)).copy(),
        QN=np.broadcast_to(QN, (M, 14, 14)).copy(), force=np.zeros((M, N, 3)),
        rho_init=np.full(M, rho_init), X=np.repeat(x_start[:, None, :], N + 1, axis=1).copy(),
        U=np.zeros((M, N, 7)))


def iiwa14_track_arrays(M: int, N: int, h: float, sigma: float = 5.0, rho_init: float = 1e-4,
                        seed: int = SEED, step: int = 0) -> PackedBatch:
    """MPC tracking batch: one start state and goal window shared by all solves, which differ
    only in the assumed flange force (hypotheses at radius ``sigma`` N around zero).
    q_ref(t) = q0 + 0.4 sin(2 pi t / 4 + j pi / 7), qd_ref by forward difference
    (Figure8Reference convention, mpc.py:414-420)."""
    rng = np.random.default_rng(seed)
    Q, R, QN = iiwa14_cost_weights()
    q0 = rng.uniform(-0.6, 0.6, size=7)
    t = (step + np.arange(N + 2)) * h
    phase = np.arange(7) * np.pi / 7.0
    q = q0[None, :] + 0.4 * np.sin(2.0 * np.pi * t[:, None] / 4.0 + phase[None, :])
    qd = np.zeros_like(q)
    qd[:-1] = (q[1:] - q[:-1]) / h
    qd[-1] = qd[-2]
    window = np.concatenate([q, qd], axis=1)[:N + 1]
    x_start = np.concatenate([q0, np.zeros(7)])
    forces = sample_force_hypotheses(np.zeros(3), sigma, M, seed=seed + 1)
    return PackedBatch(
        x_start=np.broadcast_to(x_start, (M, 14)).copy(),
        goal=np.broadcast_to(window, (M, N + 1, 14)).copy(),
        Q=np.broadcast_to(Q, (M, 14, 14)).copy(), R=np.broadcast_to(R, (M, 7, 7)).copy(),
        QN=np.broadcast_to(QN, (M, 14, 14)).copy(),
        force=np.broadcast_to(forces[:, None, :], (M, N, 3)).copy(),
        rho_init=np.full(M, rho_init),
        X=np.broadcast_to(x_start, (M, N + 1, 14)).copy(), U=np.zeros((M, N, 7)))


def arrays_to_spec(batch: PackedBatch, h: float, settings: SolverSettings, model=None) -> BatchSpec:
    """The same batch as reference-typed objects (for batch_solve and for the CPU reference)."""
    model = model if model is not None else Iiwa14()
    problems, inits = [], []
    for b in range(batch.size):
        cost = CostSpec(batch.Q[b], batch.R[b], batch.QN[b], batch.goal[b])
        force = batch.force[b]
        if np.all(force == force[0]):
            ext = ExternalForce.constant(force[0])
        else:
            raise ValueError("arrays_to_spec supports constant forces only")
        problems.append(ProblemSpec(model, cost, batch.X.shape[1] - 1, h, batch.x_start[b], ext))
        inits.append((batch.X[b].copy(), batch.U[b].copy()))
    return BatchSpec.with_rho_inits(problems, inits, settings, batch.rho_init)
