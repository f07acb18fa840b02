"""Reference-named merit / line-search operators on the GPU (sqp.py:111-201): ``constraint_l1``, ``merit``,
``merit_many``, ``line_search`` and ``adapt_rho`` with the reference's signatures.  The merit values come
from the same line-search kernel the solve uses (gato_merit_candidates); ``line_search`` takes its argmin on
the host exactly as sqp.py:189-195 does (first minimum, strict decrease); ``adapt_rho`` is scalar
bookkeeping."""

from __future__ import annotations


import numpy as np

from .batch import _engine_for, pack_problems
from .problem import ProblemSpec
from .settings import LineSearchSettings, SolverSettings


def _engine(problem: ProblemSpec, copies: int, ls: LineSearchSettings):
    st = SolverSettings(max_sqp_iterations=1, step_tolerance=None, line_search=ls)
    return _engine_for(problem.model, copies, problem.horizon, problem.timestep, st, None), st


def _evaluate(problem: ProblemSpec, Xs, Us, ls: LineSearchSettings, dX=None, dU=None):
    Xs, Us = np.asarray(Xs, dtype=float), np.asarray(Us, dtype=float)
    C = Xs.shape[0]
    eng, st = _engine(problem, C, ls)
    eng.upload(pack_problems([problem] * C, list(zip(Xs, Us)), [st.rho_init] * C))
    return eng.merit_candidates(dX, dU)


def merit_many(problem: ProblemSpec, Xs, Us, mu: float) -> np.ndarray:
    """Merit of C candidate trajectories, shapes (C, N+1, n), (C, N, m); non-finite candidates score +inf
    (sqp.py:132-166)."""
    merits, _ = _evaluate(problem, Xs, Us, LineSearchSettings(mu=mu))
    return merits[:, -1].copy()


def merit(problem: ProblemSpec, X, U, mu: float) -> float:
    """L1 merit: cost plus mu times the constraint violation, +inf for non-finite trajectories
    (sqp.py:118-129)."""
    return float(merit_many(problem, np.asarray(X, dtype=float)[None], np.asarray(U, dtype=float)[None], mu)[0])


def constraint_l1(problem: ProblemSpec, X, U) -> float:
    """L1 norm of all dynamics defects plus the initial-state defect (sqp.py:111-115)."""
    _, viols = _evaluate(problem, np.asarray(X, dtype=float)[None], np.asarray(U, dtype=float)[None],
                         LineSearchSettings())
    return float(viols[0, -1])


def line_search(problem: ProblemSpec, X, U, dX, dU, settings: LineSearchSettings,
                current_merit: float | None = None) -> tuple[float, float, bool]:
    """(alpha*, merit at alpha*, accepted) over the geometric candidate set (sqp.py:169-195): every
    candidate scored on the device in one launch, first minimum wins ties, strict decrease accepts."""
    X, U = np.asarray(X, dtype=float), np.asarray(U, dtype=float)
    merits, _ = _evaluate(problem, X[None], U[None], settings, np.asarray(dX, dtype=float)[None],
                          np.asarray(dU, dtype=float)[None])
    values = merits[0, :-1]
    if current_merit is None:
        current_merit = float(merits[0, -1])
    best = int(np.argmin(values))
    return float(settings.candidates()[best]), float(values[best]), bool(values[best] < current_merit)


def adapt_rho(rho: float, accepted: bool, settings: SolverSettings) -> float:
    """rho / factor after an accepted step, rho * factor otherwise, clamped (sqp.py:198-201)."""
    rho = rho / settings.rho_factor if accepted else rho * settings.rho_factor
    return float(min(max(rho, settings.rho_min), settings.rho_max))


__all__ = ["adapt_rho", "constraint_l1", "line_search", "merit", "merit_many"]
