"""Stage-level view of one SQP pass on the GPU in the reference's own types (qpform.py:144-397):
``KnotLinearization``, ``SchurSystem``, ``StepDirection`` and ``first_iteration_stages`` which runs the
first pass of a solve and returns what the reference's ``linearize`` -> ``form_schur`` ->
``form_preconditioner`` -> ``pcg`` -> ``recover_step`` -> ``merit_many`` chain would return at the same
point, read from the device's stage arrays.  The stair preconditioner is rebuilt on the host from the
device's Cholesky factors (the kernels never form it: pcg_kernels.cuh)."""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass

import numpy as np

from .batch import _as_settings, pack_problems
from .blocktri import BlockTriMatrix, PcgResult
from .engine import BatchEngine
from .problem import ProblemSpec
from .settings import SolverSettings


@dataclass
class KnotLinearization:
    """Expansion blocks at one knot; dynamics entries are None at the last knot (qpform.py:144-153)."""

    Q: np.ndarray
    q: np.ndarray
    A: np.ndarray | None = None
    B: np.ndarray | None = None
    e: np.ndarray | None = None
    R: np.ndarray | None = None
    r: np.ndarray | None = None


@dataclass
class SchurSystem:
    """S lam = gamma plus the pieces needed downstream (qpform.py:272-287).  theta = S.diag_blocks[1:],
    phi = S.offdiag_blocks; zeta = gamma[1:] - e."""

    S: BlockTriMatrix
    gamma: np.ndarray
    theta: np.ndarray
    phi: np.ndarray
    zeta: np.ndarray
    q_inv: np.ndarray
    r_inv: np.ndarray
    phi_inv: BlockTriMatrix | None = None


@dataclass
class StepDirection:
    """Primal step split by knot (qpform.py:362-372)."""

    dX: np.ndarray
    dU: np.ndarray

    @property
    def inf_norm(self) -> float:
        du = float(np.max(np.abs(self.dU))) if self.dU.size else 0.0
        return max(float(np.max(np.abs(self.dX))), du)


@dataclass
class StageDump:
    blocks: list            # list[KnotLinearization], N + 1 entries
    system: SchurSystem     # with phi_inv filled
    pcg: PcgResult
    direction: StepDirection
    merits: np.ndarray      # candidate merits, alpha = beta^-c
    merit0: float           # merit of (X, U) itself
    rho: float


def _unpack_lower(T, nb, n):
    out = np.zeros((nb, n, n))
    tri = T.reshape(nb, n * (n + 1) // 2)
    for i in range(n):
        for j in range(i + 1):
            out[:, i, j] = tri[:, i * (i + 1) // 2 + j]
    return out


def first_iteration_stages(problem: ProblemSpec, X, U, settings: SolverSettings | None = None) -> StageDump:
    """Run the first SQP pass of ``sqp_solve(problem, X, U, settings)`` on the GPU and return its stages."""
    st = _as_settings(settings) if settings is not None else SolverSettings()
    N, n, m = problem.horizon, problem.model.state_dim, problem.model.control_dim
    one = dataclasses.replace(st, max_sqp_iterations=1, step_tolerance=None)
    eng = BatchEngine(problem.model, 1, N, problem.timestep, one, stage_arrays=True)
    try:
        eng.solve(pack_problems([problem], [(np.asarray(X, dtype=float), np.asarray(U, dtype=float))], [st.rho_init]))
        g = {k: eng.scratch(k) for k in ("A", "B", "e", "grad", "hinv", "Sdiag", "Soff", "Linv", "gamma", "lam",
                                         "dX", "dU", "merits", "pcg_iters")}
    finally:
        eng.close()
    rho = st.rho_init
    A, B, e = g["A"].reshape(N, n, n), g["B"].reshape(N, n, m), g["e"].reshape(N, n)
    grad = g["grad"].reshape(N + 1, n + m)
    Qs = np.asarray(problem.cost.Q, dtype=float) + rho * np.eye(n)
    Qt = np.asarray(problem.cost.QN, dtype=float) + rho * np.eye(n)
    Rs = np.asarray(problem.cost.R, dtype=float) + (rho * np.eye(m) if st.regularize_r else 0.0)
    blocks = [KnotLinearization(Q=Qs, q=grad[k, :n], A=A[k], B=B[k], e=e[k], R=Rs, r=grad[k, n:]) for k in range(N)]
    blocks.append(KnotLinearization(Q=Qt, q=grad[N, :n]))
    diag, off = g["Sdiag"].reshape(N + 1, n, n), g["Soff"].reshape(N, n, n)
    gamma = g["gamma"].copy()
    q_inv = np.empty((N + 1, n, n))
    q_inv[:-1] = g["hinv"][:n * n].reshape(n, n)
    q_inv[-1] = g["hinv"][n * n:2 * n * n].reshape(n, n)
    r_inv = np.broadcast_to(g["hinv"][2 * n * n:2 * n * n + m * m].reshape(m, m), (N, m, m)).copy()
    Li = _unpack_lower(g["Linv"], N + 1, n)
    dinv = np.einsum("kli,klj->kij", Li, Li)                               # D_k^-1 = L_k^-T L_k^-1
    poff = -np.einsum("kij,kjl,klm->kim", dinv[1:], off, dinv[:-1])        # qpform.py:355-356
    system = SchurSystem(S=BlockTriMatrix(diag, off), gamma=gamma, theta=diag[1:].copy(), phi=off.copy(),
                         zeta=gamma.reshape(N + 1, n)[1:] - e, q_inv=q_inv, r_inv=r_inv,
                         phi_inv=BlockTriMatrix(dinv, poff))
    its = int(g["pcg_iters"][0])
    lam = g["lam"].copy()
    from .blocktri import densify
    res = float(np.linalg.norm(densify(system.S) @ lam - gamma))
    cap = st.pcg.iteration_cap((N + 1) * n)
    result = PcgResult(lam, its, bool(res <= st.pcg.tolerance or its < cap), res)
    C = st.line_search.num_shrinks + 1
    return StageDump(blocks, system, result, StepDirection(g["dX"].reshape(N + 1, n), g["dU"].reshape(N, m)),
                     g["merits"][:C].copy(), float(g["merits"][C]), rho)
