"""ORACLE (test infrastructure, never shipped on the product path).

CPU restatement, in numpy, of the reference package's batched SQP solve
(`trajbatch.batch_solve` -> `sqp_solve`), i.e. the hot path of SURVEY.md section 8.
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may import this.

The reference is pure Python and imports in the build container, so this restatement is
PINNED: tests/golden/make_golden.py runs the unmodified reference on seeded problems and
stores its stage-by-stage outputs under tests/golden/*.npz; tests/test_oracle_golden.py
checks every function here against those vectors, and tests/test_oracle_vs_reference.py
compares against the live reference whenever /root/reference is present.

Each function cites the reference lines it restates (paths relative to
/root/reference/pkg/src/trajbatch/).  The code is organised differently from the reference
(stacked arrays instead of per-knot objects, a flat state machine instead of exceptions for
the PCG retry) but performs the same floating-point operations in the same order wherever
the order is observable.

The iiwa14 model (not in the reference) lives in oracle/iiwa14_np.py.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field, replace

import numpy as np
import scipy.linalg


# --------------------------------------------------------------------------------------
# settings (sqp.py:32-77, blocktri.py:62-81)
# --------------------------------------------------------------------------------------

@dataclass(frozen=True)
class Settings:
    max_sqp_iterations: int = 50
    pcg_tolerance: float = 1e-8
    pcg_max_iterations: int | None = None
    mu: float = 10.0
    beta: float = 2.0
    num_shrinks: int = 8
    rho_init: float = 1e-4
    rho_min: float = 1e-8
    rho_max: float = 1e1
    rho_factor: float = 5.0
    step_tolerance: float | None = 1e-6
    feasibility_tolerance: float = 1e-6
    regularize_r: bool = True
    pcg_retry_limit: int = 3

    def step_lengths(self) -> np.ndarray:
        # sqp.py:51-52
        return self.beta ** -np.arange(self.num_shrinks + 1, dtype=float)

    def pcg_cap(self, unknowns: int) -> int:
        # blocktri.py:78-81
        return self.pcg_max_iterations if self.pcg_max_iterations is not None else 10 * unknowns


class OracleFactorizationError(RuntimeError):
    """errors.py:12-21"""

    def __init__(self, message, knot=None):
        super().__init__(message)
        self.knot = knot


class OraclePcgBreakdown(RuntimeError):
    """errors.py:24-32"""

    def __init__(self, message, iteration):
        super().__init__(message)
        self.iteration = iteration


# --------------------------------------------------------------------------------------
# analytic models of the reference (dynamics.py:145-703), restated
# --------------------------------------------------------------------------------------

class PointMasses:
    """dynamics.py:145-187 (DoubleIntegrator)."""

    name = "double_integrator"

    def __init__(self, dims=1, mass=1.0):
        self.dims, self.mass = dims, mass
        self.state_dim, self.control_dim, self.force_dim = 2 * dims, dims, dims

    def deriv_many(self, X, U, F):
        return np.concatenate([X[:, self.dims:], U + F / self.mass], axis=1)

    def deriv_jacobians_many(self, X, U, F):
        d, B = self.dims, X.shape[0]
        fx = np.zeros((B, 2 * d, 2 * d))
        fu = np.zeros((B, 2 * d, d))
        idx = np.arange(d)
        fx[:, idx, d + idx] = 1.0
        fu[:, d + idx, idx] = 1.0
        return fx, fu


class DampedPendulum:
    """dynamics.py:190-252 (Pendulum)."""

    name = "pendulum"
    state_dim, control_dim, force_dim = 2, 1, 1

    def __init__(self, mass=1.0, length=1.0, gravity=9.81, damping=0.1):
        self.mass, self.length, self.gravity, self.damping = mass, length, gravity, damping
        self.inertia = mass * length ** 2

    def deriv_many(self, X, U, F):
        th, om = X[:, 0], X[:, 1]
        acc = (U[:, 0] + F[:, 0] - self.mass * self.gravity * self.length * np.sin(th)
               - self.damping * om) / self.inertia
        return np.stack([om, acc], axis=1)

    def deriv_jacobians_many(self, X, U, F):
        B = X.shape[0]
        fx = np.zeros((B, 2, 2))
        fu = np.zeros((B, 2, 1))
        fx[:, 0, 1] = 1.0
        fx[:, 1, 0] = -self.gravity / self.length * np.cos(X[:, 0])
        fx[:, 1, 1] = -self.damping / self.inertia
        fu[:, 1, 0] = 1.0 / self.inertia
        return fx, fu


def _sym2(a, b, c):
    """Stack of symmetric 2x2 matrices [[a, b], [b, c]]."""
    M = np.empty(a.shape + (2, 2))
    M[..., 0, 0], M[..., 0, 1], M[..., 1, 0], M[..., 1, 1] = a, b, b, c
    return M


class HangingCartpole:
    """dynamics.py:255-384 (Cartpole): state [p, theta, pdot, thetadot], theta=0 down."""

    name = "cartpole"
    state_dim, control_dim, force_dim = 4, 1, 2

    def __init__(self, cart_mass=1.0, pole_mass=0.2, pole_length=0.5, gravity=9.81):
        self.cart_mass, self.pole_mass = cart_mass, pole_mass
        self.pole_length, self.gravity = pole_length, gravity

    def _mass_rhs(self, X, U, F):
        mp, L = self.pole_mass, self.pole_length
        th, thd = X[:, 1], X[:, 3]
        s, c = np.sin(th), np.cos(th)
        M = _sym2(np.full_like(th, self.cart_mass + mp), mp * L * c, np.full_like(th, mp * L ** 2))
        rhs = np.stack([U[:, 0] + F[:, 0] + mp * L * s * thd ** 2,
                        F[:, 1] - mp * self.gravity * L * s], axis=1)
        return M, rhs, s, c

    def deriv_many(self, X, U, F):
        M, rhs, _, _ = self._mass_rhs(X, U, F)
        qdd = np.linalg.solve(M, rhs[:, :, None])[:, :, 0]
        return np.concatenate([X[:, 2:], qdd], axis=1)

    def deriv_jacobians_many(self, X, U, F):
        mp, L = self.pole_mass, self.pole_length
        B = X.shape[0]
        thd = X[:, 3]
        M, rhs, s, c = self._mass_rhs(X, U, F)
        Minv = np.linalg.inv(M)
        qdd = np.einsum("bij,bj->bi", Minv, rhs)
        zero = np.zeros(B)
        dM = _sym2(zero, -mp * L * s, zero)
        drhs_th = np.stack([mp * L * c * thd ** 2, -mp * self.gravity * L * c], axis=1)
        drhs_thd = np.stack([2.0 * mp * L * s * thd, zero], axis=1)
        col_th = np.einsum("bij,bj->bi", Minv, drhs_th - np.einsum("bij,bj->bi", dM, qdd))
        col_thd = np.einsum("bij,bj->bi", Minv, drhs_thd)
        fx = np.zeros((B, 4, 4))
        fx[:, 0, 2] = fx[:, 1, 3] = 1.0
        fx[:, 2:, 1] = col_th
        fx[:, 2:, 3] = col_thd
        fu = np.zeros((B, 4, 1))
        fu[:, 2:, 0] = Minv[:, :, 0]
        return fx, fu


class PlanarTwoLink:
    """dynamics.py:387-703 (TwoLinkArm): planar 2R arm, tip-force channel J(q)^T f."""

    name = "two_link_arm"
    state_dim, control_dim, force_dim = 4, 2, 2

    def __init__(self, m1=1.0, m2=1.0, l1=0.5, l2=0.5, gravity=0.0, joint_damping=0.05):
        self.m1, self.m2, self.l1, self.l2 = m1, m2, l1, l2
        self.gravity, self.joint_damping = gravity, joint_damping
        lc1, lc2 = 0.5 * l1, 0.5 * l2
        I1, I2 = m1 * l1 ** 2 / 12.0, m2 * l2 ** 2 / 12.0
        self.lc1, self.lc2 = lc1, lc2
        self.alpha = I1 + I2 + m1 * lc1 ** 2 + m2 * (l1 ** 2 + lc2 ** 2)
        self.beta = m2 * l1 * lc2
        self.delta = I2 + m2 * lc2 ** 2

    def _common(self, X, U, F):
        a, b, d = self.alpha, self.beta, self.delta
        q1, q2, w1, w2 = X[:, 0], X[:, 1], X[:, 2], X[:, 3]
        t = dict(s1=np.sin(q1), c1=np.cos(q1), s2=np.sin(q2), c2=np.cos(q2),
                 s12=np.sin(q1 + q2), c12=np.cos(q1 + q2))
        M = _sym2(a + 2.0 * b * t["c2"], d + b * t["c2"], np.full_like(q1, d))
        tau = np.empty((X.shape[0], 2))
        tau[:, 0] = (U[:, 0]
                     + (-self.l1 * t["s1"] - self.l2 * t["s12"]) * F[:, 0]
                     + (self.l1 * t["c1"] + self.l2 * t["c12"]) * F[:, 1]
                     + b * t["s2"] * (2.0 * w1 * w2 + w2 ** 2)
                     - self.joint_damping * w1)
        tau[:, 1] = (U[:, 1]
                     - self.l2 * t["s12"] * F[:, 0]
                     + self.l2 * t["c12"] * F[:, 1]
                     - b * t["s2"] * w1 ** 2
                     - self.joint_damping * w2)
        if self.gravity != 0.0:
            g = self.gravity
            tau[:, 0] -= ((self.m1 * self.lc1 + self.m2 * self.l1) * g * t["c1"]
                          + self.m2 * self.lc2 * g * t["c12"])
            tau[:, 1] -= self.m2 * self.lc2 * g * t["c12"]
        return M, tau, t

    def deriv_many(self, X, U, F):
        M, tau, _ = self._common(X, U, F)
        qdd = np.linalg.solve(M, tau[:, :, None])[:, :, 0]
        return np.concatenate([X[:, 2:], qdd], axis=1)

    def deriv_jacobians_many(self, X, U, F):
        b = self.beta
        B = X.shape[0]
        w1, w2 = X[:, 2], X[:, 3]
        fxc, fyc = F[:, 0], F[:, 1]
        M, tau, t = self._common(X, U, F)
        Minv = np.linalg.inv(M)
        qdd = np.einsum("bij,bj->bi", Minv, tau)

        # d(J^T f)/dq (dynamics.py:643-647)
        tip = np.empty((B, 2, 2))
        tip[:, 0, 0] = ((-self.l1 * t["c1"] - self.l2 * t["c12"]) * fxc
                        + (-self.l1 * t["s1"] - self.l2 * t["s12"]) * fyc)
        tip[:, 0, 1] = -self.l2 * t["c12"] * fxc - self.l2 * t["s12"] * fyc
        tip[:, 1, 0] = tip[:, 0, 1]
        tip[:, 1, 1] = tip[:, 0, 1]
        zero = np.zeros(B)
        dM = _sym2(-2.0 * b * t["s2"], -b * t["s2"], zero)
        dcor_q2 = np.stack([-b * t["c2"] * (2.0 * w1 * w2 + w2 ** 2), b * t["c2"] * w1 ** 2], axis=1)
        dcor_w = np.empty((B, 2, 2))
        dcor_w[:, 0, 0] = -2.0 * b * t["s2"] * w2
        dcor_w[:, 0, 1] = -2.0 * b * t["s2"] * (w1 + w2)
        dcor_w[:, 1, 0] = 2.0 * b * t["s2"] * w1
        dcor_w[:, 1, 1] = 0.0
        dg = np.zeros((B, 2, 2))
        if self.gravity != 0.0:
            g = self.gravity
            dg[:, 0, 0] = (-(self.m1 * self.lc1 + self.m2 * self.l1) * g * t["s1"]
                           - self.m2 * self.lc2 * g * t["s12"])
            dg[:, 0, 1] = -self.m2 * self.lc2 * g * t["s12"]
            dg[:, 1, 0] = dg[:, 0, 1]
            dg[:, 1, 1] = dg[:, 0, 1]
        col0 = np.einsum("bij,bj->bi", Minv, tip[:, :, 0] - dg[:, :, 0])
        col1 = np.einsum("bij,bj->bi", Minv,
                         tip[:, :, 1] - dcor_q2 - dg[:, :, 1] - np.einsum("bij,bj->bi", dM, qdd))
        vel = np.matmul(Minv, -dcor_w - self.joint_damping * np.eye(2))
        fx = np.zeros((B, 4, 4))
        fx[:, 0, 2] = fx[:, 1, 3] = 1.0
        fx[:, 2:, 0] = col0
        fx[:, 2:, 1] = col1
        fx[:, 2:, 2:] = vel
        fu = np.zeros((B, 4, 2))
        fu[:, 2:, :] = Minv
        return fx, fu


def model_from_descriptor(desc):
    """Build the oracle model matching a product/reference model descriptor (by name +
    public parameters), so tests can feed one problem description to both sides."""
    name = getattr(desc, "name", None)
    if name == "double_integrator":
        return PointMasses(desc.dims, desc.mass)
    if name == "pendulum":
        return DampedPendulum(desc.mass, desc.length, desc.gravity, desc.damping)
    if name == "cartpole":
        return HangingCartpole(desc.cart_mass, desc.pole_mass, desc.pole_length, desc.gravity)
    if name == "two_link_arm":
        return PlanarTwoLink(desc.m1, desc.m2, desc.l1, desc.l2, desc.gravity, desc.joint_damping)
    if name == "iiwa14":
        from .iiwa14_np import Iiwa14
        return Iiwa14()
    raise ValueError(f"no oracle model for {name!r}")


# --------------------------------------------------------------------------------------
# RK4 discrete map and its exact Jacobians (dynamics.py:708-816)
# --------------------------------------------------------------------------------------

def rk4_rows(model, X, U, h, F):
    """dynamics.py:805-816 (step_many)."""
    k1 = model.deriv_many(X, U, F)
    k2 = model.deriv_many(X + 0.5 * h * k1, U, F)
    k3 = model.deriv_many(X + 0.5 * h * k2, U, F)
    k4 = model.deriv_many(X + h * k3, U, F)
    return X + (h / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)


def rk4_jacobian_rows(model, X, U, h, F):
    """dynamics.py:774-802 (step_jacobians_many): chain rule through the four stages."""
    rows, n = X.shape
    eye = np.broadcast_to(np.eye(n), (rows, n, n))
    stage_x = X
    sens_x = None      # d k_{s-1} / dx
    sens_u = None
    acc_x = acc_u = None
    for weight, lead in ((1.0, 0.0), (2.0, 0.5 * h), (2.0, 0.5 * h), (1.0, h)):
        if sens_x is not None:
            stage_x = X + lead * k_prev
        gx, gu = model.deriv_jacobians_many(stage_x, U, F)
        if sens_x is None:
            sens_x, sens_u = gx, gu
        else:
            sens_x, sens_u = (np.matmul(gx, eye + lead * sens_x),
                              np.matmul(gx, lead * sens_u) + gu)
        acc_x = sens_x * weight if acc_x is None else acc_x + weight * sens_x
        acc_u = sens_u * weight if acc_u is None else acc_u + weight * sens_u
        if lead != h:
            k_prev = model.deriv_many(stage_x, U, F)
    return eye + (h / 6.0) * acc_x, (h / 6.0) * acc_u


# --------------------------------------------------------------------------------------
# problem container (qpform.py:45-140)
# --------------------------------------------------------------------------------------

@dataclass
class Problem:
    """Flat restatement of CostSpec + ProblemSpec: goals expanded to (N+1, n) and the
    assumed force sampled at knot start times k*h (qpform.py:113-123)."""

    model: object
    Q: np.ndarray
    R: np.ndarray
    QN: np.ndarray
    goals: np.ndarray          # (N+1, n)
    horizon: int
    timestep: float
    x_start: np.ndarray
    forces: np.ndarray         # (N, fdim)

    @classmethod
    def from_spec(cls, spec, model=None):
        """Accepts a reference-style ProblemSpec (product or trajbatch object)."""
        N = spec.horizon
        n = spec.model.state_dim
        goal = np.asarray(spec.cost.goal, dtype=float)
        goals = goal if goal.ndim == 2 else np.broadcast_to(goal, (N + 1, n))
        force = spec.force
        fdim = spec.model.force_dim
        if force is None:
            forces = np.zeros((N, fdim))
        elif force.profile is None:
            forces = np.broadcast_to(np.asarray(force.value, dtype=float), (N, fdim))
        else:
            forces = np.stack([np.asarray(force.profile(k * spec.timestep), dtype=float)
                               for k in range(N)])
        return cls(model if model is not None else model_from_descriptor(spec.model),
                   np.asarray(spec.cost.Q, dtype=float), np.asarray(spec.cost.R, dtype=float),
                   np.asarray(spec.cost.QN, dtype=float), np.array(goals, dtype=float), N,
                   float(spec.timestep), np.asarray(spec.x_start, dtype=float),
                   np.array(forces, dtype=float))

    def defects(self, X, U):
        # qpform.py:133-140
        return rk4_rows(self.model, X[:-1], U, self.timestep, self.forces) - X[1:]

    def cost(self, X, U):
        # qpform.py:71-78
        dx = X[:-1] - self.goals[:-1]
        total = 0.5 * float(np.einsum("ki,ij,kj->", dx, self.Q, dx))
        total += 0.5 * float(np.einsum("ki,ij,kj->", U, self.R, U))
        dxN = X[-1] - self.goals[-1]
        return total + 0.5 * float(dxN @ self.QN @ dxN)


# --------------------------------------------------------------------------------------
# QP formation (qpform.py:156-397)
# --------------------------------------------------------------------------------------

@dataclass
class Expansion:
    """Stacked Taylor expansion along a trajectory (qpform.py:144-197).  Hessian blocks are
    the three distinct damped matrices; gradients use the undamped weights."""

    A: np.ndarray      # (N, n, n)
    B: np.ndarray      # (N, n, m)
    e: np.ndarray      # (N, n)
    q: np.ndarray      # (N+1, n)
    r: np.ndarray      # (N, m)
    Qs: np.ndarray     # stage state Hessian  Q + rho I
    Rs: np.ndarray     # stage control Hessian R (+ rho I)
    Qt: np.ndarray     # terminal Hessian QN + rho I


def expand(p: Problem, X, U, rho, regularize_r=True) -> Expansion:
    n, m, N = p.Q.shape[0], p.R.shape[0], p.horizon
    A, B = rk4_jacobian_rows(p.model, X[:-1], U, p.timestep, p.forces)
    e = rk4_rows(p.model, X[:-1], U, p.timestep, p.forces) - X[1:]
    q = np.empty((N + 1, n))
    q[:-1] = (X[:-1] - p.goals[:-1]) @ p.Q.T
    q[-1] = p.QN @ (X[N] - p.goals[N])
    r = U @ p.R.T
    Rs = p.R + rho * np.eye(m) if regularize_r else p.R.copy()
    return Expansion(A, B, e, q, r, p.Q + rho * np.eye(n), Rs, p.QN + rho * np.eye(n))


def spd_inverse(mat, label, knot=None):
    """qpform.py:261-268: lower Cholesky, solve against I, symmetrise."""
    try:
        factor = scipy.linalg.cho_factor(mat, lower=True, check_finite=False)
    except np.linalg.LinAlgError as exc:
        raise OracleFactorizationError(f"{label} is not positive definite: {exc}", knot) from exc
    inv = scipy.linalg.cho_solve(factor, np.eye(mat.shape[0]), check_finite=False)
    return 0.5 * (inv + inv.T)


@dataclass
class Schur:
    """qpform.py:272-287.  S is stored as in blocktri.py:19-28: diagonal blocks plus the
    sub-diagonal blocks (block k at block position (k+1, k))."""

    diag: np.ndarray           # (N+1, n, n)
    off: np.ndarray            # (N, n, n)
    gamma: np.ndarray          # ((N+1) n,)
    q_inv: np.ndarray          # (N+1, n, n)
    r_inv: np.ndarray          # (N, m, m)


def schur(ex: Expansion, x_start, X) -> Schur:
    """qpform.py:290-339."""
    N, n = ex.A.shape[0], ex.A.shape[1]
    m = ex.B.shape[2]
    # inverse order of failure reporting follows qpform.py:305-311: Q_0 .. Q_N, then R_0 ..
    Qi = spd_inverse(ex.Qs, "Q_0", 0)
    Qti = spd_inverse(ex.Qt, f"Q_{N}", N)
    Ri = spd_inverse(ex.Rs, "R_0", 0)
    q_inv = np.empty((N + 1, n, n))
    q_inv[:-1] = Qi
    q_inv[-1] = Qti
    r_inv = np.broadcast_to(Ri, (N, m, m)).copy()

    AQ = ex.A @ q_inv[:-1]
    BR = ex.B @ r_inv
    theta = AQ @ ex.A.transpose(0, 2, 1) + BR @ ex.B.transpose(0, 2, 1) + q_inv[1:]
    qinv_q = np.einsum("kij,kj->ki", q_inv, ex.q)
    zeta = (-np.einsum("kij,kj->ki", AQ, ex.q[:-1])
            - np.einsum("kij,kj->ki", BR, ex.r) + qinv_q[1:])
    diag = np.empty((N + 1, n, n))
    diag[0] = q_inv[0]
    diag[1:] = theta
    gamma = np.empty((N + 1, n))
    gamma[0] = qinv_q[0] + (np.asarray(x_start, dtype=float) - X[0])
    gamma[1:] = zeta + ex.e
    return Schur(diag, -AQ, gamma.reshape(-1), q_inv, r_inv)


def stair_preconditioner(diag, off):
    """qpform.py:342-359: (diag, off) of the symmetric stair approximate inverse."""
    nb = diag.shape[0]
    dinv = np.empty_like(diag)
    for k in range(nb):
        dinv[k] = spd_inverse(diag[k], f"S diagonal block {k}", k)
    poff = np.empty_like(off)
    for k in range(nb - 1):
        poff[k] = -dinv[k + 1] @ off[k] @ dinv[k]
    return dinv, poff


def recover(ex: Expansion, sc: Schur, lam):
    """qpform.py:375-397 -> (dX, dU); inf-norm per qpform.py:369-372."""
    N, n = ex.A.shape[0], ex.A.shape[1]
    L = np.asarray(lam, dtype=float).reshape(N + 1, n)
    gx = ex.q.copy()
    gx -= L
    gx[:-1] += np.einsum("kji,kj->ki", ex.A, L[1:])
    gu = ex.r + np.einsum("kji,kj->ki", ex.B, L[1:])
    dX = -np.einsum("kij,kj->ki", sc.q_inv, gx)
    dU = -np.einsum("kij,kj->ki", sc.r_inv, gu)
    return dX, dU


def step_inf_norm(dX, dU):
    du = float(np.max(np.abs(dU))) if dU.size else 0.0
    return max(float(np.max(np.abs(dX))), du)


# --------------------------------------------------------------------------------------
# block-tridiagonal algebra and PCG (blocktri.py:92-173)
# --------------------------------------------------------------------------------------

def bt_dense(diag, off):
    """blocktri.py:92-102."""
    nb, bd = diag.shape[0], diag.shape[1]
    out = np.zeros((nb * bd, nb * bd))
    for k in range(nb):
        out[k * bd:(k + 1) * bd, k * bd:(k + 1) * bd] = diag[k]
    for k in range(nb - 1):
        out[(k + 1) * bd:(k + 2) * bd, k * bd:(k + 1) * bd] = off[k]
        out[k * bd:(k + 1) * bd, (k + 1) * bd:(k + 2) * bd] = off[k].T
    return out


def bt_matvec(diag, off, v):
    """blocktri.py:105-120: diagonal term, then sub-diagonal, then super-diagonal."""
    nb, bd = diag.shape[0], diag.shape[1]
    V = np.asarray(v, dtype=float).reshape(nb, bd)
    out = np.einsum("kij,kj->ki", diag, V)
    if nb > 1:
        out[1:] += np.einsum("kij,kj->ki", off, V[:-1])
        out[:-1] += np.einsum("kji,kj->ki", off, V[1:])
    return out.reshape(-1)


@dataclass
class PcgOutcome:
    solution: np.ndarray
    iterations: int
    converged: bool
    residual: float


def pcg(diag, off, gamma, pdiag, poff, tolerance, cap) -> PcgOutcome:
    """blocktri.py:123-173, including the true-residual stop test (an extra matvec)."""
    gamma = np.asarray(gamma, dtype=float)
    lam = np.zeros_like(gamma)
    r = gamma.copy()
    res = float(np.linalg.norm(r))
    if res <= tolerance:
        return PcgOutcome(lam, 0, True, res)
    z = bt_matvec(pdiag, poff, r)
    p = z
    rz = float(r @ z)
    for it in range(1, cap + 1):
        Sp = bt_matvec(diag, off, p)
        curv = float(p @ Sp)
        if curv <= 0.0:
            raise OraclePcgBreakdown(
                f"non-positive curvature {curv:.3e} at PCG iteration {it}", it)
        a = rz / curv
        lam = lam + a * p
        r = r - a * Sp
        res = float(np.linalg.norm(bt_matvec(diag, off, lam) - gamma))
        if res <= tolerance:
            return PcgOutcome(lam, it, True, res)
        z = bt_matvec(pdiag, poff, r)
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return PcgOutcome(lam, cap, False, res)


# --------------------------------------------------------------------------------------
# merit, line search, rho (sqp.py:111-201)
# --------------------------------------------------------------------------------------

def violation_l1(p: Problem, X, U):
    """sqp.py:111-115."""
    total = float(np.sum(np.abs(p.x_start - X[0])))
    total += float(np.sum(np.abs(p.defects(X, U))))
    return total


def merit_value(p: Problem, X, U, mu):
    """sqp.py:118-129."""
    if not (np.all(np.isfinite(X)) and np.all(np.isfinite(U))):
        return math.inf
    with np.errstate(over="ignore", invalid="ignore"):
        value = p.cost(X, U) + mu * violation_l1(p, X, U)
    return value if math.isfinite(value) else math.inf


def merit_candidates(p: Problem, Xs, Us, mu, parts=False):
    """sqp.py:132-166: C candidate trajectories scored in one pass; non-finite -> +inf."""
    C, Np1, n = Xs.shape
    N, m = Np1 - 1, Us.shape[2]
    ok = np.isfinite(Xs).all(axis=(1, 2)) & np.isfinite(Us).all(axis=(1, 2))
    if not ok.all():
        Xs = np.where(ok[:, None, None], Xs, 0.0)
        Us = np.where(ok[:, None, None], Us, 0.0)
    forces = np.tile(p.forces, (C, 1))
    with np.errstate(over="ignore", invalid="ignore"):
        pred = rk4_rows(p.model, Xs[:, :-1].reshape(C * N, n), Us.reshape(C * N, m),
                        p.timestep, forces).reshape(C, N, n)
        gap = pred - Xs[:, 1:]
        viol = np.abs(p.x_start - Xs[:, 0]).sum(axis=1)
        viol += np.abs(gap).sum(axis=(1, 2))
        dx = Xs[:, :-1] - p.goals[:-1]
        val = 0.5 * np.einsum("cki,ij,ckj->c", dx, p.Q, dx)
        val += 0.5 * np.einsum("cki,ij,ckj->c", Us, p.R, Us)
        dxN = Xs[:, -1] - p.goals[-1]
        val += 0.5 * np.einsum("ci,ij,cj->c", dxN, p.QN, dxN)
        val += mu * viol
    out = np.where(ok & np.isfinite(val), val, math.inf)
    return (out, viol) if parts else out


def line_search(p: Problem, X, U, dX, dU, st: Settings, current):
    """sqp.py:169-195 -> (alpha, merit at alpha, accepted); first minimum wins ties."""
    alphas = st.step_lengths()
    Xs = X[None] + alphas[:, None, None] * dX[None]
    Us = U[None] + alphas[:, None, None] * dU[None]
    vals = merit_candidates(p, Xs, Us, st.mu)
    best = int(np.argmin(vals))
    return float(alphas[best]), float(vals[best]), float(vals[best]) < current, vals


def next_rho(rho, accepted, st: Settings):
    """sqp.py:198-201."""
    rho = rho / st.rho_factor if accepted else rho * st.rho_factor
    return float(min(max(rho, st.rho_min), st.rho_max))


# --------------------------------------------------------------------------------------
# SQP loop and batch (sqp.py:204-295, batch.py:92-124)
# --------------------------------------------------------------------------------------

@dataclass
class Record:
    """sqp.py:81-92."""
    iteration: int
    merit: float
    constraint_l1: float
    alpha: float | None
    rho: float
    pcg_iterations: int
    accepted: bool
    step_inf_norm: float


@dataclass
class Result:
    X: np.ndarray
    U: np.ndarray
    trace: list
    converged: bool
    stages: list = field(default_factory=list)   # optional per-iteration stage dumps


def solve(p: Problem, X_init, U_init, st: Settings | None = None, keep_stages=False,
          recurrence_residual=False) -> Result:
    """sqp.py:204-295.  ``keep_stages`` records every intermediate of every iteration for
    stage-by-stage parity tests."""
    st = st or Settings()
    N, n, m = p.horizon, p.Q.shape[0], p.R.shape[0]
    X = np.array(X_init, dtype=float).reshape(N + 1, n)
    U = np.array(U_init, dtype=float).reshape(N, m)
    rho = st.rho_init
    current = merit_value(p, X, U, st.mu)
    trace, stages, converged = [], [], False
    cap = st.pcg_cap((N + 1) * n)

    for it in range(st.max_sqp_iterations):
        retries = 0
        while True:
            try:
                ex = expand(p, X, U, rho, st.regularize_r)
                sc = schur(ex, p.x_start, X)
                pdiag, poff = stair_preconditioner(sc.diag, sc.off)
                out = pcg(sc.diag, sc.off, sc.gamma, pdiag, poff, st.pcg_tolerance, cap)
                break
            except OraclePcgBreakdown as exc:
                retries += 1
                if retries > st.pcg_retry_limit:
                    raise OraclePcgBreakdown(
                        f"SQP iteration {it}: PCG broke down {retries} times "
                        f"(last at inner iteration {exc.iteration})", exc.iteration) from exc
                rho = float(min(rho * st.rho_factor, st.rho_max))
            except OracleFactorizationError as exc:
                raise OracleFactorizationError(f"SQP iteration {it}: {exc}", exc.knot) from exc

        dX, dU = recover(ex, sc, out.solution)
        step_inf = step_inf_norm(dX, dU)
        viol = violation_l1(p, X, U)
        stage = None
        if keep_stages:
            stage = dict(A=ex.A, B=ex.B, e=ex.e, q=ex.q, r=ex.r, Sdiag=sc.diag, Soff=sc.off,
                         gamma=sc.gamma, Pdiag=pdiag, Poff=poff, lam=out.solution,
                         pcg_iterations=out.iterations, dX=dX, dU=dU, rho=rho,
                         X=X.copy(), U=U.copy())
            stages.append(stage)

        if (st.step_tolerance is not None and step_inf <= st.step_tolerance
                and viol <= st.feasibility_tolerance):
            trace.append(Record(it, current, viol, None, rho, out.iterations, False, step_inf))
            converged = True
            break

        alpha, best, accepted, vals = line_search(p, X, U, dX, dU, st, current)
        if stage is not None:
            stage["merits"] = vals
        if accepted:
            X = X + alpha * dX
            U = U + alpha * dU
            current = best
            viol = violation_l1(p, X, U)
        trace.append(Record(it, current, viol, alpha, rho, out.iterations, accepted, step_inf))
        rho = next_rho(rho, accepted, st)

    return Result(X, U, trace, converged, stages)


def solve_batch(problems, inits, settings_list):
    """batch.py:92-124 with workers=1 semantics: per-slot error isolation, input order."""
    results, errors, times = [], [], []
    start = time.perf_counter()
    for p, (X0, U0), st in zip(problems, inits, settings_list):
        t0 = time.perf_counter()
        try:
            results.append(solve(p, X0, U0, st))
            errors.append(None)
        except OracleFactorizationError as exc:
            results.append(None)
            errors.append(f"FactorizationError: {exc}")
        except OraclePcgBreakdown as exc:
            results.append(None)
            errors.append(f"PcgBreakdownError: {exc}")
        times.append(time.perf_counter() - t0)
    return results, errors, time.perf_counter() - start, times


def _pool_task(task):
    p, X0, U0, st = task
    try:
        return solve(p, X0, U0, st), None
    except OracleFactorizationError as exc:
        return None, f"FactorizationError: {exc}"
    except OraclePcgBreakdown as exc:
        return None, f"PcgBreakdownError: {exc}"


def solve_batch_parallel(problems, inits, settings_list, workers):
    """batch.py:102-124 with workers>1: forked process pool, one task per problem, results in
    input order.  Used by bench.py as the all-host-cores CPU arm."""
    import multiprocessing
    from concurrent.futures import ProcessPoolExecutor

    tasks = [(p, X0, U0, st) for p, (X0, U0), st in zip(problems, inits, settings_list)]
    start = time.perf_counter()
    if workers <= 1 or len(tasks) == 1:
        outcomes = [_pool_task(t) for t in tasks]
    else:
        ctx = multiprocessing.get_context("fork")
        with ProcessPoolExecutor(max_workers=workers, mp_context=ctx) as pool:
            chunk = max(1, len(tasks) // (4 * workers))
            outcomes = list(pool.map(_pool_task, tasks, chunksize=chunk))
    wall = time.perf_counter() - start
    return [o[0] for o in outcomes], [o[1] for o in outcomes], wall
