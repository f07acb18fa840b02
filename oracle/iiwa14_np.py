"""ORACLE (test infrastructure, never shipped on the product path).

numpy model of the KUKA LBR iiwa 14 R820 as a ``DynamicsModel`` plug-in.

The reference package has no manipulator model: its
plug-in contract is ``DynamicsModel`` (/root/reference/pkg/src/trajbatch/dynamics.py:94-142)
and its force-channel convention is the one of ``TwoLinkArm`` (dynamics.py:493-503: a
task-space force at the end effector mapped through J(q)^T).  This file restates that
contract for a 7-revolute serial chain:

    state x = [q (7); qd (7)],  control u = joint torque (7),
    force  f = world-frame linear force applied at the flange point (3),
    xdot    = [qd ; M(q)^-1 (u - ID(q, qd, 0; gravity, f))]

ID is the recursive Newton-Euler inverse dynamics in link coordinates (Featherstone's
spatial notation, motion vectors (w, v) / force vectors (n, f) kept as two 3-vectors).
The analytic partials use the identity d qdd / d(.) = -M^-1 d ID(q, qd, qdd)/d(.) with
qdd held fixed and the tangent recursion of the same Newton-Euler passes.

PARITY UNPINNED by the reference: nothing under /root/reference fixes these numbers.
What pins this file is (a) the reference's own test patterns run against it (finite
difference Jacobians, batched-vs-scalar, dynamics.py contract) in tests/test_iiwa14_model.py
and (b) an independent Lagrangian (Jacobian/energy based) evaluation in the same test file.
The parameter table below is the repo's model definition; the CUDA
model in paper_2510_07625_b200/csrc/model_iiwa14.cuh carries the same table.
"""

from __future__ import annotations

import numpy as np

NJ = 7
GRAVITY = 9.81

# parent->joint origin (xyz, metres), parent frame coordinates
ORIGIN_XYZ = np.array([
    [0.0, 0.0, 0.1575],
    [0.0, 0.0, 0.2025],
    [0.0, 0.2045, 0.0],
    [0.0, 0.0, 0.2155],
    [0.0, 0.1845, 0.0],
    [0.0, 0.0, 0.2155],
    [0.0, 0.081, 0.0],
])
# URDF rpy of each joint origin, in units of pi/2 so the fixed rotations are exact
# signed permutation matrices (roll, pitch, yaw)
ORIGIN_RPY_QUARTERS = np.array([
    [0, 0, 0],
    [1, 0, 2],
    [1, 0, 2],
    [1, 0, 0],
    [-1, 2, 0],
    [1, 0, 0],
    [-1, 2, 0],
])
MASS = np.array([4.0, 4.0, 3.0, 2.7, 1.7, 1.8, 0.3])
COM = np.array([
    [0.0, -0.03, 0.12],
    [0.0003, 0.059, 0.042],
    [0.0, 0.03, 0.13],
    [0.0, 0.067, 0.034],
    [0.0001, 0.021, 0.076],
    [0.0, 0.0006, 0.0004],
    [0.0, 0.0, 0.02],
])
INERTIA_DIAG = np.array([
    [0.1, 0.09, 0.02],
    [0.05, 0.018, 0.044],
    [0.08, 0.075, 0.01],
    [0.03, 0.01, 0.029],
    [0.02, 0.018, 0.005],
    [0.005, 0.0036, 0.0047],
    [0.001, 0.001, 0.001],
])
FLANGE_XYZ = np.array([0.0, 0.0, 0.045])   # in link-7 coordinates


def _quarter_rot(axis: int, quarters: int) -> np.ndarray:
    c = [1, 0, -1, 0][quarters % 4]
    s = [0, 1, 0, -1][quarters % 4]
    R = np.eye(3)
    a, b = [(1, 2), (2, 0), (0, 1)][axis]
    R[a, a] = c
    R[a, b] = -s
    R[b, a] = s
    R[b, b] = c
    return R


def fixed_rotations() -> np.ndarray:
    """R_T[i]: joint-frame -> parent-frame coordinates, exact entries in {0, +-1}."""
    out = np.empty((NJ, 3, 3))
    for i, (roll, pitch, yaw) in enumerate(ORIGIN_RPY_QUARTERS):
        out[i] = _quarter_rot(2, yaw) @ _quarter_rot(1, pitch) @ _quarter_rot(0, roll)
    return out


R_FIXED = fixed_rotations()
E_FIXED = np.transpose(R_FIXED, (0, 2, 1))      # parent -> joint frame


def _cross(a, b):
    return np.stack([
        a[..., 1] * b[..., 2] - a[..., 2] * b[..., 1],
        a[..., 2] * b[..., 0] - a[..., 0] * b[..., 2],
        a[..., 0] * b[..., 1] - a[..., 1] * b[..., 0],
    ], axis=-1)


def _cross_z(a):
    """a x z_hat."""
    return np.stack([a[..., 1], -a[..., 0], np.zeros_like(a[..., 0])], axis=-1)


def _z_cross(a):
    """z_hat x a."""
    return np.stack([-a[..., 1], a[..., 0], np.zeros_like(a[..., 0])], axis=-1)


class _Kin:
    """sin/cos of the joint angles; applies the parent->link rotation E_i = Rz(q_i)^T E_T."""

    def __init__(self, q):
        self.s = np.sin(q)
        self.c = np.cos(q)

    def down(self, i, vec):
        """Rotate parent coordinates into link-i coordinates. vec (..., 3) with leading
        batch axis matching q's; extra middle axes broadcast."""
        t = vec @ R_FIXED[i]                  # = (E_T vec) for row vectors
        s, c = self.s[:, i], self.c[:, i]
        while s.ndim < t.ndim - 1:
            s = s[..., None]
            c = c[..., None]
        return np.stack([
            c * t[..., 0] + s * t[..., 1],
            -s * t[..., 0] + c * t[..., 1],
            t[..., 2],
        ], axis=-1)

    def up(self, i, vec):
        """Rotate link-i coordinates into parent coordinates."""
        s, c = self.s[:, i], self.c[:, i]
        while s.ndim < vec.ndim - 1:
            s = s[..., None]
            c = c[..., None]
        t = np.stack([
            c * vec[..., 0] - s * vec[..., 1],
            s * vec[..., 0] + c * vec[..., 1],
            vec[..., 2],
        ], axis=-1)
        return t @ E_FIXED[i]                 # = R_T t for row vectors


def _inertia_apply(i, w, v):
    """Spatial inertia of link i applied to a motion vector (w, v) -> force vector (n, f)."""
    f = MASS[i] * (v + _cross(w, COM[i]))
    n = INERTIA_DIAG[i] * w + _cross(np.broadcast_to(COM[i], f.shape), f)
    return n, f


def _newton_euler(q, qd, qdd, fw, gravity=GRAVITY, keep=False):
    """Inverse dynamics tau = ID(q, qd, qdd) - J^T fw for (B, 7) stacks.

    With ``keep`` the per-link primal quantities needed by the tangent pass are returned.
    """
    B = q.shape[0]
    kin = _Kin(q)
    w = np.zeros((B, 3))
    v = np.zeros((B, 3))
    aw = np.zeros((B, 3))
    av = np.zeros((B, 3))
    av[:, 2] = gravity                       # base "accelerates upward": gravity trick
    g = fw
    W, V, AWP, AVP, NN, FF = [], [], [], [], [], []
    for i in range(NJ):
        p = ORIGIN_XYZ[i]
        w_t = kin.down(i, w)
        v_t = kin.down(i, v + _cross(w, p))
        aw_t = kin.down(i, aw)
        av_t = kin.down(i, av + _cross(aw, p))
        g = kin.down(i, g)
        w = w_t.copy()
        w[:, 2] += qd[:, i]
        v = v_t
        # a_i = X a_p + S qdd + v_i x S qd
        aw = aw_t + qd[:, i, None] * _cross_z(w)
        aw[:, 2] += qdd[:, i]
        av = av_t + qd[:, i, None] * _cross_z(v)
        hn, hf = _inertia_apply(i, w, v)
        n, f = _inertia_apply(i, aw, av)
        n = n + _cross(w, hn) + _cross(v, hf)
        f = f + _cross(w, hf)
        if i == NJ - 1:
            n = n - _cross(np.broadcast_to(FLANGE_XYZ, g.shape), g)
            f = f - g
        W.append(w); V.append(v); AWP.append(aw_t); AVP.append(av_t)
        NN.append(n); FF.append(f)
    tau = np.empty((B, NJ))
    for i in range(NJ - 1, -1, -1):
        tau[:, i] = NN[i][:, 2]
        if i > 0:
            f_up = kin.up(i, FF[i])
            n_up = kin.up(i, NN[i]) + _cross(np.broadcast_to(ORIGIN_XYZ[i], f_up.shape), f_up)
            NN[i - 1] = NN[i - 1] + n_up
            FF[i - 1] = FF[i - 1] + f_up
    if keep:
        return tau, dict(kin=kin, W=W, V=V, AWP=AWP, AVP=AVP, N=NN, F=FF, g7=g)
    return tau


def mass_matrix(q):
    """Joint-space inertia M(q), (B, 7, 7): column j = ID(q, 0, e_j) without gravity."""
    B = q.shape[0]
    M = np.empty((B, NJ, NJ))
    zero = np.zeros((B, NJ))
    nof = np.zeros((B, 3))
    for j in range(NJ):
        e = np.zeros((B, NJ))
        e[:, j] = 1.0
        M[:, :, j] = _newton_euler(q, zero, e, nof, gravity=0.0)
    return 0.5 * (M + np.transpose(M, (0, 2, 1)))


def _newton_euler_tangent(q, qd, fw, kept, dq, dqd):
    """Directional derivatives of ID at fixed qdd along D directions.

    dq, dqd: (B, D, 7).  Returns (B, D, 7).
    """
    B, D, _ = dq.shape
    kin = kept["kin"]
    zero = np.zeros((B, D, 3))
    dw, dv, daw, dav = zero, zero, zero, zero
    # world force rotated down the chain and its tangent
    g = fw
    dg = zero
    dN, dF = [], []
    for i in range(NJ):
        p = ORIGIN_XYZ[i]
        w, v = kept["W"][i][:, None, :], kept["V"][i][:, None, :]
        awp, avp = kept["AWP"][i][:, None, :], kept["AVP"][i][:, None, :]
        dqi = dq[:, :, i, None]
        dqdi = dqd[:, :, i, None]
        qdi = qd[:, None, i, None]
        g = kin.down(i, g)
        dg = kin.down(i, dg) + dqi * _cross_z(g[:, None, :])
        # d v_i = X d v_p + dq_i (v_i x S) + S dqd_i
        dw_n = kin.down(i, dw) + dqi * _cross_z(w)
        dv_n = kin.down(i, dv + _cross(dw, p)) + dqi * _cross_z(v)
        dw_n = dw_n.copy()
        dw_n[..., 2] += dqdi[..., 0]
        # d a_i = X d a_p + dq_i ((X a_p) x S) + d v_i x S qd_i + v_i x S dqd_i
        daw_n = (kin.down(i, daw) + dqi * _cross_z(awp)
                 + qdi * _cross_z(dw_n) + dqdi * _cross_z(w))
        dav_n = (kin.down(i, dav + _cross(daw, p)) + dqi * _cross_z(avp)
                 + qdi * _cross_z(dv_n) + dqdi * _cross_z(v))
        dw, dv, daw, dav = dw_n, dv_n, daw_n, dav_n
        hn, hf = _inertia_apply(i, w, v)
        dhn, dhf = _inertia_apply(i, dw, dv)
        n, f = _inertia_apply(i, daw, dav)
        n = n + _cross(dw, hn) + _cross(dv, hf) + _cross(w, dhn) + _cross(v, dhf)
        f = f + _cross(dw, hf) + _cross(w, dhf)
        if i == NJ - 1:
            n = n - _cross(np.broadcast_to(FLANGE_XYZ, dg.shape), dg)
            f = f - dg
        dN.append(n)
        dF.append(f)
    dtau = np.empty((B, D, NJ))
    for i in range(NJ - 1, -1, -1):
        dtau[:, :, i] = dN[i][..., 2]
        if i > 0:
            dqi = dq[:, :, i, None]
            Ni, Fi = kept["N"][i][:, None, :], kept["F"][i][:, None, :]
            # d(X^T F) = X^T (dF + dq_i S x* F)
            f_loc = dF[i] + dqi * _z_cross(Fi)
            n_loc = dN[i] + dqi * _z_cross(Ni)
            f_up = kin.up(i, f_loc)
            n_up = kin.up(i, n_loc) + _cross(np.broadcast_to(ORIGIN_XYZ[i], f_up.shape), f_up)
            dN[i - 1] = dN[i - 1] + n_up
            dF[i - 1] = dF[i - 1] + f_up
    return dtau


def flange_position(q):
    """World position of the flange point, (B, 3) (used by tests and the independent check)."""
    B = q.shape[0]
    kin = _Kin(q)
    p = np.broadcast_to(FLANGE_XYZ, (B, 3))
    for i in range(NJ - 1, -1, -1):
        p = kin.up(i, p) + ORIGIN_XYZ[i]
    return p


class Iiwa14:
    """7-DoF iiwa14 plug-in following the reference ``DynamicsModel`` contract
    (dynamics.py:94-142).  Duck-typed: it does not import the reference so it can run
    on the GPU box; tests/golden/make_golden.py mixes it with trajbatch.DynamicsModel."""

    name = "iiwa14"
    state_dim = 14
    control_dim = 7
    force_dim = 3
    position_dim = 7

    def __eq__(self, other):
        return isinstance(other, Iiwa14)

    def __hash__(self):
        return hash("iiwa14")

    # -- vectorised interface ------------------------------------------------ #
    def deriv_many(self, X, U, F):
        X = np.asarray(X, dtype=float)
        q, qd = X[:, :NJ], X[:, NJ:]
        bias = _newton_euler(q, qd, np.zeros_like(q), np.asarray(F, dtype=float))
        M = mass_matrix(q)
        qdd = np.linalg.solve(M, (U - bias)[:, :, None])[:, :, 0]
        return np.concatenate([qd, qdd], axis=1)

    def deriv_jacobians_many(self, X, U, F):
        X = np.asarray(X, dtype=float)
        F = np.asarray(F, dtype=float)
        B = X.shape[0]
        q, qd = X[:, :NJ], X[:, NJ:]
        bias = _newton_euler(q, qd, np.zeros_like(q), F)
        M = mass_matrix(q)
        Minv = np.linalg.inv(M)
        Minv = 0.5 * (Minv + np.transpose(Minv, (0, 2, 1)))
        qdd = np.einsum("bij,bj->bi", Minv, U - bias)
        _, kept = _newton_euler(q, qd, qdd, F, keep=True)
        eye = np.broadcast_to(np.eye(NJ), (B, NJ, NJ))
        zero = np.zeros((B, NJ, NJ))
        dq = np.concatenate([eye, zero], axis=1)       # (B, 14, 7): directions q_j then qd_j
        dqd = np.concatenate([zero, eye], axis=1)
        dtau = _newton_euler_tangent(q, qd, F, kept, dq, dqd)       # (B, 14, 7)
        dqdd = -np.einsum("bij,bdj->bid", Minv, dtau)               # (B, 7, 14)
        fx = np.zeros((B, 14, 14))
        fx[:, :NJ, NJ:] = np.eye(NJ)
        fx[:, NJ:, :] = dqdd
        fu = np.zeros((B, 14, NJ))
        fu[:, NJ:, :] = Minv
        return fx, fu

    # -- scalar interface ---------------------------------------------------- #
    def deriv(self, x, u, f):
        return self.deriv_many(np.asarray(x)[None], np.asarray(u)[None], np.asarray(f)[None])[0]

    def deriv_jacobians(self, x, u, f):
        fx, fu = self.deriv_jacobians_many(
            np.asarray(x)[None], np.asarray(u)[None], np.asarray(f)[None])
        return fx[0], fu[0]

    def gravity_torque(self, q):
        """u that holds the arm still at q (zero velocity, zero external force)."""
        q = np.asarray(q, dtype=float)[None]
        return _newton_euler(q, np.zeros_like(q), np.zeros_like(q), np.zeros((1, 3)))[0]
