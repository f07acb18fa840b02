"""oracle/iiwa14_np.py follows the reference's DynamicsModel contract (dynamics.py:94-142).
The reference has no manipulator model, so this file applies the reference's own dynamics
test patterns (test_dynamics.py:102-156) plus an independent Lagrangian evaluation."""

import numpy as np
import pytest

from oracle import iiwa14_np as I
from oracle import trajopt_np as orc


@pytest.fixture(scope="module")
def model():
    return I.Iiwa14()


def _lagrangian_terms(q):
    """Independent route: world-frame geometric Jacobians, M = sum J^T I J, gravity gradient."""
    R, p, frames = np.eye(3), np.zeros(3), []
    for i in range(7):
        p = p + R @ I.ORIGIN_XYZ[i]
        c, s = np.cos(q[i]), np.sin(q[i])
        R = R @ I.R_FIXED[i] @ np.array([[c, -s, 0], [s, c, 0], [0, 0, 1.0]])
        frames.append((R.copy(), p.copy()))
    zs = [Rp[0][:, 2] for Rp in frames]
    ps = [Rp[1] for Rp in frames]
    M, grav = np.zeros((7, 7)), np.zeros(7)
    for i, (Ri, pi) in enumerate(frames):
        com = pi + Ri @ I.COM[i]
        Jv, Jw = np.zeros((3, 7)), np.zeros((3, 7))
        for j in range(i + 1):
            Jv[:, j] = np.cross(zs[j], com - ps[j])
            Jw[:, j] = zs[j]
        M += I.MASS[i] * Jv.T @ Jv + Jw.T @ (Ri @ np.diag(I.INERTIA_DIAG[i]) @ Ri.T) @ Jw
        grav += I.MASS[i] * I.GRAVITY * Jv[2]
    tip = frames[6][1] + frames[6][0] @ I.FLANGE_XYZ
    Je = np.stack([np.cross(zs[j], tip - ps[j]) for j in range(7)], axis=1)
    return M, grav, Je, tip


def _lagrangian_qdd(q, qd, u, f, eps=1e-6):
    M, grav, Je, _ = _lagrangian_terms(q)
    dM = np.zeros((7, 7, 7))
    for k in range(7):
        d = np.zeros(7)
        d[k] = eps
        dM[:, :, k] = (_lagrangian_terms(q + d)[0] - _lagrangian_terms(q - d)[0]) / (2 * eps)
    cor = np.einsum("ijk,j,k->i", dM, qd, qd) - 0.5 * np.einsum("jki,j,k->i", dM, qd, qd)
    return np.linalg.solve(M, u + Je.T @ f - cor - grav)


def test_forward_dynamics_matches_independent_lagrangian(model, rng):
    for _ in range(6):
        x = rng.uniform(-1.5, 1.5, 14)
        u = rng.uniform(-30, 30, 7)
        f = rng.uniform(-10, 10, 3)
        ref = _lagrangian_qdd(x[:7], x[7:], u, f)
        got = model.deriv(x, u, f)
        assert np.allclose(got[:7], x[7:])
        assert np.max(np.abs(got[7:] - ref)) <= 1e-6 * max(1.0, np.max(np.abs(ref)))
        M, _, _, tip = _lagrangian_terms(x[:7])
        assert np.allclose(I.mass_matrix(x[None, :7])[0], M, atol=1e-12)
        assert np.allclose(I.flange_position(x[None, :7])[0], tip, atol=1e-14)


def test_analytic_jacobians_match_central_differences(model, rng):
    """test_dynamics.py:102-112 pattern, tolerance scaled by the magnitude of the entries."""
    B = 20
    X = rng.uniform(-1.0, 1.0, (B, 14))
    U = rng.uniform(-20, 20, (B, 7))
    F = rng.uniform(-10, 10, (B, 3))
    fx, fu = model.deriv_jacobians_many(X, U, F)
    eps = 1e-6
    # rounding noise of a central difference: a few ulps of |xdot| (up to 2e4 here) over 2 eps
    noise = 1e-9 * np.max(np.abs(model.deriv_many(X, U, F)))
    for j in range(14):
        d = np.zeros(14)
        d[j] = eps
        num = (model.deriv_many(X + d, U, F) - model.deriv_many(X - d, U, F)) / (2 * eps)
        assert np.max(np.abs(fx[:, :, j] - num)) <= noise + 1e-6 * max(1.0, np.max(np.abs(num)))
    for j in range(7):
        d = np.zeros(7)
        d[j] = eps
        num = (model.deriv_many(X, U + d, F) - model.deriv_many(X, U - d, F)) / (2 * eps)
        assert np.max(np.abs(fu[:, :, j] - num)) <= noise + 1e-6 * max(1.0, np.max(np.abs(num)))


def test_batched_matches_scalar(model, rng):
    """test_dynamics.py:115-138 pattern."""
    X = rng.uniform(-1.0, 1.0, (5, 14))
    U = rng.uniform(-20, 20, (5, 7))
    F = rng.uniform(-10, 10, (5, 3))
    many = model.deriv_many(X, U, F)
    fx, fu = model.deriv_jacobians_many(X, U, F)
    for i in range(5):
        assert np.allclose(model.deriv(X[i], U[i], F[i]), many[i], rtol=1e-13, atol=1e-13)
        a, b = model.deriv_jacobians(X[i], U[i], F[i])
        assert np.allclose(a, fx[i], rtol=1e-12, atol=1e-12) and np.allclose(b, fu[i], rtol=1e-12, atol=1e-12)


def test_equilibrium_under_gravity_compensation(model, rng):
    """test_dynamics.py:141-156 pattern: holding torque keeps the arm at rest through an RK4 step."""
    for _ in range(4):
        q = rng.uniform(-1.5, 1.5, 7)
        x = np.concatenate([q, np.zeros(7)])
        u = model.gravity_torque(q)
        assert np.max(np.abs(model.deriv(x, u, np.zeros(3)))) <= 1e-9
        out = orc.rk4_rows(model, x[None], u[None], 0.05, np.zeros((1, 3)))[0]
        assert np.max(np.abs(out - x)) <= 1e-10


def test_force_channel_is_flange_jacobian_transpose(model, rng):
    """test_dynamics.py:169-176 pattern: M (qdd(f) - qdd(0)) = J_v(q)^T f."""
    x = np.concatenate([rng.uniform(-1, 1, 7), np.zeros(7)])
    f = np.array([3.0, -2.0, 5.0])
    M, _, Je, _ = _lagrangian_terms(x[:7])
    delta = model.deriv(x, np.zeros(7), f)[7:] - model.deriv(x, np.zeros(7), np.zeros(3))[7:]
    assert np.allclose(M @ delta, Je.T @ f, atol=1e-9)


def test_fixed_rotations_are_signed_permutations():
    for R in I.R_FIXED:
        assert np.array_equal(np.abs(R).sum(axis=0), np.ones(3)) and np.array_equal(R @ R.T, np.eye(3))
        assert np.isclose(np.linalg.det(R), 1.0)
