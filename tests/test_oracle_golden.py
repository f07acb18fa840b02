"""The numpy oracle against the committed outputs of the unmodified reference
(tests/golden/*.npz, made by tests/golden/make_golden.py).  This is what pins the oracle."""

import numpy as np
import pytest

from conftest import (ALL_CASES, STAGED_CASES, load_golden, oracle_problem, oracle_settings, rel_inf,
                      trace_rows)
from oracle import trajopt_np as orc


@pytest.mark.parametrize("name", ALL_CASES)
def test_full_solve_is_bitwise_the_reference(name):
    g = load_golden(name)
    res = orc.solve(oracle_problem(g), g["X0"], g["U0"], oracle_settings(g))
    assert np.array_equal(res.X, g["X"])
    assert np.array_equal(res.U, g["U"])
    assert res.converged == bool(g["converged"])
    assert np.array_equal(trace_rows(res), g["trace"], equal_nan=True)


@pytest.mark.parametrize("name", STAGED_CASES)
def test_first_iteration_stages(name):
    g = load_golden(name)
    p, st = oracle_problem(g), oracle_settings(g)
    X, U = g["X0"], g["U0"]
    ex = orc.expand(p, X, U, st.rho_init, st.regularize_r)
    for key, val in (("A", ex.A), ("B", ex.B), ("e", ex.e), ("q", ex.q), ("r", ex.r)):
        assert np.array_equal(val, g[key]), key
    sc = orc.schur(ex, p.x_start, X)
    assert np.array_equal(sc.diag, g["Sdiag"]) and np.array_equal(sc.off, g["Soff"])
    assert np.array_equal(sc.gamma, g["gamma"])
    pd, po = orc.stair_preconditioner(sc.diag, sc.off)
    assert np.array_equal(pd, g["Pdiag"]) and np.array_equal(po, g["Poff"])
    out = orc.pcg(sc.diag, sc.off, sc.gamma, pd, po, st.pcg_tolerance, st.pcg_cap(sc.gamma.size))
    assert out.iterations == int(g["pcg_iterations"]) and out.converged == bool(g["pcg_converged"])
    assert np.array_equal(out.solution, g["lam"])
    dX, dU = orc.recover(ex, sc, out.solution)
    assert np.array_equal(dX, g["dX"]) and np.array_equal(dU, g["dU"])
    assert orc.step_inf_norm(dX, dU) == float(g["step_inf"])
    alphas = st.step_lengths()
    vals = orc.merit_candidates(p, X[None] + alphas[:, None, None] * dX[None],
                                U[None] + alphas[:, None, None] * dU[None], st.mu)
    assert np.array_equal(vals, g["merits"])
    assert orc.merit_value(p, X, U, st.mu) == float(g["merit0"])
    assert np.array_equal(orc.rk4_rows(p.model, X[:-1], U, p.timestep, p.forces), g["step_rows"])


def test_known_answers_of_the_reference_tests():
    """Closed-form expectations held by the reference's own tests."""
    # adapt_rho (test_sqp.py:165-179)
    st = orc.Settings()
    assert orc.next_rho(1e-3, True, st) == pytest.approx(2e-4)
    assert orc.next_rho(1e-3, False, st) == pytest.approx(5e-3)
    assert orc.next_rho(st.rho_min, True, st) == st.rho_min
    assert orc.next_rho(st.rho_max, False, st) == st.rho_max
    # candidates (test_sqp.py:142-144)
    assert np.array_equal(orc.Settings(num_shrinks=3).step_lengths(), [1.0, 0.5, 0.25, 0.125])
    # double-integrator step (test_dynamics.py:41-44, 78-86)
    di = orc.PointMasses(1)
    h = 0.1
    out = orc.rk4_rows(di, np.array([[0.0, 0.0]]), np.array([[1.0]]), h, np.zeros((1, 1)))
    assert np.allclose(out, [[0.005, 0.1]], atol=1e-15)
    A, B = orc.rk4_jacobian_rows(di, np.array([[0.3, -0.2]]), np.array([[0.4]]), h, np.zeros((1, 1)))
    assert np.allclose(A[0], [[1, h], [0, 1]], atol=1e-15) and np.allclose(B[0], [[h * h / 2], [h]], atol=1e-15)
    # identity PCG -> one iteration; zero rhs -> zero iterations (test_blocktri.py:61-67, 91-95)
    eye = np.broadcast_to(np.eye(2), (3, 2, 2)).copy()
    off = np.zeros((2, 2, 2))
    gamma = np.arange(1.0, 7.0)
    out = orc.pcg(eye, off, gamma, eye, off, 1e-12, 60)
    assert out.iterations == 1 and out.converged and np.allclose(out.solution, gamma)
    out = orc.pcg(eye, off, np.zeros(6), eye, off, 1e-10, 60)
    assert out.iterations == 0 and out.converged
    assert orc.Settings().pcg_cap(40) == 400   # test_blocktri.py:171-172
    # non-SPD breakdown carries the iteration (test_blocktri.py:104-108)
    with pytest.raises(orc.OraclePcgBreakdown) as info:
        orc.pcg(np.array([[[-1.0]], [[1.0]]]), np.zeros((1, 1, 1)), np.array([1.0, 0.0]),
                np.ones((2, 1, 1)), np.zeros((1, 1, 1)), 1e-8, 20)
    assert info.value.iteration >= 1


def test_failed_slot_is_isolated_in_the_oracle_batch():
    """batch.py:92-99 / test_batch.py:59-75."""
    g = load_golden("pendulum_n8")
    good = oracle_problem(g)
    import dataclasses
    bad = dataclasses.replace(good, Q=np.zeros((2, 2)), R=np.zeros((1, 1)), QN=np.zeros((2, 2)))
    st = orc.Settings(max_sqp_iterations=3, step_tolerance=None, rho_init=0.0, rho_min=0.0, regularize_r=False)
    init = (g["X0"], g["U0"])
    results, errors, _, _ = orc.solve_batch([good, bad, good], [init] * 3, [st] * 3)
    assert results[1] is None and errors[1].startswith("FactorizationError: SQP iteration 0: Q_0")
    assert results[0] is not None and np.array_equal(results[0].X, results[2].X)
