"""Live comparison of the oracle with the reference package, when it is present
(build container only; /root/reference does not exist on the GPU box)."""

import sys

import numpy as np
import pytest

from conftest import REFERENCE_SRC
from oracle import trajopt_np as orc

pytestmark = [pytest.mark.reference,
              pytest.mark.skipif(not REFERENCE_SRC.exists(), reason="reference package not mounted")]


@pytest.fixture(scope="module")
def tb():
    sys.path.insert(0, str(REFERENCE_SRC))
    import trajbatch
    return trajbatch


def _oracle_problem(tb, problem):
    return orc.Problem.from_spec(problem)


@pytest.mark.parametrize("seed", range(8))
def test_random_instances_match_bitwise(tb, seed):
    """oracles.random_problem (oracles.py:136-163) over the reference's model pool."""
    from trajbatch import oracles
    rng = np.random.default_rng(1000 + seed)
    problem, X, U = oracles.random_problem(rng)
    ref = tb.sqp_solve(problem, X, U, tb.SolverSettings(max_sqp_iterations=8))
    got = orc.solve(_oracle_problem(tb, problem), X, U, orc.Settings(max_sqp_iterations=8))
    assert np.array_equal(got.X, ref.X) and np.array_equal(got.U, ref.U)
    assert got.converged == ref.converged and len(got.trace) == len(ref.trace)
    for a, b in zip(got.trace, ref.trace):
        assert (a.merit, a.constraint_l1, a.alpha, a.rho, a.pcg_iterations, a.accepted, a.step_inf_norm) == \
               (b.merit, b.constraint_l1, b.alpha, b.rho, b.pcg_iterations, b.accepted, b.step_inf_norm)


def test_models_match_the_reference_rowwise(tb, rng):
    pairs = [(tb.DoubleIntegrator(dims=2), orc.PointMasses(2)), (tb.Pendulum(), orc.DampedPendulum()),
             (tb.Cartpole(), orc.HangingCartpole()), (tb.TwoLinkArm(), orc.PlanarTwoLink()),
             (tb.TwoLinkArm(gravity=9.81), orc.PlanarTwoLink(gravity=9.81))]
    for ref, mine in pairs:
        X = rng.standard_normal((20, ref.state_dim))
        U = rng.standard_normal((20, ref.control_dim))
        F = rng.standard_normal((20, ref.force_dim))
        assert np.array_equal(mine.deriv_many(X, U, F), ref.deriv_many(X, U, F))
        for a, b in zip(mine.deriv_jacobians_many(X, U, F), ref.deriv_jacobians_many(X, U, F)):
            assert np.array_equal(a, b)


def test_time_varying_force_is_sampled_at_knot_starts(tb):
    """qpform.py:113-123."""
    profile = tb.SwingingLoadProfile(weight=1.0)
    arm = tb.TwoLinkArm()
    cost = tb.CostSpec(np.eye(4), np.eye(2), np.eye(4), np.zeros(4))
    problem = tb.ProblemSpec(arm, cost, 6, 0.05, np.zeros(4), tb.ExternalForce.time_varying(profile, 2))
    assert np.array_equal(orc.Problem.from_spec(problem).forces, problem.force_matrix())


def test_schur_kkt_equivalence_through_the_reference_dense_solve(tb):
    """The oracle's Schur/PCG/recover step equals the reference's dense KKT solve
    (oracles.solve_kkt_dense, oracles.py:40-66; acceptance #1)."""
    from trajbatch import oracles, qpform
    rng = np.random.default_rng(2024)
    for _ in range(10):
        problem, X, U = oracles.random_problem(rng)
        blocks = qpform.linearize(problem, X, U, 1e-6)
        dz, _ = oracles.solve_kkt_dense(qpform.form_kkt(blocks, problem.x_start, X))
        p = _oracle_problem(tb, problem)
        ex = orc.expand(p, X, U, 1e-6)
        sc = orc.schur(ex, p.x_start, X)
        pd, po = orc.stair_preconditioner(sc.diag, sc.off)
        out = orc.pcg(sc.diag, sc.off, sc.gamma, pd, po, 1e-12, 10 * sc.gamma.size)
        dX, dU = orc.recover(ex, sc, out.solution)
        n, m, N = p.Q.shape[0], p.R.shape[0], p.horizon
        mine = np.concatenate([np.concatenate([dX[k], dU[k]]) for k in range(N)] + [dX[N]])
        assert np.max(np.abs(mine - dz)) / max(1.0, np.max(np.abs(dz))) <= 1e-6
