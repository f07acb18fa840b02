"""Operator-level parity through the C ABI: row-wise RK4 step and its exact Jacobians
(dynamics.py:774-816), batched PCG on explicit block-tridiagonal systems (blocktri.py:105-173)
and the warm-start shift (mpc.py:85-89), against the oracle."""

import numpy as np
import pytest

import paper_2510_07625_b200 as gb
from oracle import trajopt_np as orc
from conftest import rel_inf

pytestmark = pytest.mark.gpu

MODELS = [gb.DoubleIntegrator(dims=1), gb.DoubleIntegrator(dims=2), gb.DoubleIntegrator(dims=7, mass=2.0),
          gb.Pendulum(), gb.Cartpole(), gb.TwoLinkArm(), gb.TwoLinkArm(gravity=9.81), gb.Iiwa14()]


def _points(model, rng, rows):
    scale_u = 20.0 if model.name == "iiwa14" else 1.0
    X = rng.uniform(-1.0, 1.0, (rows, model.state_dim))
    U = scale_u * rng.uniform(-1.0, 1.0, (rows, model.control_dim))
    F = 3.0 * rng.standard_normal((rows, model.force_dim))
    return X, U, F


@pytest.mark.parametrize("model", MODELS, ids=lambda m: f"{m.name}{getattr(m, 'dims', '')}{getattr(m, 'gravity', '')}")
def test_step_and_jacobians_match_oracle(model, rng):
    """test_dynamics.py:102-138 pattern at 100 random points per model."""
    X, U, F = _points(model, rng, 100)
    omodel = orc.model_from_descriptor(model)
    h = 0.03
    out = gb.step_many(model, X, U, h, F)
    ref = orc.rk4_rows(omodel, X, U, h, F)
    assert rel_inf(out, ref) <= 1e-12
    A, B = gb.step_jacobians_many(model, X, U, h, F)
    Ar, Br = orc.rk4_jacobian_rows(omodel, X, U, h, F)
    assert rel_inf(A, Ar) <= 1e-10 and rel_inf(B, Br) <= 1e-10


def test_double_integrator_closed_form():
    """test_dynamics.py:41-44, 78-86."""
    m, h = gb.DoubleIntegrator(dims=1), 0.1
    out = gb.step_many(m, np.zeros((1, 2)), np.ones((1, 1)), h, np.zeros((1, 1)))
    assert np.allclose(out, [[0.005, 0.1]], atol=1e-15)
    A, B = gb.step_jacobians_many(m, np.array([[0.3, -0.2]]), np.array([[0.4]]), h, np.zeros((1, 1)))
    assert np.allclose(A[0], [[1, h], [0, 1]], atol=1e-15) and np.allclose(B[0], [[h * h / 2], [h]], atol=1e-15)


def test_iiwa14_jacobians_match_finite_differences_of_the_device_step(rng):
    model = gb.Iiwa14()
    X, U, F = _points(model, rng, 8)
    h, eps = 0.02, 1e-6
    A, B = gb.step_jacobians_many(model, X, U, h, F)
    for j in range(14):
        d = np.zeros(14)
        d[j] = eps
        num = (gb.step_many(model, X + d, U, h, F) - gb.step_many(model, X - d, U, h, F)) / (2 * eps)
        assert np.max(np.abs(A[:, :, j] - num)) <= 1e-6 * max(1.0, np.max(np.abs(num)))
    for j in range(7):
        d = np.zeros(7)
        d[j] = eps
        num = (gb.step_many(model, X, U + d, h, F) - gb.step_many(model, X, U - d, h, F)) / (2 * eps)
        assert np.max(np.abs(B[:, :, j] - num)) <= 1e-6 * max(1.0, np.max(np.abs(num)))


def random_block_tridiagonal(rng, nb, bd, spd=True):
    """conftest.random_block_tridiagonal of the reference tests (conftest.py:24-35)."""
    diag = np.empty((nb, bd, bd))
    off = 0.3 * rng.standard_normal((max(nb - 1, 0), bd, bd))
    for i in range(nb):
        W = rng.standard_normal((bd, bd))
        diag[i] = W @ W.T / bd + (3.0 * bd if spd else 0.0) * np.eye(bd)
        diag[i] = 0.5 * (diag[i] + diag[i].T)
    return diag, off


def test_batched_pcg_matches_oracle_and_dense_solve(rng):
    """test_blocktri.py:78-127: random SPD systems, explicit stair preconditioner."""
    for nb, bd in ((5, 2), (9, 4), (33, 14), (1, 3)):
        systems = 6
        Sd, So, Pd, Po, gam = [], [], [], [], []
        for _ in range(systems):
            d, o = random_block_tridiagonal(rng, nb, bd)
            pd, po = orc.stair_preconditioner(d, o)
            Sd.append(d), So.append(o), Pd.append(pd), Po.append(po)
            gam.append(rng.standard_normal(nb * bd))
        lam, its, conv, status, res = gb.pcg_batched(np.stack(Sd), np.stack(So), np.stack(gam), np.stack(Pd),
                                                     np.stack(Po), 1e-10)
        for s in range(systems):
            ref = orc.pcg(Sd[s], So[s], gam[s], Pd[s], Po[s], 1e-10, 10 * nb * bd)
            dense = np.linalg.solve(orc.bt_dense(Sd[s], So[s]), gam[s])
            assert conv[s] and status[s] == 0 and abs(int(its[s]) - ref.iterations) <= 1
            assert rel_inf(lam[s], dense) <= 1e-8 and res[s] <= 1e-10
            assert its[s] <= nb * bd   # finite termination, test_blocktri.py:129-137


def test_pcg_known_answers():
    """test_blocktri.py:61-67 (identity -> 1 iteration), :91-95 (zero rhs -> 0), :104-108
    (breakdown carries the iteration), :153-159 (cap respected)."""
    eye = np.broadcast_to(np.eye(2), (1, 3, 2, 2)).copy()
    off = np.zeros((1, 2, 2, 2))
    gamma = np.arange(1.0, 7.0)[None]
    lam, its, conv, status, _ = gb.pcg_batched(eye, off, gamma, eye, off, 1e-12)
    assert its[0] == 1 and conv[0] and np.allclose(lam[0], gamma[0], atol=1e-12)
    lam, its, conv, status, _ = gb.pcg_batched(eye, off, np.zeros((1, 6)), eye, off, 1e-10)
    assert its[0] == 0 and conv[0] and np.array_equal(lam[0], np.zeros(6))
    Sd = np.array([[[[-1.0]], [[1.0]]]])
    lam, its, conv, status, _ = gb.pcg_batched(Sd, np.zeros((1, 1, 1, 1)), np.array([[1.0, 0.0]]), np.ones((1, 2, 1, 1)),
                                               np.zeros((1, 1, 1, 1)), 1e-8)
    assert status[0] == 2 and its[0] >= 1 and not conv[0]
    rng = np.random.default_rng(5)
    d, o = random_block_tridiagonal(rng, 12, 3)
    ident = np.broadcast_to(np.eye(3), (12, 3, 3)).copy()
    lam, its, conv, status, _ = gb.pcg_batched(d[None], o[None], rng.standard_normal((1, 36)), ident[None],
                                               np.zeros((1, 11, 3, 3)), 1e-14, max_iterations=3)
    assert its[0] == 3 and not conv[0] and status[0] == 0


def test_shift_warm_start_on_device():
    """mpc.shift_warm_start (mpc.py:85-89; test_mpc.py:52-58)."""
    from paper_2510_07625_b200 import workloads
    M, N = 3, 6
    batch = workloads.iiwa14_reach_arrays(M, N)
    rng = np.random.default_rng(9)
    batch.X[...] = rng.standard_normal(batch.X.shape)
    batch.U[...] = rng.standard_normal(batch.U.shape)
    eng = gb.BatchEngine(gb.Iiwa14(), M, N, 0.02, workloads.fixed_budget_settings(1))
    try:
        eng.upload(batch)
        eng.shift_warm_start()
        eng.stream.synchronize()
        X, U = eng.dev["X"].cpu().numpy(), eng.dev["U"].cpu().numpy()
    finally:
        eng.close()
    assert np.array_equal(X, np.concatenate([batch.X[:, 1:], batch.X[:, -1:]], axis=1))
    assert np.array_equal(U, np.concatenate([batch.U[:, 1:], batch.U[:, -1:]], axis=1))


def test_reference_named_blocktri_operators(rng):
    """BlockTriMatrix / btmv / pcg / PcgResult / densify with the reference's signatures and checks
    (blocktri.py:19-173; test_blocktri.py patterns: dense cross-check, identity -> 1 iteration, zero rhs -> 0,
    dimension errors, breakdown on a non-SPD system)."""
    nb, bd = 6, 4
    W = rng.standard_normal((nb, bd, bd))
    diag = W @ W.transpose(0, 2, 1) + 6.0 * np.eye(bd)
    off = 0.3 * rng.standard_normal((nb - 1, bd, bd))
    S = gb.BlockTriMatrix(diag, off)
    v = rng.standard_normal(nb * bd)
    assert rel_inf(gb.btmv(S, v), gb.densify(S) @ v) <= 1e-13
    P = gb.BlockTriMatrix(np.linalg.inv(diag), np.zeros_like(off))          # block-Jacobi preconditioner
    gamma = rng.standard_normal(nb * bd)
    out = gb.pcg(S, gamma, P, gb.PcgSettings(tolerance=1e-10))
    assert isinstance(out, gb.PcgResult) and out.converged and out.final_residual_norm <= 1e-10
    assert rel_inf(out.solution, np.linalg.solve(gb.densify(S), gamma)) <= 1e-9
    eye = gb.BlockTriMatrix.identity(3, 2)
    one = gb.pcg(eye, np.arange(6.0) + 1.0, eye, gb.PcgSettings())
    assert one.iterations == 1 and one.converged
    assert gb.pcg(eye, np.zeros(6), eye, gb.PcgSettings()).iterations == 0
    with pytest.raises(gb.DimensionError):
        gb.btmv(S, np.zeros(3))
    with pytest.raises(gb.DimensionError):
        gb.BlockTriMatrix(diag, off[:-1])
    neg = gb.BlockTriMatrix(-np.tile(np.eye(2), (3, 1, 1)), np.zeros((2, 2, 2)))
    with pytest.raises(gb.PcgBreakdownError) as info:
        gb.pcg(neg, np.ones(6), eye, gb.PcgSettings())
    assert info.value.iteration == 1


def test_scalar_step_and_jacobians_follow_the_reference_contract():
    """dynamics.py:716-772: shape and finiteness checks, force vectors or ExternalForce objects."""
    model = gb.Pendulum()
    x, u = np.array([0.3, -0.2]), np.array([0.5])
    out = gb.step(model, x, u, 0.05)
    A, B = gb.step_jacobians(model, x, u, 0.05, gb.ExternalForce.constant([0.1]))
    assert out.shape == (2,) and A.shape == (2, 2) and B.shape == (2, 1)
    eps = 1e-6
    fd = (gb.step(model, x + [eps, 0], u, 0.05, [0.1]) - gb.step(model, x - [eps, 0], u, 0.05, [0.1])) / (2 * eps)
    assert np.max(np.abs(A[:, 0] - fd)) <= 1e-8
    with pytest.raises(ValueError):
        gb.step(model, np.array([np.nan, 0.0]), np.zeros(1), 0.05)
    with pytest.raises(ValueError):
        gb.step(model, np.zeros(2), np.array([np.inf]), 0.05)
    with pytest.raises(gb.DimensionError):
        gb.step(model, np.zeros(3), np.zeros(1), 0.05)
    with pytest.raises(gb.DimensionError):
        gb.step(model, np.zeros(2), np.zeros(1), 0.05, [0.0, 0.0])
    with pytest.raises(ValueError):
        gb.step(model, np.zeros(2), np.zeros(1), 0.0)


def test_reference_named_merit_and_line_search_operators(rng):
    """sqp.merit / merit_many / constraint_l1 / line_search / adapt_rho with the reference's signatures
    (sqp.py:111-201) and its test patterns: the merit = 7.5 known answer (test_sqp.py:44-53), the L1 term
    includes the initial-state row (test_sqp.py:289-296), non-finite candidates score +inf, batched equals
    single, the candidate set and the strict-decrease rule, the rho clamps (test_sqp.py:165-179)."""
    from oracle import trajopt_np as orc
    # double integrator, N = 2: a trajectory that is feasible except for the start state
    model = gb.DoubleIntegrator(dims=1)
    cost = gb.CostSpec(Q=np.eye(2), R=np.eye(1), QN=np.eye(2), goal=np.zeros(2))
    problem = gb.ProblemSpec(model=model, cost=cost, horizon=2, timestep=0.1, x_start=np.array([1.0, 0.0]))
    X = np.zeros((3, 2))
    U = np.zeros((2, 1))
    assert gb.constraint_l1(problem, X, U) == 1.0                  # only |x_start - x_0|
    assert gb.merit(problem, X, U, 7.5) == 7.5                     # zero cost + mu * 1
    # random cartpole trajectories against the oracle
    cart = gb.ProblemSpec(model=gb.Cartpole(), cost=gb.CostSpec(Q=np.diag([1.0, 2.0, 0.1, 0.1]), R=np.eye(1) * 0.1,
                                                               QN=5.0 * np.eye(4), goal=np.array([0.0, np.pi, 0, 0])),
                          horizon=6, timestep=0.05, x_start=0.1 * rng.standard_normal(4),
                          force=gb.ExternalForce.constant(0.3 * np.ones(gb.Cartpole().force_dim)))
    Xs, Us = 0.3 * rng.standard_normal((5, 7, 4)), 0.3 * rng.standard_normal((5, 6, 1))
    op = orc.Problem.from_spec(cart)
    want = np.array([orc.merit_value(op, Xs[c], Us[c], 10.0) for c in range(5)])
    got = gb.merit_many(cart, Xs, Us, 10.0)
    assert rel_inf(got, want) <= 1e-12
    assert abs(gb.merit(cart, Xs[2], Us[2], 10.0) - got[2]) <= 1e-12 * abs(got[2])
    assert abs(gb.constraint_l1(cart, Xs[1], Us[1]) - orc.violation_l1(op, Xs[1], Us[1])) <= 1e-12
    bad = Xs.copy()
    bad[1, 0, 0] = np.nan
    bad[3, 2, 1] = np.inf
    vals = gb.merit_many(cart, bad, Us, 10.0)
    assert np.isinf(vals[1]) and np.isinf(vals[3]) and rel_inf(vals[[0, 2, 4]], want[[0, 2, 4]]) <= 1e-12
    # line search: candidate set, first minimum, strict decrease
    ls = gb.LineSearchSettings(mu=10.0, beta=2.0, num_shrinks=3)
    assert np.array_equal(ls.candidates(), [1.0, 0.5, 0.25, 0.125])
    dX, dU = 0.2 * rng.standard_normal((7, 4)), 0.2 * rng.standard_normal((6, 1))
    ost = orc.Settings(mu=10.0, beta=2.0, num_shrinks=3)
    a_ref, m_ref, acc_ref, _ = orc.line_search(op, Xs[0], Us[0], dX, dU, ost, orc.merit_value(op, Xs[0], Us[0], 10.0))
    a, m, acc = gb.line_search(cart, Xs[0], Us[0], dX, dU, ls)
    assert a == a_ref and acc == acc_ref and abs(m - m_ref) <= 1e-12 * abs(m_ref)
    a0, m0, acc0 = gb.line_search(cart, Xs[0], Us[0], np.zeros_like(dX), np.zeros_like(dU), ls)
    assert a0 == 1.0 and acc0 is False                            # a zero step never strictly decreases
    st = gb.SolverSettings()
    assert gb.adapt_rho(1e-3, True, st) == 2e-4 and gb.adapt_rho(1e-3, False, st) == 5e-3
    assert gb.adapt_rho(st.rho_min, True, st) == st.rho_min and gb.adapt_rho(st.rho_max, False, st) == st.rho_max
