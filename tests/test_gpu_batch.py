"""Batch semantics on the GPU: the reference's test_batch.py / acceptance #6 expectations
(determinism, position and sharding independence, per-slot failure isolation, mixed rho) and
size-independent properties at the BASELINE.json batch sizes."""

import dataclasses

import numpy as np
import pytest

import paper_2510_07625_b200 as gb
from paper_2510_07625_b200 import _lib, workloads
from paper_2510_07625_b200.batch import pack_problems
from conftest import load_golden, product_problem, product_settings, rel_inf

pytestmark = pytest.mark.gpu


def pendulum_problem(N=16):
    cost = gb.CostSpec(Q=np.diag([1.0, 0.1]), R=np.diag([0.01]), QN=np.diag([100.0, 10.0]),
                       goal=np.array([np.pi, 0.0]))
    return gb.ProblemSpec(model=gb.Pendulum(), cost=cost, horizon=N, timestep=0.05, x_start=np.zeros(2))


def zero_init(p):
    return np.zeros((p.horizon + 1, p.model.state_dim)), np.zeros((p.horizon, p.model.control_dim))


def bitwise_equal(a, b):
    """conftest.results_bitwise_equal of the reference tests (conftest.py:38-55)."""
    if not (np.array_equal(a.X, b.X) and np.array_equal(a.U, b.U)):
        return False
    if a.converged != b.converged or len(a.trace) != len(b.trace):
        return False
    return all(dataclasses.astuple(x) == dataclasses.astuple(y) for x, y in zip(a.trace, b.trace))


def test_copies_of_one_problem_give_identical_results():
    """test_batch.py:32-39."""
    p = pendulum_problem()
    st = gb.SolverSettings(max_sqp_iterations=8, step_tolerance=None)
    out = gb.batch_solve(gb.BatchSpec([p] * 6, [zero_init(p)] * 6, st))
    assert out.ok
    assert all(bitwise_equal(out.results[0], r) for r in out.results[1:])


def test_single_problem_batch_equals_direct_solve():
    """test_batch.py:41-46."""
    p = pendulum_problem()
    st = gb.SolverSettings(max_sqp_iterations=8, step_tolerance=None)
    out = gb.batch_solve(gb.BatchSpec([p], [zero_init(p)], st))
    assert bitwise_equal(out.results[0], gb.sqp_solve(p, *zero_init(p), st))


def test_failed_slot_is_isolated():
    """test_batch.py:59-75: zero cost with rho = 0 cannot be factored; neighbours are unaffected."""
    good = pendulum_problem()
    bad = dataclasses.replace(good, cost=gb.CostSpec(np.zeros((2, 2)), np.zeros((1, 1)), np.zeros((2, 2)),
                                                      np.zeros(2)))
    st = gb.SolverSettings(max_sqp_iterations=3, step_tolerance=None, rho_init=0.0, rho_min=0.0,
                           regularize_r=False)
    out = gb.batch_solve(gb.BatchSpec([good, bad, good], [zero_init(good)] * 3, st))
    assert out.results[0] is not None and out.results[2] is not None and out.results[1] is None
    assert out.errors[1].startswith("FactorizationError: SQP iteration 0: Q_0 is not positive definite")
    assert bitwise_equal(out.results[0], out.results[2])
    alone = gb.batch_solve(gb.BatchSpec([good], [zero_init(good)], st))
    assert bitwise_equal(out.results[0], alone.results[0])
    with pytest.raises(gb.FactorizationError) as info:
        gb.sqp_solve(bad, *zero_init(bad), st)
    assert info.value.knot == 0


def test_singular_control_weight_names_r_block():
    good = pendulum_problem()
    bad = dataclasses.replace(good, cost=gb.CostSpec(np.eye(2), np.zeros((1, 1)), np.eye(2), np.zeros(2)))
    st = gb.SolverSettings(max_sqp_iterations=2, step_tolerance=None, regularize_r=False)
    out = gb.batch_solve(gb.BatchSpec([bad], [zero_init(bad)], st))
    assert out.errors[0].startswith("FactorizationError: SQP iteration 0: R_0 is not positive definite")


def test_mixed_rho_batch_matches_single_solves():
    """test_batch.py:93-106."""
    p = pendulum_problem()
    st = gb.SolverSettings(max_sqp_iterations=6, step_tolerance=None)
    rhos = [1e-6, 1e-3, 1e-1, 1.0]
    out = gb.batch_solve(gb.BatchSpec.with_rho_inits([p] * 4, [zero_init(p)] * 4, st, rhos))
    for rho, res in zip(rhos, out.results):
        single = gb.sqp_solve(p, *zero_init(p), dataclasses.replace(st, rho_init=rho))
        assert bitwise_equal(res, single)


def test_heterogeneous_models_and_settings_are_grouped():
    """batch.py:45-52 only requires equal n, m, N: two models with the same dimensions and a
    per-problem settings override in one batch."""
    a = product_problem(load_golden("twolink_n8"))
    b = product_problem(load_golden("twolink_gravity_n8"))
    ga, gb_ = load_golden("twolink_n8"), load_golden("twolink_gravity_n8")
    st = product_settings(ga)
    longer = dataclasses.replace(st, max_sqp_iterations=9)
    out = gb.batch_solve(gb.BatchSpec([a, b, a], [(ga["X0"], ga["U0"]), (gb_["X0"], gb_["U0"]), (ga["X0"], ga["U0"])],
                                      st, overrides=[None, None, longer]))
    assert out.ok and [len(r.trace) for r in out.results] == [6, 6, 9]
    assert rel_inf(out.results[0].X, ga["X"]) <= 1e-6 and rel_inf(out.results[1].X, gb_["X"]) <= 1e-6


def test_result_is_independent_of_batch_position_and_sharding():
    """Analogue of test_batch.py:48-57 (worker counts): a solve's result is bitwise the same
    alone, inside a batch of 32, and inside either half when the batch is split into shards."""
    M, N, h = 32, 16, 0.02
    batch = workloads.iiwa14_reach_arrays(M, N)
    st = workloads.fixed_budget_settings(3)
    whole = gb.BatchEngine(gb.Iiwa14(), M, N, h, st)
    half = gb.BatchEngine(gb.Iiwa14(), M // 2, N, h, st)
    one = gb.BatchEngine(gb.Iiwa14(), 1, N, h, st)
    try:
        full = whole.solve(batch)
        lo = half.solve(batch.slice(0, M // 2))
        hi = half.solve(batch.slice(M // 2, M))
        assert np.array_equal(np.concatenate([lo.X, hi.X]), full.X)
        assert np.array_equal(np.concatenate([lo.U, hi.U]), full.U)
        assert np.array_equal(np.concatenate([lo.trace, hi.trace]), full.trace, equal_nan=True)
        for b in (0, 13, 31):
            single = one.solve(batch.slice(b, b + 1))
            assert np.array_equal(single.X[0], full.X[b]) and np.array_equal(single.trace[0], full.trace[b], equal_nan=True)
    finally:
        for e in (whole, half, one):
            e.close()


def test_repeated_solves_are_bitwise_deterministic():
    """test_sqp.py:271-276 / test_blocktri.py:139-151."""
    batch = workloads.iiwa14_track_arrays(8, 16, 0.02)
    eng = gb.BatchEngine(gb.Iiwa14(), 8, 16, 0.02, workloads.fixed_budget_settings(3))
    try:
        a, b = eng.solve(batch), eng.solve(batch)
    finally:
        eng.close()
    assert np.array_equal(a.X, b.X) and np.array_equal(a.trace, b.trace, equal_nan=True)


@pytest.mark.parametrize("M,N,h,kind", [(32, 32, 0.02, "track"), (128, 64, 0.05, "reach")])
def test_baseline_size_properties(M, N, h, kind):
    """BASELINE.json configs[1] and configs[2] at full size, through size-independent
    properties: the PCG solution satisfies S lam = gamma to the PCG tolerance (checked on the
    host from the device's own S and gamma), the recovered step satisfies the linearised
    dynamics rows of the KKT system, merits are monotone, and a sample of solves matches the
    oracle within the north-star tolerance."""
    from oracle import trajopt_np as orc
    from oracle.iiwa14_np import Iiwa14
    batch = workloads.iiwa14_track_arrays(M, N, h) if kind == "track" else workloads.iiwa14_reach_arrays(M, N)
    iters = 1 if kind == "track" else 5
    st = workloads.fixed_budget_settings(iters)
    eng = gb.BatchEngine(gb.Iiwa14(), M, N, h, st)
    try:
        one = gb.BatchEngine(gb.Iiwa14(), M, N, h, dataclasses.replace(st, max_sqp_iterations=1), stage_arrays=True)
        try:
            one.solve(batch)
            n, m = 14, 7
            Sd = one.scratch("Sdiag").reshape(M, N + 1, n, n)
            So = one.scratch("Soff").reshape(M, N, n, n)
            gam = one.scratch("gamma").reshape(M, (N + 1) * n)
            lam = one.scratch("lam").reshape(M, (N + 1) * n)
            A = one.scratch("A").reshape(M, N, n, n)
            B = one.scratch("B").reshape(M, N, n, m)
            e = one.scratch("e").reshape(M, N, n)
            dX = one.scratch("dX").reshape(M, N + 1, n)
            dU = one.scratch("dU").reshape(M, N, m)
            its = one.scratch("pcg_iters").reshape(M, -1)[:, 0]
        finally:
            one.close()
        for b in range(0, M, max(1, M // 8)):
            res = orc.bt_matvec(Sd[b], So[b], lam[b]) - gam[b]
            assert np.linalg.norm(res) <= 5e-6, "PCG residual"
            # linearised dynamics: dx_{k+1} - A dx_k - B du_k = e_k ; dx_0 = x_s - x_0
            lin = dX[b, 1:] - np.einsum("kij,kj->ki", A[b], dX[b, :-1]) - np.einsum("kij,kj->ki", B[b], dU[b]) - e[b]
            assert np.max(np.abs(lin)) <= 1e-4 * max(1.0, np.max(np.abs(dX[b])))
            assert np.max(np.abs(dX[b, 0] - (batch.x_start[b] - batch.X[b, 0]))) <= 1e-6
        assert its.min() >= 1 and its.max() <= 200
        full = eng.solve(batch)
        assert np.all(full.info[:, _lib.INFO_STATUS] == 0) and np.all(full.info[:, _lib.INFO_N_RECORDS] == iters)
        merits = full.trace[:, :, _lib.TRACE_MERIT]
        assert np.all(np.diff(merits, axis=1) <= 0)
        ost = orc.Settings(max_sqp_iterations=iters, pcg_tolerance=1e-6, pcg_max_iterations=200, step_tolerance=None)
        # eight solves spread over the batch DIRECTLY against the numpy oracle (bitwise the reference), in a pool
        import os
        rows = sorted(set(int(r) for r in np.linspace(0, M - 1, 8)))
        probs = [orc.Problem(Iiwa14(), batch.Q[b], batch.R[b], batch.QN[b], batch.goal[b], N, h, batch.x_start[b],
                             batch.force[b]) for b in rows]
        refs, errs, _ = orc.solve_batch_parallel(probs, [(batch.X[b], batch.U[b]) for b in rows], [ost] * len(rows),
                                                 min(len(rows), os.cpu_count() or 1))
        assert all(e is None for e in errs)
        for b, ref in zip(rows, refs):
            assert rel_inf(full.X[b], ref.X) <= 1e-4 and rel_inf(full.U[b], ref.U) <= 1e-4
            assert rel_inf(full.X[b], ref.X) <= 1e-7, "measured: 1e-9 .. 1e-13"
            pcg_ref = np.array([r.pcg_iterations for r in ref.trace])
            assert np.max(np.abs(full.trace[b, :, _lib.TRACE_PCG_ITERATIONS] - pcg_ref)) <= 1
            assert np.array_equal(full.trace[b, :, _lib.TRACE_ALPHA], np.array([r.alpha for r in ref.trace]))
    finally:
        eng.close()


@pytest.mark.parametrize("M,N,h,kind", [(32, 32, 0.02, "track"), (128, 64, 0.05, "reach"), (256, 16, 0.02, "reach"),
                                          (1024, 64, 0.05, "reach")])
def test_every_solve_of_the_baseline_batches_matches_the_compiled_oracle(M, N, h, kind):
    """BASELINE.json configs[1], configs[2] and the per-GPU shard of configs[4] at full size, EVERY solve: the compiled C restatement
    (oracle/trajopt_c.c, itself checked against the bitwise-pinned numpy oracle in tests/test_oracle_c.py)
    is fast enough to serve as the checker for whole batches.  Trajectories within 1e-6 relative (the
    north-star bar is 1e-4), identical SQP iteration counts, PCG counts within +-1, identical step
    lengths and accept decisions."""
    from oracle import trajopt_c as oc
    from oracle import trajopt_np as orc
    batch = workloads.iiwa14_track_arrays(M, N, h) if kind == "track" else workloads.iiwa14_reach_arrays(M, N)
    iters = 1 if kind == "track" else 5
    st = workloads.fixed_budget_settings(iters)
    eng = gb.BatchEngine(gb.Iiwa14(), M, N, h, st)
    try:
        got = eng.solve(batch)
    finally:
        eng.close()
    ost = orc.Settings(max_sqp_iterations=iters, pcg_tolerance=1e-6, pcg_max_iterations=200, step_tolerance=None)
    X, U, trace, info = oc.solve_batch(batch.x_start, batch.goal, batch.Q, batch.R, batch.QN, batch.force,
                                       batch.rho_init, batch.X, batch.U, h, ost)
    assert np.all(info[:, 2] == 0) and np.all(got.info[:, _lib.INFO_STATUS] == 0)
    assert np.array_equal(got.info[:, _lib.INFO_N_RECORDS], info[:, 0])
    worst = max(max(rel_inf(got.X[b], X[b]), rel_inf(got.U[b], U[b])) for b in range(M))
    assert worst <= 1e-6, f"worst trajectory error over {M} solves: {worst:.3e}"
    assert np.max(np.abs(got.trace[:, :, _lib.TRACE_PCG_ITERATIONS] - trace[:, :, 4])) <= 1
    assert np.array_equal(got.trace[:, :, _lib.TRACE_ALPHA], trace[:, :, 2])
    assert np.array_equal(got.trace[:, :, _lib.TRACE_ACCEPTED], trace[:, :, 5])
    assert rel_inf(got.trace[:, :, _lib.TRACE_MERIT], trace[:, :, 0]) <= 1e-8


def test_more_configurations_than_the_engine_cache_holds():
    """batch_solve with more homogeneous groups (here: 20 timesteps) than the engine cache has slots (16): eviction
    is least-recently-used and never closes an engine the running call still has work on (the old
    popitem() closed the newest engine and lost the batch)."""
    import dataclasses as dc
    from paper_2510_07625_b200 import batch as gbatch
    gbatch.clear_engine_cache()
    cost = gb.CostSpec(Q=np.diag([1.0, 0.1]), R=np.diag([0.01]), QN=np.diag([100.0, 10.0]), goal=np.array([np.pi, 0.0]))
    base = gb.ProblemSpec(model=gb.Pendulum(), cost=cost, horizon=8, timestep=0.05, x_start=np.zeros(2))
    problems = [dc.replace(base, timestep=0.03 + 0.002 * i) for i in range(20)]
    zero = (np.zeros((9, 2)), np.zeros((8, 1)))
    st = gb.SolverSettings(max_sqp_iterations=3, step_tolerance=None)
    out = gb.batch_solve(gb.BatchSpec(problems, [zero] * 20, st))
    assert out.ok and all(r is not None and len(r.trace) == 3 for r in out.results)
    for i in (0, 7, 19):      # each slot equals its single solve
        single = gb.sqp_solve(problems[i], *zero, st)
        assert np.array_equal(single.X, out.results[i].X)
    assert len(gbatch._ENGINES) <= 20
    again = gb.batch_solve(gb.BatchSpec(problems[:4], [zero] * 4, st))     # after the call the cache shrinks on demand
    assert again.ok and len(gbatch._ENGINES) <= 20
    gbatch.clear_engine_cache()


def test_a_problem_that_cannot_be_packed_fails_alone():
    """batch.py:92-99: an exception raised for one problem (here: an initial trajectory of the wrong size and a
    force of the wrong dimension) is that slot's error string; the rest of the batch is solved."""
    cost = gb.CostSpec(Q=np.diag([1.0, 0.1]), R=np.diag([0.01]), QN=np.diag([100.0, 10.0]), goal=np.array([np.pi, 0.0]))
    good = gb.ProblemSpec(model=gb.Pendulum(), cost=cost, horizon=8, timestep=0.05, x_start=np.zeros(2))
    zero = (np.zeros((9, 2)), np.zeros((8, 1)))
    bad_init = (np.zeros((7, 2)), np.zeros((8, 1)))
    st = gb.SolverSettings(max_sqp_iterations=3, step_tolerance=None)
    out = gb.batch_solve(gb.BatchSpec([good, good, good], [zero, bad_init, zero], st))
    assert out.results[0] is not None and out.results[2] is not None and out.results[1] is None
    assert out.errors[0] is None and out.errors[2] is None
    assert out.errors[1].startswith("ValueError: cannot reshape array of size 14 into shape (9,2)")
    assert np.array_equal(out.results[0].X, out.results[2].X)
    gb.batch.clear_engine_cache()
