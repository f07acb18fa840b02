"""PCG breakdown handling on the device (sqp.py:240-248): a non-positive curvature raises rho and
repeats the pass without advancing the solve; more than pcg_retry_limit breakdowns in one
iteration fail the slot with the reference's PcgBreakdownError string.  Problems are badly scaled
on purpose (weights spread over 16 decades, rho ~ 0) so that S is numerically indefinite; the
exact breakdown point is rounding dependent, so the comparison with the oracle is on the retry
semantics, and on the numbers only where both took the same rho path."""

import numpy as np
import pytest

import paper_2510_07625_b200 as gb
from oracle import trajopt_np as orc

pytestmark = pytest.mark.gpu


def badly_scaled(seed):
    rng = np.random.default_rng(seed)
    model = gb.Pendulum() if seed % 2 else gb.TwoLinkArm()
    n, m, N = model.state_dim, model.control_dim, 6
    Q = np.diag(10.0 ** rng.uniform(-14, 2, n))
    R = np.diag(10.0 ** rng.uniform(-14, 2, m))
    QN = np.diag(10.0 ** rng.uniform(-14, 2, n))
    goal = rng.standard_normal(n)
    x_start = rng.standard_normal(n)
    X = rng.standard_normal((N + 1, n))
    U = rng.standard_normal((N, m))
    problem = gb.ProblemSpec(model, gb.CostSpec(Q, R, QN, goal), N, 0.05, x_start)
    return problem, X, U


def oracle_run(problem, X, U, st):
    p = orc.Problem.from_spec(problem)
    ost = orc.Settings(max_sqp_iterations=st.max_sqp_iterations, pcg_tolerance=st.pcg.tolerance, rho_init=st.rho_init,
                       rho_min=st.rho_min, rho_factor=st.rho_factor, step_tolerance=None)
    return orc.solve_batch([p], [(X, U)], [ost])


SEEDS = list(range(0, 40))


def test_breakdown_raises_rho_and_the_solve_recovers():
    """rho_init = 1e-13, factor 1000: a breakdown at iteration 0 shows up as a recorded rho of
    1e-10, 1e-7 or 1e-4 (1..3 retries).  The breakdown point is rounding dependent, so the test asks
    for the semantics over a family of seeds: every slot ends ok or with a well-formed error, at
    least one slot recovered through retries, and wherever the device and the oracle took the same
    rho path the merits agree."""
    st = gb.SolverSettings(max_sqp_iterations=3, step_tolerance=None, rho_init=1e-13, rho_min=0.0, rho_factor=1000.0,
                           pcg=gb.PcgSettings(tolerance=1e-12))
    cases = [badly_scaled(seed) for seed in SEEDS]
    by_model = {}
    for seed, (problem, X, U) in zip(SEEDS, cases):
        by_model.setdefault(problem.model.name, []).append((seed, problem, X, U))
    recovered, compared = 0, 0
    for group in by_model.values():
        out = gb.batch_solve(gb.BatchSpec([g[1] for g in group], [(g[2], g[3]) for g in group], st))
        for (seed, problem, X, U), res, err in zip(group, out.results, out.errors):
            if err is not None:
                assert res is None
                assert err.startswith(("PcgBreakdownError: SQP iteration", "FactorizationError: SQP iteration")), err
                continue
            assert len(res.trace) == 3
            rhos = np.array([r.rho for r in res.trace])
            assert np.all(rhos >= 0.0) and np.all(rhos <= st.rho_max)
            if rhos[0] > 1.5e-13:
                recovered += 1
                # iteration 0 can only have seen rho_init * factor^k, k = 1..3
                assert min(abs(rhos[0] / 1e-13 / 1000.0 ** k - 1.0) for k in (1, 2, 3)) <= 1e-9
            ref, ref_err, _, _ = oracle_run(problem, X, U, st)
            cap = 10 * 7 * problem.model.state_dim
            settled = ref_err[0] is None and all(r.pcg_iterations < cap for r in res.trace) and \
                all(r.pcg_iterations < cap for r in ref[0].trace)
            # where PCG ran into its cap the multipliers are whatever the stagnated iteration left
            if settled and np.allclose(rhos, [r.rho for r in ref[0].trace], rtol=1e-12):
                merits = np.array([r.merit for r in res.trace])
                ref_merits = np.array([r.merit for r in ref[0].trace])
                if np.all(np.isfinite(ref_merits)):
                    compared += 1
                    assert np.max(np.abs(merits - ref_merits)) <= 1e-3 * max(1.0, np.max(np.abs(ref_merits)))
    assert recovered >= 1, "no solve of the family went through a PCG-breakdown retry"
    assert compared >= 1


def test_too_many_breakdowns_fail_the_slot_with_the_reference_message():
    """rho = 0 cannot be raised (0 * factor = 0): a breakdown repeats until the retry limit and the
    slot fails with the reference's message (sqp.py:242-247); neighbours are unaffected."""
    st = gb.SolverSettings(max_sqp_iterations=3, step_tolerance=None, rho_init=0.0, rho_min=0.0,
                           pcg=gb.PcgSettings(tolerance=1e-12))
    failures = 0
    for seed in SEEDS:
        problem, X, U = badly_scaled(seed)
        n, m = problem.model.state_dim, problem.model.control_dim
        good = gb.ProblemSpec(problem.model, gb.CostSpec(np.eye(n), np.eye(m), np.eye(n), np.zeros(n)), 6, 0.05,
                              np.zeros(n))
        zero = (np.zeros_like(X), np.zeros_like(U))
        out = gb.batch_solve(gb.BatchSpec([good, problem, good], [zero, (X, U), zero], st))
        assert out.results[0] is not None and out.results[2] is not None, "neighbours must be unaffected"
        err = out.errors[1]
        if err is not None and err.startswith("PcgBreakdownError"):
            failures += 1
            assert err.startswith("PcgBreakdownError: SQP iteration") and "PCG broke down 4 times (last at inner iteration" in err
            assert out.results[1] is None
            with pytest.raises(gb.PcgBreakdownError) as info:
                gb.sqp_solve(problem, X, U, st)
            assert info.value.iteration >= 1
        if failures >= 3:
            break
    assert failures >= 1, "no badly scaled problem exhausted the retry limit"


@pytest.mark.parametrize("loop_mode", [1, 3])
def test_retried_and_failed_solves_reach_the_host_buffer_whole(monkeypatch, loop_mode):
    """The same badly scaled family through the control-step call (gato_solve_host): with results sent by k_update
    as each solve finishes, a solve that went through PCG-breakdown retries (it stays active across the repeated
    pass) or that exhausted them (frozen by the PCG kernel, not by k_update) must leave the same bytes in the host
    mirror as the copy-engine route."""
    from paper_2510_07625_b200.batch import pack_problems
    from paper_2510_07625_b200.engine import BatchEngine, INPUT_FIELDS
    from paper_2510_07625_b200 import _lib
    st = gb.SolverSettings(max_sqp_iterations=3, step_tolerance=None, rho_init=1e-13, rho_min=0.0, rho_factor=1000.0,
                           pcg=gb.PcgSettings(tolerance=1e-12))
    group = [c for c in (badly_scaled(seed) for seed in SEEDS) if c[0].model.name == "pendulum"]
    problems = [g[0] for g in group]
    packed = pack_problems(problems, [(g[1], g[2]) for g in group], [st.rho_init] * len(group))
    M, N = len(group), problems[0].horizon
    results = []
    for limit in ("0", None):
        if limit is None:
            monkeypatch.delenv("GATO_ZERO_COPY_MAX", raising=False)
        else:
            monkeypatch.setenv("GATO_ZERO_COPY_MAX", limit)
        eng = BatchEngine(problems[0].model, M, N, problems[0].timestep, st, loop_mode=loop_mode)
        try:
            results.append(eng.step(packed, fields=INPUT_FIELDS))
        finally:
            eng.close()
    a, b = results
    for name in ("X", "U", "trace", "info"):
        assert np.array_equal(getattr(a, name), getattr(b, name), equal_nan=True), name
    retried = a.trace[:, 0, _lib.TRACE_RHO] > 1.5e-13
    assert np.any(retried & (a.info[:, _lib.INFO_STATUS] == 0)), "no solve recovered through a retry"
