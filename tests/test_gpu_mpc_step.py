"""The caller-side rows of the hot path on the GPU: one control step through
a single C-ABI call (gato_solve_host), best-of-batch selection on the device (mpc.py:283-298) and the
reference's bench_scaling protocol (batch.py:127-169)."""

import numpy as np
import pytest

import paper_2510_07625_b200 as gb
from paper_2510_07625_b200 import _lib, mpc, workloads
from paper_2510_07625_b200.engine import INPUT_FIELDS

pytestmark = pytest.mark.gpu


def test_step_is_bitwise_the_staged_solve():
    M, N = 6, 12
    batch = workloads.iiwa14_reach_arrays(M, N)
    st = workloads.fixed_budget_settings(2)
    eng = gb.BatchEngine(gb.Iiwa14(), M, N, 0.02, st)
    try:
        staged = eng.solve(batch)
        fused = eng.step(batch, fields=INPUT_FIELDS)
        view = eng.step(batch, fields=INPUT_FIELDS, copy=False)
        assert view.X.base is not None     # a view of the pinned mirror, not a copy
    finally:
        eng.close()
    for name in ("X", "U", "trace", "info"):
        assert np.array_equal(getattr(staged, name), getattr(fused, name), equal_nan=name == "trace"), name
        assert np.array_equal(getattr(staged, name), getattr(view, name), equal_nan=name == "trace"), name


def test_mpc_step_with_device_shift_matches_host_shift():
    """upload(x_start, goal, force) + device shift + solve in one call == the same control step
    assembled on the host with mpc.shift_warm_start (mpc.py:85-89)."""
    M, N = 4, 10
    batch = workloads.iiwa14_reach_arrays(M, N)
    st = workloads.fixed_budget_settings(1)
    eng = gb.BatchEngine(gb.Iiwa14(), M, N, 0.02, st)
    try:
        first = eng.solve(batch)
        nxt = gb.PackedBatch(first.X[:, 1, :].copy(), batch.goal, batch.Q, batch.R, batch.QN, batch.force,
                             batch.rho_init, batch.X, batch.U)
        stepped = eng.step(nxt, shift=True)            # X, U stay on the device and are shifted there
        Xs = np.concatenate([first.X[:, 1:], first.X[:, -1:]], axis=1)
        Us = np.concatenate([first.U[:, 1:], first.U[:, -1:]], axis=1)
        host = eng.solve(gb.PackedBatch(nxt.x_start, batch.goal, batch.Q, batch.R, batch.QN, batch.force,
                                        batch.rho_init, Xs, Us))
    finally:
        eng.close()
    assert np.array_equal(stepped.X, host.X) and np.array_equal(stepped.U, host.U)
    assert np.array_equal(stepped.trace, host.trace, equal_nan=True)


def test_step_rejects_scattered_fields():
    M, N = 2, 4
    batch = workloads.iiwa14_reach_arrays(M, N)
    eng = gb.BatchEngine(gb.Iiwa14(), M, N, 0.02, workloads.fixed_budget_settings(1))
    try:
        with pytest.raises(ValueError):
            eng.step(batch, fields=("x_start", "Q"))
    finally:
        eng.close()


def test_best_of_batch_on_device_matches_the_host_rule():
    """Nested rho grid (mpc.py:61-78) over copies of one problem: the device argmin picks what
    mpc.best_of_batch picks from the unpacked results, and a failed slot is skipped."""
    from paper_2510_07625_b200.batch import pack_problems, unpack_results
    N = 16
    cost = gb.CostSpec(Q=np.diag([1.0, 0.1]), R=np.diag([0.01]), QN=np.diag([100.0, 10.0]),
                       goal=np.array([np.pi, 0.0]))
    problem = gb.ProblemSpec(model=gb.Pendulum(), cost=cost, horizon=N, timestep=0.05, x_start=np.zeros(2))
    bad = gb.ProblemSpec(model=gb.Pendulum(), cost=gb.CostSpec(Q=-100.0 * np.eye(2), R=np.diag([0.01]), QN=np.eye(2),
                                                               goal=np.array([np.pi, 0.0])),
                         horizon=N, timestep=0.05, x_start=np.zeros(2))
    M = 9
    rhos = mpc.rho_grid(M)
    problems = [problem] * (M - 1) + [bad]
    inits = [(np.zeros((N + 1, 2)), np.zeros((N, 1)))] * M
    st = gb.SolverSettings(max_sqp_iterations=6, step_tolerance=None)
    eng = gb.BatchEngine(gb.Pendulum(), M, N, 0.05, st)
    try:
        res = eng.solve(pack_problems(problems, inits, list(rhos)))
        idx, merit = eng.best_of_batch()
    finally:
        eng.close()
    results, errors = unpack_results(res)
    assert errors[-1] is not None and "FactorizationError" in errors[-1]
    want = mpc.best_of_batch(results)
    assert idx == want and idx != M - 1
    assert merit == results[want].final_merit


def test_bench_scaling_rows_follow_the_reference_schema():
    cost = gb.CostSpec(Q=np.eye(2), R=0.1 * np.eye(1), QN=10.0 * np.eye(2), goal=np.array([np.pi, 0.0]))
    template = gb.ProblemSpec(model=gb.Pendulum(), cost=cost, horizon=8, timestep=0.05, x_start=np.zeros(2))
    rows = gb.bench_scaling(template, [1, 4], [8, 16], workers=1, repeats=3, budget_iterations=2)
    assert [(r["M"], r["N"]) for r in rows] == [(1, 8), (4, 8), (1, 16), (4, 16)]     # N outer, M inner
    for r in rows:
        assert list(r)[:5] == ["M", "N", "median_ms", "p90_ms", "workers"]             # batch.py:161-167
        assert r["p90_ms"] >= r["median_ms"] > 0 and r["workers"] == 1
        assert r["device_ms"] > 0 and r["solve_iterations_per_s"] > 0
    with pytest.raises(ValueError):
        gb.bench_scaling(gb.ProblemSpec(model=gb.Pendulum(), cost=gb.CostSpec(
            Q=np.eye(2), R=0.1 * np.eye(1), QN=np.eye(2), goal=np.zeros((9, 2))), horizon=8, timestep=0.05,
            x_start=np.zeros(2)), [1], [8])


@pytest.mark.parametrize("model_name", ["two_link_arm", "iiwa14", "pendulum"])
@pytest.mark.parametrize("position_only", [False, True])
def test_select_hypothesis_matches_the_plant_rollout(model_name, position_only):
    """mpc.select_hypothesis (mpc.py:130-147): every candidate force rolls the plant over one control
    period in RK4 substeps (dynamics.py:843-864); distances and the chosen index against the oracle's
    row-wise RK4 applied substep by substep."""
    from oracle import trajopt_np as orc
    rng = np.random.default_rng(31)
    model = {"two_link_arm": gb.TwoLinkArm(), "iiwa14": gb.Iiwa14(), "pendulum": gb.Pendulum()}[model_name]
    omodel = orc.model_from_descriptor(model)
    n, m, fd = model.state_dim, model.control_dim, model.force_dim
    M, period, h_plant = 37, 0.01, 0.001
    x_prev = 0.3 * rng.standard_normal(n)
    u = 0.5 * rng.standard_normal(m)
    forces = np.stack([c.value for c in mpc.sample_hypotheses(np.zeros(fd), 2.0, M, seed=5)])
    truth = 11                                    # the measurement comes from candidate 11's force
    X = np.tile(x_prev, (M, 1))
    for _ in range(10):
        X = orc.rk4_rows(omodel, X, np.tile(u, (M, 1)), h_plant, forces)
    x_meas = X[truth] + 1e-9 * rng.standard_normal(n)
    sel = slice(0, n // 2) if position_only else slice(None)
    want = np.linalg.norm((X - x_meas)[:, sel], axis=1)
    idx, err = gb.select_hypothesis(model, x_prev, u, x_meas, forces, period, h_plant, position_only,
                                    return_errors=True)
    # one-dimensional force channels only have the two candidates center -+ sigma: ties go to the first
    assert idx == int(np.argmin(want)) and np.array_equal(forces[idx], forces[truth])
    assert np.max(np.abs(err - want)) <= 1e-11 * max(1.0, want.max())
    with pytest.raises(ValueError):
        gb.select_hypothesis(model, x_prev, u, x_meas, forces, 0.0105, h_plant)


def test_mpc_advance_is_the_three_host_steps_in_one_kernel():
    """gato_mpc_advance: x_start <- X[:, 1], shift (mpc.py:85-89), goal window advanced along a path
    (shared or per solve, clamped at its end) -- against numpy on the downloaded buffers."""
    import torch
    M, N = 5, 9
    batch = workloads.iiwa14_reach_arrays(M, N)
    eng = gb.BatchEngine(gb.Iiwa14(), M, N, 0.02, workloads.fixed_budget_settings(1))
    rng = np.random.default_rng(2)
    try:
        first = eng.solve(batch)
        path = rng.standard_normal((N + 4, 14))
        eng.mpc_advance(torch.as_tensor(path, device="cuda"), step=2)
        eng.stream.synchronize()
        X, U = eng.dev["X"].cpu().numpy(), eng.dev["U"].cpu().numpy()
        assert np.array_equal(eng.dev["x_start"].cpu().numpy(), first.X[:, 1])
        assert np.array_equal(X, np.concatenate([first.X[:, 1:], first.X[:, -1:]], axis=1))
        assert np.array_equal(U, np.concatenate([first.U[:, 1:], first.U[:, -1:]], axis=1))
        rows = np.minimum(2 + np.arange(N + 1), len(path) - 1)          # clamped at the end of the path
        assert np.array_equal(eng.dev["goal"].cpu().numpy(), np.broadcast_to(path[rows], (M, N + 1, 14)))
        per_solve = rng.standard_normal((M, N + 6, 14))
        eng.mpc_advance(torch.as_tensor(per_solve, device="cuda"), step=0)
        eng.stream.synchronize()
        assert np.array_equal(eng.dev["goal"].cpu().numpy(), per_solve[:, :N + 1])
        goal_before = eng.dev["goal"].clone()
        eng.mpc_advance()                                                # no path: goals untouched
        eng.stream.synchronize()
        assert torch.equal(eng.dev["goal"], goal_before)
        with pytest.raises(ValueError):
            eng.mpc_advance(torch.zeros((3, 7), device="cuda", dtype=torch.float64))
    finally:
        eng.close()


@pytest.mark.parametrize("loop_mode", [0, 3])
def test_fused_control_step_equals_advance_then_solve(loop_mode):
    """gato_solve_mpc (BatchEngine.mpc_step): the control step's state hand-over, shift and goal window ride in the
    first kernel of the solve.  Over several consecutive control steps it must leave exactly what
    gato_mpc_advance followed by gato_solve leaves (graph loop mode: the first node's arguments are patched per
    launch; stream loop mode: passed directly)."""
    import torch
    M, N, h = 5, 12, 0.02
    batch = workloads.iiwa14_track_arrays(M, N, h)
    st = workloads.fixed_budget_settings(1)
    rng = np.random.default_rng(3)
    path = torch.as_tensor(np.cumsum(0.01 * rng.standard_normal((40, 14)), axis=0), device="cuda")
    a = gb.BatchEngine(gb.Iiwa14(), M, N, h, st, loop_mode=loop_mode)
    b = gb.BatchEngine(gb.Iiwa14(), M, N, h, st, loop_mode=loop_mode)
    try:
        a.upload(batch)
        b.upload(batch)
        for e in (a, b):
            e.launch()
            e.finish()
        for s in range(4):
            a.mpc_advance(path, s)
            a.launch()
            a.finish()
            b.mpc_step(path, s)
            b.finish()
            ra, rb = a.download(), b.download()
            assert np.array_equal(ra.X, rb.X) and np.array_equal(ra.U, rb.U), f"control step {s}"
            assert np.array_equal(ra.trace, rb.trace, equal_nan=True) and np.array_equal(ra.info, rb.info)
            assert torch.equal(a.dev["goal"], b.dev["goal"]) and torch.equal(a.dev["x_start"], b.dev["x_start"])
        assert b.launch_count() == a.launch_count()
    finally:
        a.close()
        b.close()


def _engine_with_env(monkeypatch, zero_copy_max, *args, **kwargs):
    if zero_copy_max is None:
        monkeypatch.delenv("GATO_ZERO_COPY_MAX", raising=False)
    else:
        monkeypatch.setenv("GATO_ZERO_COPY_MAX", str(zero_copy_max))
    return gb.BatchEngine(*args, **kwargs)     # the limit is read in gato_create


@pytest.mark.parametrize("loop_mode", [1, 3])
def test_host_step_moved_by_kernels_equals_the_copy_engine_path(monkeypatch, loop_mode):
    """gato_solve_host in the latency regime: inputs read from the pinned host buffer by the solve's first kernel,
    results sent by k_update as each solve finishes.  Same bytes in the host mirror as with cudaMemcpyAsync on both
    sides -- over consecutive control steps, with solves that finish in different passes (tolerance mode) and one
    that fails (its rows are sent by the pass that froze it)."""
    M, N, h = 6, 12, 0.02
    batch = workloads.iiwa14_track_arrays(M, N, h)
    batch.Q[4] = -batch.Q[4]                              # FactorizationError: Q_0 not positive definite
    batch.goal[2] = batch.X[2]                            # already at the goal: exits at once
    st = gb.SolverSettings(max_sqp_iterations=6)          # tolerance mode, early exits
    a = _engine_with_env(monkeypatch, 0, gb.Iiwa14(), M, N, h, st, loop_mode=loop_mode)
    b = _engine_with_env(monkeypatch, None, gb.Iiwa14(), M, N, h, st, loop_mode=loop_mode)
    try:
        ra = a.step(batch, fields=INPUT_FIELDS)
        rb = b.step(batch, fields=INPUT_FIELDS)
        for s in range(3):
            for name in ("X", "U", "trace", "info"):
                assert np.array_equal(getattr(ra, name), getattr(rb, name), equal_nan=True), (s, name)
            assert ra.info[4, _lib.INFO_STATUS] != 0 and np.any(ra.info[:, _lib.INFO_N_RECORDS] < 6)
            nxt = gb.PackedBatch(ra.X[:, 1, :].copy(), batch.goal + 0.01 * (s + 1), batch.Q, batch.R, batch.QN,
                                 batch.force, batch.rho_init, batch.X, batch.U)
            ra = a.step(nxt, shift=True)
            rb = b.step(nxt, shift=True)
        # the device copies agree with what was sent
        down = b.download()
        assert np.array_equal(down.X, rb.X) and np.array_equal(down.trace, rb.trace, equal_nan=True)
        assert np.array_equal(down.info, rb.info)
    finally:
        a.close()
        b.close()


def test_host_step_with_a_span_that_is_not_only_results_or_not_pinned(monkeypatch):
    """Fallbacks of the same call: a result span that also covers input arrays goes through the copy kernel
    (k_copy_words), pageable host memory through cudaMemcpyAsync -- same bytes either way."""
    import ctypes as C
    M, N, h = 3, 8, 0.02
    batch = workloads.iiwa14_reach_arrays(M, N)
    st = workloads.fixed_budget_settings(2)
    eng = _engine_with_env(monkeypatch, None, gb.Iiwa14(), M, N, h, st)
    try:
        ref = eng.solve(batch)
        eng.upload(batch)
        eng.stream.synchronize()
        cin, cout = eng._span("x_start", "force"), eng._span("rho_init", "info")   # rho_init, X, U, trace, info
        base_d = eng.arena.data_ptr()

        def call(host_base):
            eng._check(eng.lib.gato_solve_host(
                eng.handle, C.c_void_p(eng.stream.cuda_stream),
                C.c_void_p(base_d + 8 * cin.start), C.c_void_p(host_base + 8 * cin.start), 8 * (cin.stop - cin.start), 0,
                C.c_void_p(base_d + 8 * cout.start), C.c_void_p(host_base + 8 * cout.start),
                8 * (cout.stop - cout.start)), "gato_solve_host")

        eng.pinned.zero_()
        for name in ("x_start", "goal", "force"):
            eng.pin_np[name][...] = getattr(batch, name)
        call(eng.pinned.data_ptr())
        for name in ("X", "U", "trace", "info"):
            assert np.array_equal(eng.pin_np[name], getattr(ref, name), equal_nan=True), name
        assert np.array_equal(eng.pin_np["rho_init"], batch.rho_init)
        pageable = np.zeros(eng.arena_doubles)
        for name in ("x_start", "goal", "force"):
            o, c = eng.offsets[name]
            pageable[o:o + c] = np.asarray(getattr(batch, name)).reshape(-1)
        eng.upload(batch)
        eng.stream.synchronize()
        call(pageable.ctypes.data)
        o, c = eng.offsets["X"]
        assert np.array_equal(pageable[o:o + c].reshape(ref.X.shape), ref.X)
        o, c = eng.offsets["trace"]
        assert np.array_equal(pageable[o:o + c].reshape(ref.trace.shape), ref.trace, equal_nan=True)
    finally:
        eng.close()


def test_step_from_a_separate_input_mirror_repeats_bitwise():
    """step(mirror=): the inputs (cold iterate included) come from a second pinned buffer, so the same problem batch
    can be solved again and again although every step's results overwrite X and U of the engine's own mirror."""
    M, N = 5, 10
    batch = workloads.iiwa14_reach_arrays(M, N)
    eng = gb.BatchEngine(gb.Iiwa14(), M, N, 0.02, workloads.fixed_budget_settings(2))
    try:
        ref = eng.solve(batch)
        mirror = eng.input_mirror()
        mirror.write(batch)
        for _ in range(3):
            out = eng.step(None, fields=INPUT_FIELDS, mirror=mirror)
            assert np.array_equal(out.X, ref.X) and np.array_equal(out.U, ref.U)
            assert np.array_equal(out.trace, ref.trace, equal_nan=True) and np.array_equal(out.info, ref.info)
        assert np.array_equal(mirror.arrays["X"], batch.X)      # untouched by the results
    finally:
        eng.close()


def test_bound_step_is_the_step_call():
    M, N = 4, 10
    batch = workloads.iiwa14_reach_arrays(M, N)
    st = workloads.fixed_budget_settings(1)
    a = gb.BatchEngine(gb.Iiwa14(), M, N, 0.02, st)
    b = gb.BatchEngine(gb.Iiwa14(), M, N, 0.02, st)
    try:
        for e in (a, b):
            e.solve(batch)
        call = b.bind_step(shift=True)
        for s in range(3):
            for e in (a, b):
                e.host_inputs()["goal"][...] = batch.goal + 0.01 * (s + 1)
            ra = a.step(None, shift=True)
            rb = call()
            assert np.array_equal(ra.X, rb.X) and np.array_equal(ra.trace, rb.trace, equal_nan=True)
        with pytest.raises(ValueError):
            b.bind_step(fields=("x_start", "Q"))
    finally:
        a.close()
        b.close()
