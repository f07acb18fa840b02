"""Host-side mirror of the reference's batch API: types, validation, packing, error strings,
and the C-ABI library's exported surface.  No GPU compute here."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2510_07625_b200 as gb
from paper_2510_07625_b200 import _lib, batch, workloads
from conftest import ROOT, load_golden, product_problem, product_settings


def pendulum_problem(N=16):
    cost = gb.CostSpec(Q=np.diag([1.0, 0.1]), R=np.diag([0.01]), QN=np.diag([100.0, 10.0]),
                       goal=np.array([np.pi, 0.0]))
    return gb.ProblemSpec(model=gb.Pendulum(), cost=cost, horizon=N, timestep=0.05, x_start=np.zeros(2))


def zero_init(p):
    return np.zeros((p.horizon + 1, p.model.state_dim)), np.zeros((p.horizon, p.model.control_dim))


class TestLibrary:
    def test_library_exports_every_declared_symbol(self):
        header = (ROOT / "include" / "gato_b200.h").read_text()
        declared = set(re.findall(r"\b(gato_[a-z_0-9]+)\s*\(", header))
        declared -= {"gato_handle"}
        lib = _lib.load()
        for name in sorted(declared):
            assert hasattr(lib, name), f"{name} declared in include/gato_b200.h but not exported"
        assert declared == set(_lib.EXPORTS), "ctypes table and header disagree"
        assert b"sm_100a" in lib.gato_version()

    def test_struct_layouts_match_the_header(self):
        # 14 int32 + 9 double + 8 double; 11 pointers
        assert ctypes.sizeof(_lib.GatoConfig) == 14 * 4 + 17 * 8
        assert ctypes.sizeof(_lib.GatoBuffers) == 11 * 8

    def test_invalid_config_is_rejected_without_a_gpu(self):
        lib = _lib.load()
        handle = ctypes.c_void_p()
        cfg = _lib.GatoConfig()
        cfg.abi_version = 999
        assert lib.gato_create(ctypes.byref(cfg), ctypes.byref(handle)) == -1

    def test_no_cuda_device_fails_loudly(self):
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
        p = pendulum_problem()
        with pytest.raises(gb.BackendUnavailableError):
            gb.batch_solve(gb.BatchSpec([p], [zero_init(p)], gb.SolverSettings()))
        with pytest.raises(gb.BackendUnavailableError):
            gb.step_many(gb.Pendulum(), np.zeros((1, 2)), np.zeros((1, 1)), 0.1, np.zeros((1, 1)))

    def test_product_package_never_imports_the_oracle(self):
        for path in (ROOT / "paper_2510_07625_b200").rglob("*.py"):
            text = path.read_text()
            assert "import oracle" not in text and "from oracle" not in text, path


class TestValidation:
    """Eager validation with the reference's exception types (batch.py:38-52, qpform.py:92-111,
    sqp.py:71-77, blocktri.py:72-76)."""

    def test_batch_spec_checks(self):
        p = pendulum_problem()
        with pytest.raises(ValueError):
            gb.BatchSpec([], [], gb.SolverSettings())
        with pytest.raises(ValueError):
            gb.BatchSpec([p, p], [zero_init(p)], gb.SolverSettings())
        with pytest.raises(ValueError):
            gb.BatchSpec([p], [zero_init(p)], gb.SolverSettings(), overrides=[None, None])
        with pytest.raises(ValueError):   # heterogeneous horizon, test_batch.py:108-113
            gb.BatchSpec([p, pendulum_problem(8)], [zero_init(p)] * 2, gb.SolverSettings())

    def test_problem_spec_checks(self):
        cost = gb.CostSpec(np.eye(2), np.eye(1), np.eye(2), np.zeros(2))
        with pytest.raises(ValueError):
            gb.ProblemSpec(gb.Pendulum(), cost, 0, 0.1, np.zeros(2))
        with pytest.raises(ValueError):
            gb.ProblemSpec(gb.Pendulum(), cost, 4, -0.1, np.zeros(2))
        with pytest.raises(gb.DimensionError):
            gb.ProblemSpec(gb.Pendulum(), cost, 4, 0.1, np.zeros(3))
        with pytest.raises(gb.DimensionError):
            gb.ProblemSpec(gb.Cartpole(), cost, 4, 0.1, np.zeros(4))
        with pytest.raises(gb.DimensionError):
            gb.ProblemSpec(gb.Pendulum(), gb.CostSpec(np.eye(2), np.eye(1), np.eye(2), np.zeros((3, 2))), 4, 0.1,
                           np.zeros(2))
        with pytest.raises(ValueError):
            gb.CostSpec(np.array([[1.0, 2.0], [0.0, 1.0]]), np.eye(1), np.eye(2), np.zeros(2))

    def test_settings_checks(self):
        with pytest.raises(ValueError):
            gb.SolverSettings(rho_init=1e2)
        with pytest.raises(ValueError):
            gb.SolverSettings(rho_factor=1.0)
        with pytest.raises(ValueError):
            gb.SolverSettings(max_sqp_iterations=0)
        with pytest.raises(ValueError):
            gb.LineSearchSettings(beta=1.0)
        with pytest.raises(ValueError):
            gb.PcgSettings(tolerance=-1.0)
        assert gb.PcgSettings().iteration_cap(40) == 400
        assert np.array_equal(gb.LineSearchSettings(num_shrinks=3).candidates(), [1.0, 0.5, 0.25, 0.125])

    def test_workers_must_be_positive(self):
        p = pendulum_problem()
        with pytest.raises(ValueError):
            gb.batch_solve(gb.BatchSpec([p], [zero_init(p)], gb.SolverSettings()), workers=0)


class TestPacking:
    def test_pack_broadcasts_goals_and_constant_forces(self):
        g = load_golden("iiwa14_reach_n8_b0")
        p = product_problem(g)
        packed = batch.pack_problems([p, p], [(g["X0"], g["U0"])] * 2, [1e-4, 1e-2])
        assert packed.goal.shape == (2, 9, 14) and np.array_equal(packed.goal[1], g["goal"])
        assert packed.force.shape == (2, 8, 3) and np.array_equal(packed.rho_init, [1e-4, 1e-2])
        assert packed.X.flags.c_contiguous and packed.Q.dtype == np.float64

    def test_time_varying_force_sampled_at_knot_start_times(self):
        profile = lambda t: np.array([t, 2.0 * t])  # noqa: E731
        cost = gb.CostSpec(np.eye(4), np.eye(2), np.eye(4), np.zeros(4))
        p = gb.ProblemSpec(gb.TwoLinkArm(), cost, 5, 0.1, np.zeros(4), gb.ExternalForce.time_varying(profile, 2))
        rows = batch._force_rows(p)
        assert np.allclose(rows[:, 0], 0.1 * np.arange(5)) and np.allclose(rows[:, 1], 0.2 * np.arange(5))
        assert np.array_equal(rows, p.force_matrix())

    def test_with_rho_inits_builds_overrides(self):
        p = pendulum_problem()
        spec = gb.BatchSpec.with_rho_inits([p] * 3, [zero_init(p)] * 3, gb.SolverSettings(), [1e-6, 1e-3, 1.0])
        assert [spec.effective_settings(i).rho_init for i in range(3)] == [1e-6, 1e-3, 1.0]

    def test_shard_bounds_partition_the_batch(self):
        for M in (1, 7, 32, 1000):
            for G in (1, 2, 3, 8):
                b = gb.shard_bounds(M, G)
                assert b[0][0] == 0 and b[-1][1] == M
                assert all(b[i][1] == b[i + 1][0] for i in range(G - 1))
                sizes = [hi - lo for lo, hi in b]
                assert max(sizes) - min(sizes) <= 1

    def test_error_rendering_matches_reference_strings(self):
        info = np.zeros(8, dtype=np.int32)
        assert batch.render_error(info) is None
        info[[_lib.INFO_STATUS, _lib.INFO_FAIL_ITER, _lib.INFO_FAIL_KNOT, _lib.INFO_FAIL_BLOCK,
              _lib.INFO_FAIL_AUX]] = [1, 2, 0, _lib.BLOCK_Q, 1]
        assert batch.render_error(info).startswith("FactorizationError: SQP iteration 2: Q_0 is not positive definite")
        info[[_lib.INFO_FAIL_KNOT, _lib.INFO_FAIL_BLOCK]] = [5, _lib.BLOCK_S]
        assert "S diagonal block 5 is not positive definite" in batch.render_error(info)
        info[[_lib.INFO_STATUS, _lib.INFO_FAIL_AUX, _lib.INFO_RETRIES]] = [2, 7, 4]
        assert batch.render_error(info) == ("PcgBreakdownError: SQP iteration 2: PCG broke down 4 times "
                                            "(last at inner iteration 7)")

    def test_unpack_results_builds_reference_shaped_objects(self):
        M, it = 2, 3
        trace = np.zeros((M, it, 8))
        trace[0, :2] = [[1.5, 0.1, 0.5, 1e-4, 9, 1, 0.3, 0], [1.2, 0.0, np.nan, 2e-5, 9, 0, 1e-7, 1]]
        info = np.zeros((M, 8), dtype=np.int32)
        info[0, [_lib.INFO_N_RECORDS, _lib.INFO_CONVERGED]] = [2, 1]
        info[1, [_lib.INFO_STATUS, _lib.INFO_FAIL_BLOCK]] = [1, _lib.BLOCK_R]
        res = gb.PackedResult(np.ones((M, 5, 2)), np.ones((M, 4, 1)), trace, info, 1.0)
        results, errors = batch.unpack_results(res)
        assert errors[0] is None and results[1] is None and "FactorizationError" in errors[1]
        r = results[0]
        assert r.converged and r.iterations == 2 and r.trace[1].alpha is None and r.trace[0].alpha == 0.5
        assert r.trace[0].accepted is True and r.trace[0].pcg_iterations == 9 and r.final_merit == 1.2

    def test_reference_objects_are_accepted_duck_typed(self):
        from conftest import REFERENCE_SRC
        if not REFERENCE_SRC.exists():
            pytest.skip("reference not mounted")
        import sys
        sys.path.insert(0, str(REFERENCE_SRC))
        import trajbatch as tb
        from paper_2510_07625_b200.models import device_model
        assert device_model(tb.TwoLinkArm(gravity=9.81))[0] == 3
        st = batch._as_settings(tb.SolverSettings(max_sqp_iterations=7, step_tolerance=None))
        assert isinstance(st, gb.SolverSettings) and st.max_sqp_iterations == 7 and st.step_tolerance is None


class TestWorkloads:
    def test_batches_are_prefixes_of_larger_batches(self):
        a, b = workloads.iiwa14_reach_arrays(4, 8), workloads.iiwa14_reach_arrays(9, 8)
        assert np.array_equal(a.x_start, b.x_start[:4]) and np.array_equal(a.goal, b.goal[:4])

    def test_tracking_batch_differs_only_in_force(self):
        t = workloads.iiwa14_track_arrays(5, 8, 0.02)
        assert np.all(t.goal == t.goal[0]) and np.all(t.x_start == t.x_start[0])
        assert np.allclose(np.linalg.norm(t.force[1:, 0], axis=1), 5.0) and np.all(t.force[0] == 0)

    def test_arrays_to_spec_round_trip(self):
        a = workloads.iiwa14_reach_arrays(3, 8)
        spec = workloads.arrays_to_spec(a, 0.02, workloads.fixed_budget_settings(5))
        packed = batch.pack_problems(spec.problems, spec.inits, [spec.effective_settings(i).rho_init for i in range(3)])
        for f in ("x_start", "goal", "Q", "R", "QN", "force", "rho_init", "X", "U"):
            assert np.array_equal(getattr(packed, f), getattr(a, f)), f
