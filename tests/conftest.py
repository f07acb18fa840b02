"""Shared test helpers.  GPU tests are marked ``gpu``; everything else runs on CPU."""

import math
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN_DIR = Path(__file__).resolve().parent / "golden"
REFERENCE_SRC = Path("/root/reference/pkg/src")

STAGED_CASES = ["pendulum_n8", "cartpole_n8", "twolink_n8", "twolink_gravity_n8", "di1_n4", "di2_n4",
                "di7_n8", "pendulum_n8_tol", "twolink_n8_tol", "iiwa14_random_n8", "iiwa14_reach_n8_b0",
                "iiwa14_reach_n8_b1", "iiwa14_track_n16_b0", "iiwa14_track_n16_b2",
                # time-varying force + non-default line search + unregularised R; rho clamps; PCG cap reached
                "twolink_profile_n8", "cartpole_rho_n8", "iiwa14_pcgcap_n16"]
FINAL_ONLY_CASES = ["pendulum_swingup_n64", "iiwa14_reach_n32_c1", "iiwa14_reach_n16_tol"]
ALL_CASES = STAGED_CASES + FINAL_ONLY_CASES


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")
    config.addinivalue_line("markers", "reference: needs /root/reference (build container only)")


def load_golden(name):
    with np.load(GOLDEN_DIR / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def product_model(g):
    """Product model descriptor of a golden case."""
    import paper_2510_07625_b200 as gb
    name, p = str(g["model"]), g["model_params"]
    if name == "double_integrator":
        return gb.DoubleIntegrator(dims=int(p[0]), mass=float(p[1]))
    if name == "pendulum":
        return gb.Pendulum(*map(float, p[:4]))
    if name == "cartpole":
        return gb.Cartpole(*map(float, p[:4]))
    if name == "two_link_arm":
        return gb.TwoLinkArm(*map(float, p[:6]))
    if name == "iiwa14":
        return gb.Iiwa14()
    raise ValueError(name)


def product_settings(g):
    import paper_2510_07625_b200 as gb
    s = g["settings"]
    return gb.SolverSettings(
        max_sqp_iterations=int(s[0]),
        pcg=gb.PcgSettings(tolerance=float(s[1]), max_iterations=None if s[2] < 0 else int(s[2])),
        line_search=gb.LineSearchSettings(mu=float(s[3]), beta=float(s[4]), num_shrinks=int(s[5])),
        rho_init=float(s[6]), rho_min=float(s[7]), rho_max=float(s[8]), rho_factor=float(s[9]),
        step_tolerance=None if math.isnan(s[10]) else float(s[10]), feasibility_tolerance=float(s[11]),
        regularize_r=bool(s[12]), pcg_retry_limit=int(s[13]))


class KnotTable:
    """Force profile that returns the golden file's per-knot force at t = k*h."""

    def __init__(self, table, h):
        self.table, self.h = np.asarray(table, dtype=float), float(h)

    def __call__(self, t):
        return self.table[int(round(t / self.h))]


def product_problem(g):
    import paper_2510_07625_b200 as gb
    model = product_model(g)
    force, h = g["force"], float(g["timestep"])
    if np.all(force == force[0]):
        ext = gb.ExternalForce.constant(force[0])
    else:   # the reference sampled its profile at the knot start times k*h (qpform.py:113-123)
        ext = gb.ExternalForce.time_varying(KnotTable(force, h), force.shape[1])
    return gb.ProblemSpec(model=model, cost=gb.CostSpec(g["Q"], g["R"], g["QN"], g["goal"]),
                          horizon=int(g["horizon"]), timestep=h, x_start=g["x_start"], force=ext)


def oracle_settings(g):
    from oracle import trajopt_np as orc
    s = g["settings"]
    return orc.Settings(
        max_sqp_iterations=int(s[0]), pcg_tolerance=float(s[1]),
        pcg_max_iterations=None if s[2] < 0 else int(s[2]), mu=float(s[3]), beta=float(s[4]),
        num_shrinks=int(s[5]), rho_init=float(s[6]), rho_min=float(s[7]), rho_max=float(s[8]),
        rho_factor=float(s[9]), step_tolerance=None if math.isnan(s[10]) else float(s[10]),
        feasibility_tolerance=float(s[11]), regularize_r=bool(s[12]), pcg_retry_limit=int(s[13]))


def oracle_problem(g):
    from oracle import trajopt_np as orc
    model = orc.model_from_descriptor(product_model(g))
    return orc.Problem(model, g["Q"], g["R"], g["QN"], g["goal"], int(g["horizon"]), float(g["timestep"]),
                       g["x_start"], g["force"])


def rel_inf(actual, reference):
    """oracles.relative_inf_error (oracles.py:166-168)."""
    reference = np.asarray(reference, dtype=float)
    denom = max(1.0, float(np.max(np.abs(reference)))) if reference.size else 1.0
    return float(np.max(np.abs(np.asarray(actual) - reference))) / denom if reference.size else 0.0


def trace_rows(result):
    """Trace of an oracle/product result in the golden layout."""
    return np.array([[r.iteration, r.merit, r.constraint_l1, np.nan if r.alpha is None else r.alpha, r.rho,
                      r.pcg_iterations, float(r.accepted), r.step_inf_norm] for r in result.trace],
                    dtype=float).reshape(-1, 8)


@pytest.fixture
def rng():
    return np.random.default_rng(12345)
