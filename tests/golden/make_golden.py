"""Generates tests/golden/*.npz by running the UNMODIFIED reference package
(/root/reference/pkg/src/trajbatch) on seeded problems.  Run in the build container only:

    python tests/golden/make_golden.py

The reference is pure Python and cannot travel to the GPU box, so its stage-by-stage outputs
are committed here as small fixtures: inputs, the first iteration's intermediates
(linearize -> form_schur -> form_preconditioner -> pcg -> recover_step -> merit_many) and
the result of the full sqp_solve.  The iiwa14 model is not part of the reference; for those
cases the reference *solver* is run unmodified with oracle/iiwa14_np.py plugged in through
the reference's own DynamicsModel interface (dynamics.py:94-142).
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import dataclasses

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
REF = Path(os.environ.get("TRAJBATCH_REF", "/root/reference/pkg/src"))
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))

import trajbatch as tb  # noqa: E402
from trajbatch import oracles  # noqa: E402
from trajbatch.qpform import form_preconditioner, form_schur, linearize, recover_step  # noqa: E402
from trajbatch.sqp import merit, merit_many  # noqa: E402

from oracle.iiwa14_np import Iiwa14 as OracleIiwa14  # noqa: E402
from paper_2510_07625_b200 import workloads  # noqa: E402

OUT = Path(__file__).resolve().parent


class RefIiwa14(OracleIiwa14, tb.DynamicsModel):
    """oracle/iiwa14_np.py behind the reference's DynamicsModel base class."""
    name = "iiwa14"
    state_dim = 14
    control_dim = 7
    force_dim = 3


MODEL_PARAMS = {
    "double_integrator": lambda m: [m.dims, m.mass],
    "pendulum": lambda m: [m.mass, m.length, m.gravity, m.damping],
    "cartpole": lambda m: [m.cart_mass, m.pole_mass, m.pole_length, m.gravity],
    "two_link_arm": lambda m: [m.m1, m.m2, m.l1, m.l2, m.gravity, m.joint_damping],
    "iiwa14": lambda m: [],
}


def settings_vector(st) -> np.ndarray:
    return np.array([
        st.max_sqp_iterations, st.pcg.tolerance,
        -1 if st.pcg.max_iterations is None else st.pcg.max_iterations,
        st.line_search.mu, st.line_search.beta, st.line_search.num_shrinks, st.rho_init, st.rho_min,
        st.rho_max, st.rho_factor, np.nan if st.step_tolerance is None else st.step_tolerance,
        st.feasibility_tolerance, float(st.regularize_r), st.pcg_retry_limit], dtype=float)


def trace_array(trace) -> np.ndarray:
    return np.array([[r.iteration, r.merit, r.constraint_l1,
                      np.nan if r.alpha is None else r.alpha, r.rho, r.pcg_iterations,
                      float(r.accepted), r.step_inf_norm] for r in trace], dtype=float).reshape(-1, 8)


ONLY = set(sys.argv[1:])      # python make_golden.py [case ...]: regenerate only the named cases


def dump(name, problem, X0, U0, settings, stages=True):
    if ONLY and name not in ONLY:
        return
    N, n = problem.horizon, problem.model.state_dim
    goal = problem.cost.goal if problem.cost.goal.ndim == 2 else np.broadcast_to(problem.cost.goal, (N + 1, n))
    params = np.zeros(8)
    p = MODEL_PARAMS[problem.model.name](problem.model)
    params[:len(p)] = p
    data = dict(
        model=np.array(problem.model.name), model_params=params, horizon=N, timestep=problem.timestep,
        x_start=problem.x_start, goal=np.array(goal), Q=problem.cost.Q, R=problem.cost.R, QN=problem.cost.QN,
        force=np.array(problem.force_matrix()), X0=X0, U0=U0, settings=settings_vector(settings))
    if stages:
        rho = settings.rho_init
        blocks = linearize(problem, X0, U0, rho, settings.regularize_r)
        system = form_schur(blocks, problem.x_start, X0)
        phi_inv = form_preconditioner(system)
        pres = tb.pcg(system.S, system.gamma, phi_inv, settings.pcg)
        direction = recover_step(system, blocks, pres.solution)
        alphas = settings.line_search.candidates()
        Xs = X0[None] + alphas[:, None, None] * direction.dX[None]
        Us = U0[None] + alphas[:, None, None] * direction.dU[None]
        data.update(
            A=np.stack([b.A for b in blocks[:-1]]), B=np.stack([b.B for b in blocks[:-1]]),
            e=np.stack([b.e for b in blocks[:-1]]), q=np.stack([b.q for b in blocks]),
            r=np.stack([b.r for b in blocks[:-1]]),
            Sdiag=system.S.diag_blocks, Soff=system.S.offdiag_blocks, gamma=system.gamma,
            Pdiag=phi_inv.diag_blocks, Poff=phi_inv.offdiag_blocks, q_inv=system.q_inv, r_inv=system.r_inv,
            lam=pres.solution, pcg_iterations=pres.iterations, pcg_converged=pres.converged,
            dX=direction.dX, dU=direction.dU, step_inf=direction.inf_norm,
            merits=merit_many(problem, Xs, Us, settings.line_search.mu),
            merit0=merit(problem, X0, U0, settings.line_search.mu),
            step_rows=tb.dynamics.step_many(problem.model, X0[:-1], U0, problem.timestep, problem.force_matrix()))
    result = tb.sqp_solve(problem, X0, U0, settings)
    data.update(X=result.X, U=result.U, trace=trace_array(result.trace), converged=result.converged)
    np.savez_compressed(OUT / f"{name}.npz", **data)
    last = result.trace[-1]
    print(f"{name:28s} its={len(result.trace):3d} conv={result.converged!s:5s} merit={last.merit:.6g} "
          f"pcg={[r.pcg_iterations for r in result.trace][:6]}")


def fixed(iters, tol=1e-8, cap=None, **kw):
    return tb.SolverSettings(max_sqp_iterations=iters, pcg=tb.PcgSettings(tolerance=tol, max_iterations=cap),
                             step_tolerance=None, **kw)


def random_case(name, seed, model, N, settings):
    rng = np.random.default_rng(seed)
    problem, X, U = oracles.random_problem(rng, model=model, N=N)
    dump(name, problem, X, U, settings)


def to_ref_problem(batch, b, h, model):
    cost = tb.CostSpec(batch.Q[b], batch.R[b], batch.QN[b], batch.goal[b])
    return tb.ProblemSpec(model=model, cost=cost, horizon=batch.X.shape[1] - 1, timestep=h,
                          x_start=batch.x_start[b], force=tb.ExternalForce.constant(batch.force[b, 0]))


def main():
    # the reference's own analytic models, random dense SPD costs, infeasible random inits
    random_case("pendulum_n8", 101, tb.Pendulum(), 8, fixed(6))
    random_case("cartpole_n8", 102, tb.Cartpole(), 8, fixed(6))
    random_case("twolink_n8", 103, tb.TwoLinkArm(), 8, fixed(6))
    random_case("twolink_gravity_n8", 104, tb.TwoLinkArm(gravity=9.81), 8, fixed(6))
    random_case("di1_n4", 105, tb.DoubleIntegrator(dims=1), 4, fixed(4))
    random_case("di2_n4", 106, tb.DoubleIntegrator(dims=2), 4, fixed(4))
    random_case("di7_n8", 107, tb.DoubleIntegrator(dims=7), 8, fixed(4))
    random_case("pendulum_n8_tol", 108, tb.Pendulum(), 8, tb.SolverSettings())
    random_case("twolink_n8_tol", 109, tb.TwoLinkArm(), 8, tb.SolverSettings())

    # pendulum swing-up of the reference's test_sqp.py:26-34 / :201-211 (tolerance mode)
    cost = tb.CostSpec(Q=np.diag([1.0, 0.1]), R=np.diag([0.01]), QN=np.diag([100.0, 10.0]),
                       goal=np.array([np.pi, 0.0]))
    swing = tb.ProblemSpec(model=tb.Pendulum(), cost=cost, horizon=64, timestep=0.05, x_start=np.zeros(2))
    dump("pendulum_swingup_n64", swing, np.zeros((65, 2)), np.zeros((64, 1)),
         tb.SolverSettings(max_sqp_iterations=200), stages=False)

    # iiwa14 through the unmodified reference solver
    iiwa = RefIiwa14()
    random_case("iiwa14_random_n8", 110, iiwa, 8, fixed(5, tol=1e-8))
    reach = workloads.iiwa14_reach_arrays(2, 8)
    for b in range(2):
        dump(f"iiwa14_reach_n8_b{b}", to_ref_problem(reach, b, 0.02, iiwa), reach.X[b], reach.U[b],
             fixed(5, tol=1e-6, cap=200))
    track = workloads.iiwa14_track_arrays(3, 16, 0.02)
    for b in (0, 2):
        dump(f"iiwa14_track_n16_b{b}", to_ref_problem(track, b, 0.02, iiwa), track.X[b], track.U[b],
             fixed(3, tol=1e-6, cap=200))
    # BASELINE.json configs[0]: single solve, N=32, fixed SQP/PCG budget (final results only)
    c1 = workloads.iiwa14_reach_arrays(1, 32)
    dump("iiwa14_reach_n32_c1", to_ref_problem(c1, 0, 0.02, iiwa), c1.X[0], c1.U[0],
         fixed(5, tol=1e-6, cap=200), stages=False)
    # settings off the defaults, a time-varying force profile (dynamics.py:71-91), R not regularised
    rng = np.random.default_rng(111)
    arm = tb.TwoLinkArm(gravity=9.81)
    prob, X, U = oracles.random_problem(rng, model=arm, N=8)
    prob = dataclasses.replace(prob, force=tb.ExternalForce.time_varying(
        tb.dynamics.SwingingLoadProfile(weight=1.5, amplitude=2.0, frequency_hz=2.0), 2))
    dump("twolink_profile_n8", prob, X, U,
         tb.SolverSettings(max_sqp_iterations=5, pcg=tb.PcgSettings(tolerance=1e-8), step_tolerance=None,
                           regularize_r=False, line_search=tb.LineSearchSettings(mu=5.0, beta=3.0, num_shrinks=4)))
    # rho clamped at both ends (sqp.py:198-201)
    random_case("cartpole_rho_n8", 112, tb.Cartpole(), 8,
                tb.SolverSettings(max_sqp_iterations=6, pcg=tb.PcgSettings(tolerance=1e-8), step_tolerance=None,
                                  rho_init=1e-2, rho_factor=10.0, rho_min=1e-3, rho_max=1e-1))
    # PCG stopped by its iteration cap (blocktri.py:78-81,173): the real-time budget regime
    capped = workloads.iiwa14_reach_arrays(1, 16)
    dump("iiwa14_pcgcap_n16", to_ref_problem(capped, 0, 0.02, iiwa), capped.X[0], capped.U[0],
         fixed(3, tol=1e-6, cap=20))
    # tolerance mode on iiwa14
    t16 = workloads.iiwa14_reach_arrays(1, 16)
    dump("iiwa14_reach_n16_tol", to_ref_problem(t16, 0, 0.05, iiwa), t16.X[0], t16.U[0],
         tb.SolverSettings(pcg=tb.PcgSettings(tolerance=1e-6)), stages=False)


if __name__ == "__main__":
    main()
