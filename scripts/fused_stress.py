"""Randomised stress of the fused Schur + PCG path against the unfused one (bitwise) and of both against the compiled
C oracle (tolerance): random batch sizes, horizons, timesteps, goals, force hypotheses, rho, iteration budgets,
tolerance / fixed-budget mode, plus solves with dense weights mixed into fused batches.
    python scripts/fused_stress.py [cases] [seed]"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2510_07625_b200 as gb  # noqa: E402
from oracle import trajopt_c as oc  # noqa: E402
from oracle import trajopt_np as orc  # noqa: E402
from paper_2510_07625_b200 import workloads  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
bad = 0
worst = 0.0
for c in range(cases):
    M = int(rng.integers(1, 9))
    N = int(rng.choice([1, 2, 3, 5, 8, 9, 15, 16, 17, 31, 32, 33, 40, 47, 63, 64]))
    h = float(rng.choice([0.01, 0.02, 0.05]))
    iters = int(rng.integers(1, 5))
    tol_mode = rng.random() < 0.25
    batch = (workloads.iiwa14_track_arrays(M, N, h, seed=int(rng.integers(1 << 30))) if rng.random() < 0.4
             else workloads.iiwa14_reach_arrays(M, N, seed=int(rng.integers(1 << 30))))
    batch.rho_init[:] = 10.0 ** rng.uniform(-6, -2, size=M)
    batch.X += 0.05 * rng.standard_normal(batch.X.shape)      # infeasible initial guesses
    batch.U += 0.5 * rng.standard_normal(batch.U.shape)
    scale = 10.0 ** rng.uniform(-1, 1, size=(M, 14))
    for b in range(M):                                        # per-solve diagonal weights
        batch.Q[b] = np.diag(np.diag(batch.Q[b]) * scale[b])
    dense = rng.random(M) < 0.2
    for b in np.nonzero(dense)[0]:                            # some solves with dense SPD weights (unfused inside a fused batch)
        G = rng.standard_normal((14, 14))
        batch.Q[b] = batch.Q[b] + 0.02 * (G @ G.T)
    st = gb.SolverSettings(max_sqp_iterations=iters, pcg=gb.PcgSettings(tolerance=1e-6 if not tol_mode else 1e-8, max_iterations=200),
                           step_tolerance=1e-6 if tol_mode else None)
    fused = gb.BatchEngine(gb.Iiwa14(), M, N, h, st, fused=True)
    plain = gb.BatchEngine(gb.Iiwa14(), M, N, h, st, fused=False)
    try:
        a, p = fused.solve(batch), plain.solve(batch)
    finally:
        fused.close()
        plain.close()
    same = (np.array_equal(a.X, p.X) and np.array_equal(a.U, p.U) and np.array_equal(a.trace, p.trace, equal_nan=True)
            and np.array_equal(a.info, p.info))
    ost = orc.Settings(max_sqp_iterations=iters, pcg_tolerance=st.pcg.tolerance, pcg_max_iterations=200,
                       step_tolerance=st.step_tolerance)
    X, U, trace, info = oc.solve_batch(batch.x_start, batch.goal, batch.Q, batch.R, batch.QN, batch.force, batch.rho_init,
                                       batch.X, batch.U, h, ost)
    ok_status = np.array_equal(a.info[:, 2] != 0, info[:, 2] != 0)
    good = (a.info[:, 2] == 0) & (a.info[:, 0] == info[:, 0])
    err = 0.0
    for b in np.nonzero(good)[0]:
        n = int(info[b, 0])
        if np.array_equal(a.trace[b, :n, 5], trace[b, :n, 5]):     # same accept decisions: comparable point
            err = max(err, float(np.max(np.abs(a.X[b] - X[b])) / max(1.0, np.max(np.abs(X[b])))))
    worst = max(worst, err)
    flag = "" if (same and ok_status and err <= 1e-5) else "   <-- CHECK"
    bad += bool(flag)
    print(f"case {c:3d}: M={M} N={N:2d} h={h} its={iters} tol={int(tol_mode)} dense={int(dense.sum())} fused==unfused {same} "
          f"status-match {ok_status} err-vs-C {err:.1e}{flag}", flush=True)
print(f"{cases} cases, {bad} to check, worst error vs the C oracle {worst:.2e}")
