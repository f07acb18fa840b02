"""Small solves of every kernel variant, for compute-sanitizer (memcheck / racecheck / synccheck).
    compute-sanitizer --tool racecheck python scripts/sanitize_small.py"""
import os
import sys
from pathlib import Path

os.environ.setdefault("GATO_LOOP_MODE", "3")   # plain stream launches: racecheck cannot follow conditional graph nodes

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2510_07625_b200 as gb  # noqa: E402
from paper_2510_07625_b200 import workloads  # noqa: E402
from conftest import load_golden, product_problem, product_settings  # noqa: E402

# iiwa14: quadrant PCG (N=8, N=40, N=64 = the full CTA; with GATO_PCG_Q=1 in the environment N=8 runs the
# row-resident k_pcg_rt instead), fat-thread PCG with O^ and L resident (N=70), O^ resident only (N=100),
# everything in global memory (N=150); the control-step call, best-of-batch, hypothesis selection
# ... and the Schur phase fused into k_pcg_q (fused=True; N = 9: a warp with idle quads, N = 64: the full CTA)
for N, iters, fused in ((8, 2, None), (40, 1, None), (64, 1, None), (70, 1, None), (100, 1, None), (150, 1, None),
                        (9, 2, True), (33, 1, True), (64, 1, True)):
    batch = workloads.iiwa14_reach_arrays(3, N)
    eng = gb.BatchEngine(gb.Iiwa14(), 3, N, 0.02, workloads.fixed_budget_settings(iters), loop_mode=3, fused=fused)
    res = eng.solve(batch)
    eng.shift_warm_start()
    eng.stream.synchronize()
    eng.step(batch, shift=True)
    eng.best_of_batch()
    print("iiwa14 N", N, "status", res.info[:, 2].tolist(), "pcg", res.trace[:, 0, 4].tolist())
    eng.close()
# round-2 additions: the 1024-thread long-horizon k_pcg (N = 300), the control step folded into the solve's first
# kernel (k_prologue modes 1 and 2: step(shift=True) above, mpc_step here), and a fused batch in which one solve has
# dense weights (k_hessinv's schur_list, k_schur_listed, the record-reading k_pcg_q build on the side stream)
import torch  # noqa: E402

batch = workloads.iiwa14_reach_arrays(1, 300)
eng = gb.BatchEngine(gb.Iiwa14(), 1, 300, 0.02, workloads.fixed_budget_settings(1), loop_mode=3)
res = eng.solve(batch)
print("iiwa14 N 300 status", res.info[:, 2].tolist(), "pcg", res.trace[:, 0, 4].tolist())
eng.close()
batch = workloads.iiwa14_track_arrays(3, 12, 0.02)
path = torch.as_tensor(np.cumsum(0.01 * np.random.default_rng(3).standard_normal((40, 14)), axis=0), device="cuda")
eng = gb.BatchEngine(gb.Iiwa14(), 3, 12, 0.02, workloads.fixed_budget_settings(1), loop_mode=3)
eng.upload(batch)
eng.launch()
eng.finish()
for s in range(2):
    eng.mpc_step(path, s)
    eng.finish()
print("mpc_step status", eng.download().info[:, 2].tolist())
eng.close()
batch = workloads.iiwa14_reach_arrays(4, 16)
G = np.random.default_rng(5).standard_normal((14, 14))
batch.Q[1] = batch.Q[1] + 0.05 * (G @ G.T)
batch.R[3] = batch.R[3] + 1e-4 * np.ones((7, 7))
eng = gb.BatchEngine(gb.Iiwa14(), 4, 16, 0.02, workloads.fixed_budget_settings(2), loop_mode=3, fused=True)
res = eng.solve(batch)
print("mixed fused batch status", res.info[:, 2].tolist(), "pcg", res.trace[:, 0, 4].tolist())
eng.close()
# the reference's analytic models (k_linearize_simple, small block sizes)
for name in ("pendulum_n8", "cartpole_n8", "twolink_n8", "di7_n8"):
    g = load_golden(name)
    r = gb.sqp_solve(product_problem(g), g["X0"], g["U0"], product_settings(g))
    print(name, len(r.trace), float(np.max(np.abs(r.X - g["X"]))))
# operators
rng = np.random.default_rng(0)
X, U, F = rng.standard_normal((5, 14)), rng.standard_normal((5, 7)), rng.standard_normal((5, 3))
gb.step_many(gb.Iiwa14(), X, U, 0.02, F)
gb.step_jacobians_many(gb.Iiwa14(), X, U, 0.02, F)
gb.select_hypothesis(gb.Iiwa14(), X[0], U[0], X[1], F, 0.004, 0.001)
d = np.tile(np.eye(3) * 4.0, (2, 5, 1, 1))
o = 0.1 * rng.standard_normal((2, 4, 3, 3))
gb.pcg_batched(d, o, rng.standard_normal((2, 15)), np.tile(np.eye(3) / 4.0, (2, 5, 1, 1)), np.zeros((2, 4, 3, 3)), 1e-10)
print("done")
