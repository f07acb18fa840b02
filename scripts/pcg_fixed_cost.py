"""Fixed cost of the PCG kernel (fill + O^ prologue + step recovery) versus its per-iteration cost: the
same workload solved with PCG iteration caps 1, 11, 21 and uncapped; kernel time from gato_solve_profiled.
    python scripts/pcg_fixed_cost.py [c2|c3|c5]"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2510_07625_b200 as gb  # noqa: E402
from paper_2510_07625_b200 import workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
M, N, h = {"c2": (32, 32, 0.02), "c3": (128, 64, 0.05), "c5": (1024, 64, 0.05)}[name]
batch = workloads.iiwa14_reach_arrays(M, N)
for cap in (1, 11, 21, 200):
    eng = gb.BatchEngine(gb.Iiwa14(), M, N, h, workloads.fixed_budget_settings(1, pcg_max_iterations=cap))
    try:
        eng.upload(batch)
        eng.solve_profiled()
        ms = [eng.solve_profiled()["pcg"] for _ in range(10)]
        its = eng.solve(batch).trace[:, 0, 4].mean()
    finally:
        eng.close()
    print(f"{name} cap {cap:3d}: pcg kernel {1e3 * float(np.median(ms)):8.1f} us, mean iterations {its:.1f}")
