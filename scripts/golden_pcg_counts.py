"""How many golden cases reproduce the reference's PCG iteration counts exactly (the parity bar is +-1).
    python scripts/golden_pcg_counts.py          (needs a GPU)"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2510_07625_b200 as gb  # noqa: E402
from conftest import ALL_CASES, load_golden, product_problem, product_settings  # noqa: E402

same = 0
worst_x = 0.0
for name in ALL_CASES:
    g = load_golden(name)
    res = gb.sqp_solve(product_problem(g), g["X0"], g["U0"], product_settings(g))
    got = np.array([r.pcg_iterations for r in res.trace])
    ref = g["trace"][:, 5].astype(int)
    n = min(len(got), len(ref))
    d = int(np.max(np.abs(got[:n] - ref[:n]))) if n else 0
    ex = float(np.max(np.abs(res.X - g["X"])) / max(1.0, float(np.max(np.abs(g["X"])))))
    worst_x = max(worst_x, ex)
    same += d == 0 and len(got) == len(ref)
    print(f"{name:28s} sqp its {len(got)}/{len(ref)}  max |pcg diff| {d}  rel err X {ex:.2e}")
print(f"{same} of {len(ALL_CASES)} cases with identical PCG counts; worst relative trajectory error {worst_x:.2e}")
