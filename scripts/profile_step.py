"""Minimal driver for ncu: a few solves of one workload through the C ABI.
    ncu ... python scripts/profile_step.py c3 [reps] [loop_mode]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_2510_07625_b200 as gb  # noqa: E402
from paper_2510_07625_b200 import workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
mode = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = bench.WORKLOADS[name]
batch = bench.make_batch(w, w["M"])
eng = gb.BatchEngine(gb.Iiwa14(), w["M"], w["N"], w["h"], workloads.fixed_budget_settings(w["sqp"]), loop_mode=mode)
for _ in range(reps):
    res = eng.solve(batch)
print(name, "device ms", res.device_ms, "pcg its", res.trace[:, :w["sqp"], 4].mean())
eng.close()
