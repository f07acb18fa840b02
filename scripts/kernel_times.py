"""Per-kernel device times (CUDA events between kernels) of one workload:
    python scripts/kernel_times.py c3 [reps]"""
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_2510_07625_b200 as gb  # noqa: E402
from paper_2510_07625_b200 import workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
w = bench.WORKLOADS[name]
batch = bench.make_batch(w, w["M"])
eng = gb.BatchEngine(gb.Iiwa14(), w["M"], w["N"], w["h"], workloads.fixed_budget_settings(w["sqp"]))
out = []
for _ in range(reps + 1):
    eng.upload(batch)
    eng.stream.synchronize()
    out.append(eng.solve_profiled())
eng.close()
print(name, {k: round(statistics.median(o[k] for o in out[1:]), 4) for k in out[0]})
