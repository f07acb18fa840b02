"""Soak of the control-step call: two engines in lockstep over many consecutive control steps, one moving its host
data with the copy engines (GATO_ZERO_COPY_MAX=0), one with the solve's own kernels (default); the host mirrors
must hold the same bytes after every step.   python scripts/host_step_soak.py [steps]"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2510_07625_b200 as gb  # noqa: E402
from paper_2510_07625_b200 import workloads  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
w = bench.WORKLOADS["c2"]
M, N = w["M"], w["N"]
batch = bench.make_batch(w, M)
path = bench.tracking_reference(w, steps + N + 8, workloads.SEED)
engines = []
for limit in ("0", None):
    if limit is None:
        os.environ.pop("GATO_ZERO_COPY_MAX", None)
    else:
        os.environ["GATO_ZERO_COPY_MAX"] = limit
    eng = gb.BatchEngine(gb.Iiwa14(), M, N, w["h"], workloads.fixed_budget_settings(1), timing=False)
    eng.upload(batch)
    eng.stream.synchronize()
    engines.append(eng)
fields = ("x_start", "goal", "force")
bad = 0
for s in range(steps):
    outs = []
    for eng in engines:
        host_in = eng.host_inputs()
        host_in["goal"][...] = path[s:s + N + 1][None]
        out = eng.step(None, fields=fields, shift=True, copy=False)
        outs.append(out)
    a, b = outs
    same = (np.array_equal(a.X, b.X) and np.array_equal(a.U, b.U) and np.array_equal(a.trace, b.trace, equal_nan=True)
            and np.array_equal(a.info, b.info))
    bad += not same
    for eng, out in zip(engines, outs):
        eng.host_inputs()["x_start"][...] = out.X[:, 1, :]
print(f"{steps} consecutive control steps (32 solves x 32 knots), copy engines vs kernel-moved host data: "
      f"{bad} steps with differing bytes; all solves ok: {bool(np.all(a.info[:, 2] == 0))}")
for eng in engines:
    eng.close()
sys.exit(1 if bad else 0)
