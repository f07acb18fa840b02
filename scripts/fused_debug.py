"""Fused vs unfused first pass: compares what the fused Schur phase leaves in global memory (gamma, gammaw, grad,
packed L inside the matrix record) and the step (lam, dX, dU) with the unfused kernels' arrays.
    python scripts/fused_debug.py [N] [M]"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2510_07625_b200 as gb  # noqa: E402
from paper_2510_07625_b200 import workloads  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
M = int(sys.argv[2]) if len(sys.argv) > 2 else 2
batch = workloads.iiwa14_reach_arrays(M, N)
st = workloads.fixed_budget_settings(1)
out = {}
for name, flag in (("fused", False), ("plain", True)):
    eng = gb.BatchEngine(gb.Iiwa14(), M, N, 0.02, st, stage_arrays=flag)
    res = eng.solve(batch)
    out[name] = {k: eng.scratch(k) for k in ("gamma", "gammaw", "grad", "pmats", "lam", "dX", "dU", "lbw")}
    out[name]["X"] = res.X
    out[name]["trace"] = res.trace
    eng.close()
n, nb = 14, N + 1
BSP, TRP = 198, 106
for k in ("gamma", "gammaw", "grad", "lam", "dX", "dU", "X", "trace"):
    a, b = out["fused"][k], out["plain"][k]
    d = np.abs(np.nan_to_num(a) - np.nan_to_num(b))
    print(f"{k:8s} max abs diff {d.max():.3e}  (first bad index {int(np.argmax(d > 0)) if d.max() > 0 else -1}, size {a.size})")
rec = N * BSP + 2 * nb * TRP
for b in range(M):
    fa, pa = out["fused"]["pmats"][b * rec:(b + 1) * rec], out["plain"]["pmats"][b * rec:(b + 1) * rec]
    Lf_f = fa[N * BSP + nb * TRP:].reshape(nb, TRP)[:, :105]
    Lf_p = pa[N * BSP + nb * TRP:].reshape(nb, TRP)[:, :105]
    d = np.abs(Lf_f - Lf_p)
    print(f"solve {b}: packed L max abs diff per block row:", np.array2string(d.max(axis=1), precision=2))
g_f, g_p = out["fused"]["gamma"].reshape(M, nb, n), out["plain"]["gamma"].reshape(M, nb, n)
print("gamma diff block row 1:", np.array2string(np.abs(g_f - g_p)[0, 1], precision=2))
print("gamma diff block row 2:", np.array2string(np.abs(g_f - g_p)[0, 2], precision=2))
fa, pa = out["fused"]["pmats"][:rec], out["plain"]["pmats"][:rec]
Lf_f = fa[N * BSP + nb * TRP:].reshape(nb, TRP)[1, :105]
Lf_p = pa[N * BSP + nb * TRP:].reshape(nb, TRP)[1, :105]
D = np.zeros((14, 14))
for r in range(14):
    for c in range(r + 1):
        D[r, c] = abs(Lf_f[r * (r + 1) // 2 + c] - Lf_p[r * (r + 1) // 2 + c])
np.set_printoptions(linewidth=250)
print("L diff block row 1 (rows x cols):")
print(np.array2string(D, precision=1))
