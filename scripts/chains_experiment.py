"""Do two half-batch solves on two streams overlap usefully (one half's PCG with the other half's
dynamics kernels)?   python scripts/chains_experiment.py [M] [N] [K]"""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np, torch
import paper_2510_07625_b200 as gb
from paper_2510_07625_b200 import workloads

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
N = int(sys.argv[2]) if len(sys.argv) > 2 else 64
K = int(sys.argv[3]) if len(sys.argv) > 3 else 5
h = 0.05 if N >= 64 else 0.02
st = workloads.fixed_budget_settings(K)
batch = workloads.iiwa14_reach_arrays(M, N)

def run(parts, reps=8):
    bounds = [(i * M // parts, (i + 1) * M // parts) for i in range(parts)]
    engs = [gb.BatchEngine(gb.Iiwa14(), hi - lo, N, h, st) for lo, hi in bounds]
    subs = [batch.slice(lo, hi) for lo, hi in bounds]
    times = []
    for r in range(reps + 2):
        for e, s in zip(engs, subs):
            e.upload(s)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for e in engs:
            e.launch()
        torch.cuda.synchronize()
        times.append(1e3 * (time.perf_counter() - t0))
    outs = [e.download() for e in engs]
    for e in engs:
        e.close()
    X = np.concatenate([o.X for o in outs])
    return float(np.median(times[2:])), X

base, X1 = run(1)
for parts in (2, 3, 4):
    t, Xp = run(parts)
    print(f"M={M} N={N} K={K}: 1 chain {base:.3f} ms, {parts} chains {t:.3f} ms  ({base / t:.2f}x)  bitwise equal: {np.array_equal(X1, Xp)}")
