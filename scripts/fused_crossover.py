"""Fused (Schur inside k_pcg_q) vs unfused (k_schur + record) step time over a batch x horizon grid: the
measurement behind the dispatch rule in gato_api.cu.   python scripts/fused_crossover.py"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2510_07625_b200 as gb  # noqa: E402
from paper_2510_07625_b200 import workloads  # noqa: E402


def step_ms(M, N, fused, iters=2, reps=15):
    os.environ["GATO_FUSED"] = "2" if fused else "0"      # 2: force, 0: off
    batch = workloads.iiwa14_reach_arrays(M, N)
    eng = gb.BatchEngine(gb.Iiwa14(), M, N, 0.05 if N == 64 else 0.02, workloads.fixed_budget_settings(iters))
    try:
        ts = []
        for _ in range(reps):
            eng.upload(batch)
            eng.launch()
            eng.stream.synchronize()
            ts.append(eng.download().device_ms)
        return float(np.median(ts[3:])) / iters
    finally:
        eng.close()


print("M,N,unfused_ms_per_pass,fused_ms_per_pass,fused_over_unfused")
for N in (8, 16, 32, 48, 64):
    for M in (1, 8, 16, 32, 48, 64, 96, 128, 148, 192, 256, 512):
        u, f = step_ms(M, N, False), step_ms(M, N, True)
        print(f"{M},{N},{u:.4f},{f:.4f},{f / u:.3f}", flush=True)
