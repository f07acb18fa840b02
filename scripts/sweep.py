"""batch x horizon sweep (BASELINE.json configs[3]) in the reference's bench_scaling protocol
(batch.py:127-169): every cell solves M iiwa14 reach problems of horizon N from the cold
initialisation for exactly 5 SQP iterations; one warm-up discarded, median and p90 of the wall time
of `repeats` end-to-end calls.  Emits the reference's CSV schema (M,N,median_ms,p90_ms,workers)
plus device time and throughput columns.

    python scripts/sweep.py [--out gpurun_out/sweep.csv] [--max-batch 512]"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2510_07625_b200 as gb  # noqa: E402
from paper_2510_07625_b200 import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/sweep.csv")
    ap.add_argument("--max-batch", type=int, default=512)
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--cpu", action="store_true",
                    help="add the CPU reference (baseline/_ref, else its oracle port; forked pool over all host cores): one wave of "
                         "min(M, cores) solves is timed per horizon and scaled by ceil(M / cores) waves "
                         "(SURVEY.md 8d: prefix + linear scaling for cells that would take minutes)")
    args = ap.parse_args()
    header = "M,N,median_ms,p90_ms,workers,device_ms,sqp_iteration_rate_hz,solve_iterations_per_s,pcg_its_mean"
    if args.cpu:
        header += ",cpu_port_ms_est,cpu_cores,speedup_vs_cpu_port"
    rows = [header]
    cpu_wave = {}
    M_list = [m for m in (1, 2, 4, 8, 16, 32, 64, 128, 256, 512) if m <= args.max_batch]
    for N in (16, 32, 64, 128):
        h = 0.05 if N >= 64 else 0.02
        for M in M_list:
            batch = workloads.iiwa14_reach_arrays(M, N)
            eng = gb.BatchEngine(gb.Iiwa14(), M, N, h, workloads.fixed_budget_settings(args.iters))
            eng.solve(batch)   # warm-up discarded
            wall, dev = [], []
            for _ in range(args.repeats):
                t0 = time.perf_counter()
                res = eng.solve(batch)
                wall.append(1e3 * (time.perf_counter() - t0))
                dev.append(res.device_ms)
            eng.close()
            wall.sort()
            med = wall[len(wall) // 2]
            p90 = wall[min(len(wall) - 1, int(np.ceil(0.9 * len(wall))) - 1)]
            d = float(np.median(dev))
            row = (f"{M},{N},{med:.4f},{p90:.4f},gpu,{d:.4f},{args.iters * 1e3 / d:.1f},"
                   f"{M * args.iters * 1e3 / d:.1f},{res.trace[:, :args.iters, 4].mean():.1f}")
            if args.cpu:
                import math
                import os
                import bench
                cores = os.cpu_count() or 1
                count = min(M, cores)
                if (N, count) not in cpu_wave:
                    w = dict(M=count, N=N, h=h, kind="reach", sqp=args.iters)
                    arm = bench.CpuArm("sweep", w)       # the unmodified reference (baseline/_ref) if installed
                    arm.step()                                               # warm-up (imports, pool)
                    cpu_wave[(N, count)] = 1e3 * arm.step()[0]
                cpu_ms = cpu_wave[(N, count)] * math.ceil(M / cores)
                row += f",{cpu_ms:.1f},{cores},{cpu_ms / med:.0f}"
            rows.append(row)
            print(rows[-1], flush=True)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text("\n".join(rows) + "\n")


if __name__ == "__main__":
    main()
