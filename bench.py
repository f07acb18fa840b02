#!/usr/bin/env python
"""bench.py -- headline benchmark of the batched SQP solve (BASELINE.json metric).

    python bench.py --gpus N --steps K --warmup W [--workload c2] [--impl reference]

One "step" = one batched solve call over one batch of synthetic iiwa14 problems
(SURVEY.md section 8d).  Default workload = BASELINE.json configs[1]: MPC tracking,
batch 32, N = 32 knots, one SQP iteration per control step, warm-started by the device-side
shift of the previous solution.  Metric: solve-iterations per second (solves x SQP iterations
completed per second, whole job over all GPUs); the batched SQP iteration rate (Hz), solves/s
and p50 call latency are reported beside it.

Rank 0 prints ONE JSON line.  N > 1: one process per GPU under torchrun, every rank runs the
per-GPU workload on its own shard of solves (weak scaling, no collective on the solve path;
the only communication is the final gather of the last step's results to rank 0).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: (batch per GPU, horizon, timestep, kind, SQP iterations per step)
    "c1": dict(M=1, N=32, h=0.02, kind="reach", sqp=5, desc="iiwa14 reach, single solve, N=32, 5 SQP its"),
    "c2": dict(M=32, N=32, h=0.02, kind="track", sqp=1,
               desc="iiwa14 MPC tracking, batch=32, N=32, 1 SQP it per control step (real-time regime)"),
    "c3": dict(M=128, N=64, h=0.05, kind="reach", sqp=5,
               desc="iiwa14 reach, batch=128, N=64, 5 SQP its, 9-candidate parallel line search"),
    "c5": dict(M=1024, N=64, h=0.05, kind="reach", sqp=5, desc="iiwa14 reach, batch=1024 per GPU, N=64, 5 SQP its"),
}
METRIC = "sqp_solve_iterations_per_sec"
UNIT = "solve-iterations/s"

# SURVEY.md section 8d / BASELINE.md section 4: algorithmic flops (FMA = 2), n=14, m=7, C=9
F_LIN, F_SCHUR, F_PREC, F_REC, F_LS, F_HESS = 95_000, 16_506, 13_720, 1_127, 21_000, 11_662


def f_pcg(N):
    return 784 * (3 * N + 1) + 168 * (N + 1)


def flops_solve_iteration(N, P, C=9):
    return N * F_LIN + N * F_SCHUR + (N + 1) * F_PREC + P * f_pcg(N) + N * F_REC + C * N * F_LS + F_HESS


def ncu_traffic(workload, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`, from the newest committed
    `ncu --set full` capture of this workload (profiles/rNN_ncu_kernels.json); None if not captured."""
    files = sorted((ROOT / "profiles").glob("r*_ncu_kernels.json"))
    for f in reversed(files):
        try:
            return float(json.loads(f.read_text())[workload][kernel]["dram_bytes_per_launch"])
        except Exception:
            continue
    return None


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="gato", choices=["gato", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=None, help="override the per-GPU batch size")
    ap.add_argument("--horizon", type=int, default=None)
    ap.add_argument("--sqp-iters", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    return ap.parse_args()


def workload_config(args):
    w = dict(WORKLOADS[args.workload])
    if args.batch:
        w["M"] = args.batch
    if args.horizon:
        w["N"] = args.horizon
    if args.sqp_iters:
        w["sqp"] = args.sqp_iters
    return w


def make_batch(w, M, seed_offset=0):
    from paper_2510_07625_b200 import workloads
    if w["kind"] == "track":
        return workloads.iiwa14_track_arrays(M, w["N"], w["h"], seed=workloads.SEED + seed_offset)
    return workloads.iiwa14_reach_arrays(M, w["N"], seed=workloads.SEED + seed_offset)


def tracking_reference(w, steps, seed):
    """Goal windows of consecutive control steps: (steps, N+1, 14) from the same generator."""
    from paper_2510_07625_b200 import workloads
    rng = np.random.default_rng(seed)
    q0 = rng.uniform(-0.6, 0.6, size=7)
    N, h = w["N"], w["h"]
    t = np.arange(steps + N + 2) * h
    phase = np.arange(7) * np.pi / 7.0
    q = q0[None, :] + 0.4 * np.sin(2.0 * np.pi * t[:, None] / 4.0 + phase[None, :])
    qd = np.zeros_like(q)
    qd[:-1] = (q[1:] - q[:-1]) / h
    qd[-1] = qd[-2]
    return np.concatenate([q, qd], axis=1)


# --------------------------------------------------------------------------------------
# clocks
# --------------------------------------------------------------------------------------

class ClockSampler:
    """Samples SM clock and throttle reasons of one GPU during the timed region (NVML)."""

    REASONS = {
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
        0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting", 0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._thread = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.dev = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.dev, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.dev, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.dev)
                for bit, name in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.02)

    def __enter__(self):
        if self.nv is not None:
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread is not None:
            self._thread.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------------------
# CPU arm: the oracle port of the reference's CPU implementation, all host cores
# --------------------------------------------------------------------------------------

def cpu_problems(w, batch, count):
    from oracle import trajopt_np as orc
    from oracle.iiwa14_np import Iiwa14
    probs = [orc.Problem(Iiwa14(), batch.Q[b], batch.R[b], batch.QN[b], batch.goal[b], w["N"], w["h"],
                         batch.x_start[b], batch.force[b]) for b in range(count)]
    inits = [(batch.X[b], batch.U[b]) for b in range(count)]
    st = orc.Settings(max_sqp_iterations=w["sqp"], pcg_tolerance=1e-6, pcg_max_iterations=200, step_tolerance=None)
    return probs, inits, [st] * count


def cpu_step(w, batch, count, cores):
    """One bounded CPU sample: `count` solves of the workload over a forked pool of `cores`
    workers (the reference's batch_solve(workers=cores), batch.py:102-124). -> seconds."""
    from oracle import trajopt_np as orc
    probs, inits, sts = cpu_problems(w, batch, count)
    _, errors, wall = orc.solve_batch_parallel(probs, inits, sts, cores)
    assert all(e is None for e in errors), errors
    return wall


def cpu_baseline(w, batch, budget_s):
    cores = os.cpu_count() or 1
    count = min(batch.size, cores)
    t1 = cpu_step(w, batch, count, cores)               # also warms the imports
    reps = max(1, min(5, int(budget_s / max(t1, 1e-3)) - 1))
    times = [cpu_step(w, batch, count, cores) for _ in range(reps)]
    t = statistics.median(times)
    return {"value": count * w["sqp"] / t, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{count} of the workload's solves x {w['sqp']} SQP iteration(s), forked pool of {cores} "
                      f"workers (reference batch_solve semantics), median of {reps} run(s) after 1 warm-up",
            "seconds_per_sample": t}


def cpu_baseline_c(w, batch, budget_s):
    """Second CPU arm: the compiled C restatement of the same algorithm (oracle/trajopt_c.c, POSIX threads
    over the solves) on all host cores, bounded sample.  Not the reference's own implementation (that is
    the numpy arm above); reported so that the GPU/CPU ratio can also be read against compiled code."""
    from oracle import trajopt_c as oc
    from oracle import trajopt_np as orc
    cores = os.cpu_count() or 1
    st = orc.Settings(max_sqp_iterations=w["sqp"], pcg_tolerance=1e-6, pcg_max_iterations=200, step_tolerance=None)
    count = min(batch.size, 8 * cores)

    def once():
        t0 = time.perf_counter()
        oc.solve_batch(batch.x_start[:count], batch.goal[:count], batch.Q[:count], batch.R[:count], batch.QN[:count],
                       batch.force[:count], batch.rho_init[:count], batch.X[:count], batch.U[:count], w["h"], st,
                       threads=cores)
        return time.perf_counter() - t0

    t1 = once()
    reps = max(1, min(5, int(budget_s / max(t1, 1e-3)) - 1))
    t = statistics.median([once() for _ in range(reps)])
    return {"value": count * w["sqp"] / t, "unit": UNIT, "cores": cores, "kind": "port-c",
            "sample": f"{count} of the workload's solves x {w['sqp']} SQP iteration(s), {cores} POSIX threads, "
                      f"median of {reps} run(s) after 1 warm-up", "seconds_per_sample": t}


def run_reference_arm(args, w, rank, world):
    """bench.py --impl reference: the reference's CPU implementation of the path (numpy; here its
    bitwise-pinned oracle port, since /root/reference does not exist on the GPU box) timed on the
    host cores.  Rank 0 only."""
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    batch = make_batch(w, w["M"])
    count = min(batch.size, cores)
    t_cal = cpu_step(w, batch, count, cores)
    budget = 150.0
    steps = max(1, min(args.steps, int(budget / max(t_cal, 1e-3)) - args.warmup))
    warm = min(args.warmup, max(0, int(0.2 * budget / max(t_cal, 1e-3))))
    for _ in range(warm):
        cpu_step(w, batch, count, cores)
    times = [cpu_step(w, batch, count, cores) for _ in range(steps)]
    total = sum(times)
    value = steps * count * w["sqp"] / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "requested_steps": args.steps, "warmup": warm, "ms_per_step": 1e3 * total / steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.workload}: {w['desc']}", "batch_per_gpu": w["M"], "horizon": w["N"],
                   "timestep": w["h"], "sqp_iterations_per_step": w["sqp"],
                   "note": "CPU arm: each step solves a bounded sample of the batch"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{count} of {w['M']} solves x {w['sqp']} SQP iteration(s) per step, forked "
                                   f"pool of {cores} workers"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------------------

def run_gpu_arm(args, w, rank, local_rank, world):
    import torch
    import torch.distributed as dist

    import paper_2510_07625_b200 as gb
    from paper_2510_07625_b200 import _lib, sharding, workloads
    from paper_2510_07625_b200.engine import PackedBatch, measure_fp64_peak

    # GATO_DIST_BACKEND=gloo lets the multi-rank path be exercised on a box with fewer GPUs than
    # ranks (ranks wrap around the visible devices, collectives go through host memory)
    backend = os.environ.get("GATO_DIST_BACKEND", "nccl")
    local_rank = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(local_rank)
    device = torch.device("cuda", local_rank)
    coll_device = device if backend == "nccl" else torch.device("cpu")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(backend)

    M, N, h, K_sqp = w["M"], w["N"], w["h"], w["sqp"]
    settings = workloads.fixed_budget_settings(K_sqp)
    # every rank owns its own shard of solves of the global batch (contiguous index range)
    global_batch = make_batch(w, M * world)
    batch = global_batch.slice(rank * M, (rank + 1) * M)
    eng = gb.BatchEngine(gb.Iiwa14(), M, N, h, settings, device=local_rank)
    track = w["kind"] == "track"
    total_steps = args.warmup + args.steps
    ref_path = tracking_reference(w, 2 * total_steps + 4, workloads.SEED) if track else None
    ref_dev = torch.as_tensor(ref_path, device=device) if track else None
    X0 = torch.as_tensor(batch.X, device=device)
    U0 = torch.as_tensor(batch.U, device=device)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)
    stream = eng.stream

    def device_step(s):
        """Inputs resident in HBM.  track: MPC control step s (measured state = predicted next
        state, warm start = device shift, goal window advanced); reach: solve from the cold init."""
        with torch.cuda.stream(stream):
            if track:
                eng.mpc_advance(ref_dev, s)    # one kernel: measured state, device shift, goal window
            else:
                eng.dev["X"].copy_(X0)
                eng.dev["U"].copy_(U0)
            eng.launch()

    # ---- device-resident throughput: K steps, CUDA events per step, L2 flushed between steps ----
    eng.upload(batch)
    stream.synchronize()
    for s in range(args.warmup):
        device_step(s)
    eng.finish()
    stream.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clocks:
        wall0 = time.perf_counter()
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(1.0)                      # evict L2 (126 MB) between timed steps, untimed
                starts[i].record(stream)
            device_step(args.warmup + i)
            ends[i].record(stream)
        torch.cuda.synchronize()
        wall1 = time.perf_counter()
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in zip(starts, ends)]
    dev_ms = float(sum(step_ms))
    launches_per_step = eng.launch_count() + (1 if track else 0)   # + k_mpc_advance
    res_last = eng.download()
    status_ok = bool(np.all(res_last.info[:, _lib.INFO_STATUS] == 0))
    pcg_last = res_last.trace[:, :K_sqp, _lib.TRACE_PCG_ITERATIONS]

    # ---- end to end through the public array API: host inputs in, host results out ----
    e2e_steps = args.steps
    lat = []
    eng.upload(batch)
    stream.synchronize()
    host_x = batch.x_start.copy()
    step_inputs = PackedBatch(host_x, batch.goal.copy(), batch.Q, batch.R, batch.QN, batch.force, batch.rho_init,
                              batch.X, batch.U)
    h2d_fields = ("x_start", "goal", "force") if track else ("x_start", "goal", "Q", "R", "QN", "force",
                                                              "rho_init", "X", "U")
    h2d_bytes = sum(getattr(step_inputs, f).nbytes for f in h2d_fields)

    host_in = eng.host_inputs()      # pinned staging buffers of the inputs, written in place

    def e2e_step(s):
        # BatchEngine.step = one gato_solve_host call: pinned H2D of the inputs, (device shift,) solve, D2H;
        # the caller fills the pinned inputs in place and reads the results from the pinned mirror
        if track:
            host_in["goal"][...] = ref_path[s:s + N + 1][None]
            out = eng.step(None, fields=h2d_fields, shift=True, copy=False)
            host_in["x_start"][...] = out.X[:, 1, :]       # "measured" state for the next control step
        else:
            for f in h2d_fields:
                host_in[f][...] = getattr(step_inputs, f)
            out = eng.step(None, fields=h2d_fields, copy=False)
        return out

    for s in range(min(args.warmup, 5)):
        out = e2e_step(s)
    d2h_bytes = out.nbytes()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_e2e0 = time.perf_counter()
    for i in range(e2e_steps):
        t0 = time.perf_counter()
        out = e2e_step(args.warmup + i)
        lat.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t_e2e0
    if world > 1:
        dist.barrier()

    # ---- per-kernel device times (CUDA events between the kernels, plain stream launches) ----
    prof = []
    for _ in range(6):
        eng.upload(batch)
        stream.synchronize()
        prof.append(eng.solve_profiled())
    prof = prof[1:]
    kern_ms = {k: statistics.median(p[k] for p in prof) for k in prof[0]}
    eng.stream.synchronize()
    prof_res = eng.download()
    P_prof = prof_res.trace[:, :K_sqp, _lib.TRACE_PCG_ITERATIONS]

    # ---- max over ranks ----
    agg = torch.tensor([dev_ms, e2e_s, wall1 - wall0], dtype=torch.float64, device=coll_device)
    if world > 1:
        dist.all_reduce(agg, op=dist.ReduceOp.MAX)
        gathered = sharding.gather_results(res_last, [M] * world, rank, world, device=coll_device)
    else:
        gathered = res_last
    dev_ms_max, e2e_s_max, wall_max = (float(v) for v in agg.tolist())

    if rank == 0:
        units_per_step = world * M * K_sqp
        value = units_per_step * args.steps / (dev_ms_max * 1e-3)
        e2e_value = units_per_step * e2e_steps / e2e_s_max
        ms_per_step = dev_ms_max / args.steps
        # roofline of the dominant kernel
        fp64_peak = measure_fp64_peak()
        peaks = {}
        peaks_file = ROOT / "MEASURED_PEAKS.json"
        if peaks_file.exists():
            peaks = json.loads(peaks_file.read_text())
        hbm_peak, hbm_src = (peaks["hbm_gbs"], "MEASURED_PEAKS.json") if "hbm_gbs" in peaks else (6650.0, "fallback")
        fam_flops = {
            "linearize": M * K_sqp * N * F_LIN,
            "schur": M * K_sqp * (N * F_SCHUR + (N + 1) * F_PREC + F_HESS),
            "pcg": float(np.sum(P_prof) * f_pcg(N) + M * K_sqp * N * F_REC),
            "linesearch": M * K_sqp * 9 * N * F_LS,
        }
        fam_ms = {"linearize": kern_ms["linearize"], "schur": kern_ms["schur"] + kern_ms["hessinv"],
                  "pcg": kern_ms["pcg"], "linesearch": kern_ms["linesearch"]}
        dominant = max(fam_ms, key=fam_ms.get)
        # the PCG family (model_ops.cuh: launch_pcg): quadrants of O^ in registers up to N = 64, one thread
        # per block row above
        pcg_kernel = "k_pcg_q" if N <= 64 else "k_pcg"
        kernel_names = {"linearize": "k_lin_tangent_iiwa", "schur": "k_schur", "pcg": pcg_kernel,
                        "linesearch": "k_linesearch"}
        launches_dom = K_sqp
        achieved = fam_flops[dominant] / (fam_ms[dominant] * 1e-3) / 1e12
        total_flops = float(np.sum([flops_solve_iteration(N, p) for p in P_prof.reshape(-1)]))
        # compulsory HBM bytes of a solve-iteration in the fused-in-L2 design
        alg_bytes = (3 * (N + 1) * 14 + 2 * N * 7 + N * 3 + 441) * 8 * M * K_sqp
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.workload}: {w['desc']}", "model": "iiwa14", "batch_per_gpu": M,
                       "global_batch": M * world, "horizon": N, "timestep": h, "sqp_iterations_per_step": K_sqp,
                       "pcg_tolerance": 1e-6, "line_search_candidates": 9, "parallelism": f"dp{world} (solves sharded)",
                       "l2": "256 MiB buffer written between timed steps (L2 flushed, untimed)",
                       "loop_mode": {1: "cuda-graph WHILE node", 2: "cuda-graph unrolled", 3: "stream launches"}[eng.loop_mode]},
            "sqp_iteration_rate_hz": K_sqp * 1e3 / ms_per_step, "solves_per_sec": world * M * 1e3 / ms_per_step,
            "p50_latency_ms": 1e3 * statistics.median(lat), "p90_latency_ms": 1e3 * sorted(lat)[int(0.9 * (len(lat) - 1))],
            "wall_ms_per_step_incl_flush": 1e3 * wall_max / args.steps,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d_bytes),
                    "d2h_bytes_per_step": int(d2h_bytes), "ms_per_step": 1e3 * e2e_s_max / e2e_steps},
            "gpu_launches": int(launches_per_step * args.steps),
            "gpu_launches_per_step": int(launches_per_step),
            "clocks": clocks.summary(),
            "roofline": {
                "bound": "fp64", "kernel": kernel_names[dominant],
                "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved / fp64_peak,
                "peak_source": "in-run DFMA probe (gato_measure_fp64_peak); MEASURED_PEAKS.json carries no fp64 figure",
                "launch_ms": fam_ms[dominant] / launches_dom, "algorithmic_flops_per_launch": fam_flops[dominant] / launches_dom,
                "traffic": ncu_traffic(args.workload, kernel_names[dominant]),
                "hbm": {"achieved": alg_bytes / (kern_ms["total"] * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                        "frac": alg_bytes / (kern_ms["total"] * 1e-3) / 1e9 / hbm_peak, "peak_source": hbm_src,
                        "algorithmic_bytes_per_step": alg_bytes},
                "step": {"achieved": total_flops / (kern_ms["total"] * 1e-3) / 1e12, "unit": "TFLOP/s",
                         "frac": total_flops / (kern_ms["total"] * 1e-3) / 1e12 / fp64_peak,
                         "algorithmic_flops_per_step": total_flops},
            },
            "kernel_ms_per_step": {k: round(v, 5) for k, v in kern_ms.items()},
            "kernel_tflops": {k: fam_flops[k] / (fam_ms[k] * 1e-3) / 1e12 for k in fam_flops},
            "pcg_iterations_mean": float(np.mean(pcg_last)),
            "all_solves_ok": status_ok and bool(np.all(gathered.info[:, _lib.INFO_STATUS] == 0)),
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(w, batch, args.cpu_budget_s)
            line["e2e_speedup_vs_cpu_baseline"] = e2e_value / line["cpu_baseline"]["value"]
            try:   # the compiled arm is an extra: never let it take the bench line down
                line["cpu_baseline_c"] = cpu_baseline_c(w, batch, min(args.cpu_budget_s, 10.0))
                line["e2e_speedup_vs_cpu_baseline_c"] = e2e_value / line["cpu_baseline_c"]["value"]
            except Exception as exc:  # noqa: BLE001
                line["cpu_baseline_c"] = {"unavailable": f"{type(exc).__name__}: {exc}"}
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse_args()
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    w = workload_config(args)
    if args.impl == "reference":
        run_reference_arm(args, w, rank, world)
        return
    run_gpu_arm(args, w, rank, local_rank, world)


if __name__ == "__main__":
    main()
