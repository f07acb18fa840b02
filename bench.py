#!/usr/bin/env python
"""bench.py -- headline benchmark of the batched SQP solve (BASELINE.json metric).

    python bench.py --gpus N --steps K --warmup W [--workload c2] [--impl reference]

One "step" = one batched solve call over one batch of synthetic iiwa14 problems
(SURVEY.md section 8d).  Metric: solve-iterations per second (solves x SQP iterations completed per
second, whole job over all GPUs); the batched SQP iteration rate (Hz), solves/s and p50 call latency
are reported beside it.

N = 1 (default): workload c2 = BASELINE.json configs[1]: MPC tracking, batch 32, N = 32 knots, one SQP
iteration per control step, warm-started by the device-side shift of the previous solution.  The same
process also times the throughput configurations c3 (batch 128, N = 64: configs[2]) and c5 (batch 1024,
N = 64: the per-GPU shard of configs[4]) and reports them under "configs", each with its own value, e2e
and roofline.

N > 1: one process per GPU.  Launched by the driver under torchrun (RANK / LOCAL_RANK / WORLD_SIZE in
the environment); started WITHOUT them, `--gpus N` re-executes itself under torch.distributed.run with
N ranks.  Default workload c5 = configs[4]: batch 1024 per GPU, N = 64, solves sharded by contiguous
batch-index range, no collective on the solve path, final gather of X, U, trace, info to rank 0 (weak
scaling: "value").  The line also carries the strong-scaling run (4096 solves in total split over the
ranks) and, for both, the same workload timed on rank 0 alone while the others wait ("n1": the
single-GPU number the N-GPU number is to be read against).  On a box with fewer GPUs than ranks (or with
GATO_DIST_BACKEND=gloo) the ranks wrap around the visible devices and the collectives go through gloo.

Rank 0 prints ONE JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
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
STRONG_TOTAL = 4096          # configs[4]: batch 1024-4096 sharded by solve
METRIC = "sqp_solve_iterations_per_sec"
UNIT = "solve-iterations/s"
PCG_TOL, PCG_CAP, CANDIDATES = 1e-6, 200, 9

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
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS),
                    help="default: c2 on one GPU, c5 on several")
    ap.add_argument("--batch", type=int, default=None, help="override the per-GPU batch size")
    ap.add_argument("--horizon", type=int, default=None)
    ap.add_argument("--sqp-iters", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra-configs", action="store_true", help="N = 1: skip the c3 / c5 sub-records")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    return ap.parse_args()


def workload_name(args):
    return args.workload or ("c2" if args.gpus <= 1 else "c5")


def workload_config(args, name=None):
    w = dict(WORKLOADS[name or workload_name(args)])
    if name is None:
        if args.batch:
            w["M"] = args.batch
        if args.horizon:
            w["N"] = args.horizon
        if args.sqp_iters:
            w["sqp"] = args.sqp_iters
    return w


def config_dict(name, w, world):
    """The `config` object of the JSON line: identical in the GPU arm and in the reference arm."""
    return {"workload": f"{name}: {w['desc']}", "model": "iiwa14", "batch_per_gpu": w["M"],
            "global_batch": w["M"] * world, "horizon": w["N"], "timestep": w["h"],
            "sqp_iterations_per_step": w["sqp"], "pcg_tolerance": PCG_TOL, "pcg_max_iterations": PCG_CAP,
            "line_search_candidates": CANDIDATES, "parallelism": f"dp{world} (solves sharded by batch index)",
            "sequence": ("MPC: every step starts from the previous step's solution shifted one knot, measured "
                         "state = predicted next state, goal window advanced" if w["kind"] == "track"
                         else "every step solves the batch from its cold initial guess"),
            "l2": "GPU arm: a 256 MiB buffer is written between timed steps (L2 flushed, untimed)",
            "timing": "GPU arm: CUDA events recorded by bench.py on the launching stream around every step; the "
                      "library's own per-launch event pair is switched off (GATO_FLAG_UNTIMED)"}


def make_batch(w, M, lo=0, seed_offset=0):
    """Solves [lo, lo + M) of the workload's global batch (any batch is a prefix of a larger one)."""
    from paper_2510_07625_b200 import workloads
    if w["kind"] == "track":
        full = workloads.iiwa14_track_arrays(lo + M, w["N"], w["h"], seed=workloads.SEED + seed_offset)
    else:
        full = workloads.iiwa14_reach_arrays(lo + M, w["N"], seed=workloads.SEED + seed_offset)
    return full.slice(lo, lo + M) if lo else full


def tracking_reference(w, steps, seed):
    """Goal windows of consecutive control steps: (steps, N+1, 14) from the same generator."""
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
    """SM clock and throttle reasons of one GPU during the timed region (NVML), sampled by the timing
    loop itself right after it has enqueued a step, so every timed step contributes a sample taken while
    the GPU is busy."""

    REASONS = {
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
        0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting", 0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.dev = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.dev, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def sample(self):
        if self.nv is None:
            return
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.dev, self.nv.NVML_CLOCK_SM))
            mask = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.dev)
            for bit, name in self.REASONS.items():
                if mask & bit:
                    self.reasons.add(name)
        except Exception:
            pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_min_mhz": float(min(self.samples)),
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------------------
# CPU arm: the reference's own CPU implementation (baseline/_ref, installed by build()) when it is
# there, else its bitwise-pinned numpy port (oracle/trajopt_np.py); all host cores
# --------------------------------------------------------------------------------------

class CpuArm:
    """The workload as the CPU implementation sees it: one step = `count` of the batch's solves, solved by
    `batch_solve(spec, workers)` (batch.py:102-124: forked pool, one task per problem).  For the tracking
    workload the steps form the same MPC sequence as on the GPU: the next step starts from this step's
    solution shifted one knot (mpc.py:85-89), with the predicted next state as the measurement and the goal
    window advanced."""

    def __init__(self, name, w, count=None):
        from oracle import ref_bridge
        self.name, self.w = name, w
        self.tb = ref_bridge.load()
        self.kind = "reference" if self.tb is not None else "port"
        self.cores = os.cpu_count() or 1
        self.batch = make_batch(w, w["M"])
        self.count = min(count or w["M"], w["M"])
        self.step_index = 0
        if w["kind"] == "track":
            from paper_2510_07625_b200 import workloads
            self.path = tracking_reference(w, 4096, workloads.SEED)
        self.X = self.batch.X[:self.count].copy()
        self.U = self.batch.U[:self.count].copy()
        self.x_start = self.batch.x_start[:self.count].copy()
        self.goal = self.batch.goal[:self.count].copy()

    def _solve(self, workers):
        """-> (wall seconds of the batch call, sum of per-solve seconds, X, U)."""
        w, c = self.w, self.count
        from paper_2510_07625_b200.engine import PackedBatch
        b = self.batch
        cur = PackedBatch(self.x_start, self.goal, b.Q[:c], b.R[:c], b.QN[:c], b.force[:c], b.rho_init[:c],
                          self.X, self.U)
        if self.tb is not None:
            from oracle import ref_bridge
            problems, inits = ref_bridge.problems_from_arrays(cur, w["h"])
            st = ref_bridge.fixed_budget_settings(w["sqp"], PCG_TOL, PCG_CAP)
            spec = self.tb.BatchSpec.with_rho_inits(problems, inits, st, list(b.rho_init[:c]))
            out = self.tb.batch_solve(spec, workers=workers)
            assert out.ok, out.errors
            X = np.stack([r.X for r in out.results])
            U = np.stack([r.U for r in out.results])
            return out.wall_time, float(sum(out.solve_times)), X, U
        from oracle import trajopt_np as orc
        from oracle.iiwa14_np import Iiwa14
        probs = [orc.Problem(Iiwa14(), cur.Q[i], cur.R[i], cur.QN[i], cur.goal[i], w["N"], w["h"], cur.x_start[i],
                             cur.force[i]) for i in range(c)]
        st = orc.Settings(max_sqp_iterations=w["sqp"], pcg_tolerance=PCG_TOL, pcg_max_iterations=PCG_CAP,
                          step_tolerance=None)
        t0 = time.perf_counter()
        res, errors, wall = orc.solve_batch_parallel(probs, [(cur.X[i], cur.U[i]) for i in range(c)], [st] * c, workers)
        assert all(e is None for e in errors), errors
        return wall, time.perf_counter() - t0, np.stack([r.X for r in res]), np.stack([r.U for r in res])

    def step(self, workers=None, advance=True):
        wall, solve_sum, X, U = self._solve(self.cores if workers is None else workers)
        if advance and self.w["kind"] == "track":
            N = self.w["N"]
            self.x_start = X[:, 1, :].copy()
            self.X = np.concatenate([X[:, 1:], X[:, -1:]], axis=1)
            self.U = np.concatenate([U[:, 1:], U[:, -1:]], axis=1)
            self.step_index += 1
            self.goal = np.broadcast_to(self.path[self.step_index:self.step_index + N + 1],
                                        self.goal.shape).copy()
        return wall, solve_sum

    def describe(self, extra=""):
        src = ("unmodified reference package (baseline/_ref: trajbatch.batch_solve, oracle iiwa14 model behind its "
               "DynamicsModel interface)" if self.kind == "reference"
               else "numpy port of the reference (oracle/trajopt_np.py, bitwise-pinned)")
        return (f"{self.count} of the workload's {self.w['M']} solves x {self.w['sqp']} SQP iteration(s) per step, "
                f"{src}, forked pool of {self.cores} workers{extra}")


def cpu_baseline(name, w, budget_s):
    """cpu_baseline of the GPU line: bounded sample, all cores; plus the single-worker leg of the reference's
    own protocol (batch.py:153-168: wall time and sum(solve_times) / workers)."""
    arm = CpuArm(name, w)
    t_cal, _ = arm.step()                                   # also warms the imports
    if t_cal * 3 > budget_s and arm.count > arm.cores:      # too slow for the budget: one solve per core
        arm = CpuArm(name, w, count=arm.cores)
        t_cal, _ = arm.step()
    reps = max(1, min(5, int(budget_s / max(t_cal, 1e-3)) - 1))
    runs = [arm.step() for _ in range(reps)]
    t = statistics.median(r[0] for r in runs)
    units = arm.count * w["sqp"]
    out = {"value": units / t, "unit": UNIT, "cores": arm.cores, "kind": arm.kind,
           "sample": arm.describe(f", median of {reps} step(s) after 1 warm-up"),
           "seconds_per_sample": t, "wall_time_s": t,
           "sum_solve_times_over_workers_s": statistics.median(r[1] for r in runs) / arm.cores}
    # w = 1 leg on a slice that keeps it within the budget
    n1 = max(1, min(arm.count, int(arm.count * (0.5 * budget_s) / max(t * arm.cores, 1e-3))))
    one = CpuArm(name, w, count=n1)
    w1, s1 = one.step(workers=1, advance=False)
    out["workers_1"] = {"value": n1 * w["sqp"] / w1, "unit": UNIT, "cores": 1, "solves": n1, "wall_time_s": w1,
                        "sum_solve_times_over_workers_s": s1}
    return out


def cpu_baseline_c(w, budget_s):
    """Second CPU arm: the compiled C restatement of the same algorithm (oracle/trajopt_c.c, POSIX threads
    over the solves) on all host cores, bounded sample.  Not the reference's own implementation (that is
    the arm above); reported so that the GPU/CPU ratio can also be read against compiled code."""
    from oracle import trajopt_c as oc
    from oracle import trajopt_np as orc
    batch = make_batch(w, w["M"])
    cores = os.cpu_count() or 1
    st = orc.Settings(max_sqp_iterations=w["sqp"], pcg_tolerance=PCG_TOL, pcg_max_iterations=PCG_CAP,
                      step_tolerance=None)
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


def run_reference_arm(args):
    """bench.py --impl reference: the reference's CPU implementation of the path timed on the host cores, on
    the GPU arm's config and sequence.  Each step solves the whole batch when `warmup + steps` of them fit the
    time budget (c1, c2), otherwise a bounded sample of it (one solve per core)."""
    name = workload_name(args)
    w = workload_config(args)
    arm = CpuArm(name, w)
    t_cal, _ = arm.step()
    budget = 240.0
    total = args.warmup + args.steps
    if t_cal * total > budget and arm.count > arm.cores:
        arm = CpuArm(name, w, count=arm.cores)
        t_cal, _ = arm.step()
    steps = max(1, min(args.steps, int(budget / max(t_cal, 1e-3)) - args.warmup))
    warm = min(args.warmup, max(0, int(budget / max(t_cal, 1e-3)) - steps))
    arm = CpuArm(name, w, count=arm.count)          # restart the sequence at control step 0
    for _ in range(warm):
        arm.step()
    runs = [arm.step() for _ in range(steps)]
    total_s = sum(r[0] for r in runs)
    units = arm.count * w["sqp"]
    value = steps * units / total_s
    one = CpuArm(name, w, count=min(arm.count, max(1, arm.cores // 4)))
    w1, s1 = one.step(workers=1, advance=False)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "requested_steps": args.steps, "warmup": warm, "ms_per_step": 1e3 * total_s / steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(name, w, max(1, args.gpus)),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": arm.cores, "kind": arm.kind,
                         "sample": arm.describe(), "solves_per_step": arm.count,
                         "full_batch": arm.count == w["M"],
                         "wall_time_s_per_step": total_s / steps,
                         "sum_solve_times_over_workers_s_per_step": sum(r[1] for r in runs) / steps / arm.cores,
                         "workers_1": {"value": one.count * w["sqp"] / w1, "unit": UNIT, "cores": 1,
                                       "solves": one.count, "wall_time_s": w1,
                                       "sum_solve_times_over_workers_s": s1}},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------------------

class GpuArm:
    """One engine + one shard of one workload on this rank's GPU."""

    def __init__(self, name, w, M, lo, device_index, loop_mode=0):
        import torch

        import paper_2510_07625_b200 as gb
        from paper_2510_07625_b200 import workloads
        self.torch, self.gb = torch, gb
        self.name, self.w, self.M, self.N, self.h, self.K = name, w, M, w["N"], w["h"], w["sqp"]
        self.track = w["kind"] == "track"
        self.device = torch.device("cuda", device_index)
        self.batch = make_batch(w, M, lo)
        self.eng = gb.BatchEngine(gb.Iiwa14(), M, self.N, self.h, workloads.fixed_budget_settings(self.K, PCG_TOL, PCG_CAP),
                                  device=device_index, loop_mode=loop_mode, timing=False)   # timed by this file's events
        self.stream = self.eng.stream
        self.ref_path = tracking_reference(w, 8192, workloads.SEED) if self.track else None
        self.ref_dev = torch.as_tensor(self.ref_path, device=self.device) if self.track else None
        self.X0 = torch.as_tensor(self.batch.X, device=self.device)
        self.U0 = torch.as_tensor(self.batch.U, device=self.device)

    def close(self):
        self.eng.close()

    def device_step(self, s):
        """Inputs resident in HBM.  track: MPC control step s (measured state = predicted next state, warm
        start = device shift, goal window advanced); reach: solve from the cold init."""
        eng = self.eng
        with self.torch.cuda.stream(self.stream):
            if self.track:
                eng.mpc_step(self.ref_dev, s)       # ONE launch: measured state, device shift, goal window + the solve
            else:
                eng.dev["X"].copy_(self.X0)
                eng.dev["U"].copy_(self.U0)
                eng.launch()

    def device_run(self, warmup, steps, flush, clocks=None, barrier=None):
        """K timed steps, CUDA events per step on the launching stream, L2 flushed between steps (untimed).
        -> (sum of the step times in ms, wall seconds incl. flushes, result of the last step)"""
        torch, eng, stream = self.torch, self.eng, self.stream
        eng.upload(self.batch)
        stream.synchronize()
        for s in range(warmup):
            self.device_step(s)
        eng.finish()
        stream.synchronize()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        if barrier:
            barrier()
        torch.cuda.synchronize()
        wall0 = time.perf_counter()
        for i in range(steps):
            with torch.cuda.stream(stream):
                flush.fill_(1.0)                      # evict L2 (126 MB) between timed steps, untimed
                starts[i].record(stream)
            self.device_step(warmup + i)
            ends[i].record(stream)
            if clocks is not None:
                clocks.sample()                       # the GPU is working on step i (or its flush) right now
        torch.cuda.synchronize()
        wall1 = time.perf_counter()
        if barrier:
            barrier()
        dev_ms = float(sum(a.elapsed_time(b) for a, b in zip(starts, ends)))
        return dev_ms, wall1 - wall0, eng.download()

    def e2e_run(self, warmup, steps, barrier=None):
        """The same steps through the array API with HOST buffers: BatchEngine.step = one gato_solve_host call
        (pinned H2D of the step's inputs, device shift, solve, D2H of X, U, trace, info).
        -> (seconds, per-call latencies, h2d bytes, d2h bytes)"""
        from paper_2510_07625_b200.engine import PackedBatch
        eng, batch, N = self.eng, self.batch, self.N
        eng.upload(batch)
        self.stream.synchronize()
        step_inputs = PackedBatch(batch.x_start.copy(), batch.goal.copy(), batch.Q, batch.R, batch.QN, batch.force,
                                  batch.rho_init, batch.X, batch.U)
        fields = ("x_start", "goal", "force") if self.track else ("x_start", "goal", "Q", "R", "QN", "force",
                                                                   "rho_init", "X", "U")
        h2d = sum(getattr(step_inputs, f).nbytes for f in fields)
        host_in = eng.host_inputs()      # pinned staging buffers of the inputs, written in place
        mirror = None
        if not self.track:               # the cold problem batch lives in its own pinned buffer: the engine's mirror
            mirror = eng.input_mirror()  # receives the results, which overwrite X and U
            mirror.write(step_inputs, fields)

        call = eng.bind_step(fields, shift=self.track, mirror=mirror)   # gato_solve_host with its arguments bound
        goal_in, x_in, path = host_in["goal"], host_in["x_start"], self.ref_path

        def step(s):
            if self.track:
                goal_in[...] = path[s:s + N + 1]               # this control step's goal window, every solve
                out = call()
                x_in[...] = out.X[:, 1, :]                     # "measured" state for the next control step
            else:
                out = call()
            return out

        for s in range(min(warmup, 5)):
            out = step(s)
        d2h = out.nbytes()
        if barrier:
            barrier()
        self.torch.cuda.synchronize()
        lat = []
        t_begin = time.perf_counter()
        for i in range(steps):
            t0 = time.perf_counter()
            out = step(warmup + i)
            lat.append(time.perf_counter() - t0)
        self.torch.cuda.synchronize()
        seconds = time.perf_counter() - t_begin
        if barrier:
            barrier()
        return seconds, lat, int(h2d), int(d2h)

    def profile(self, runs=5):
        """Per-kernel device times (CUDA events between the kernels, plain stream launches)."""
        from paper_2510_07625_b200 import _lib
        prof = []
        for _ in range(runs + 1):
            self.eng.upload(self.batch)
            self.stream.synchronize()
            prof.append(self.eng.solve_profiled())
        prof = prof[1:]
        kern_ms = {k: statistics.median(p[k] for p in prof) for k in prof[0]}
        self.stream.synchronize()
        res = self.eng.download()
        return kern_ms, res.trace[:, :self.K, _lib.TRACE_PCG_ITERATIONS]

    def roofline(self, kern_ms, P_prof, fp64_peak, hbm_peak, hbm_src):
        M, N, K = self.M, self.N, self.K
        fam_flops = {
            "linearize": M * K * N * F_LIN,
            "schur": M * K * (N * F_SCHUR + (N + 1) * F_PREC + F_HESS),
            "pcg": float(np.sum(P_prof) * f_pcg(N) + M * K * N * F_REC),
            "linesearch": M * K * 9 * N * F_LS,
        }
        fam_ms = {"linearize": kern_ms["linearize"], "schur": kern_ms["schur"] + kern_ms["hessinv"],
                  "pcg": kern_ms["pcg"], "linesearch": kern_ms["linesearch"]}
        fused = self.eng.fused
        if fused:
            # the Schur system is formed inside the PCG kernel: its flops and the (empty) k_schur launch belong to
            # that kernel's family; k_hessinv stays on its own
            fam_flops["pcg"] += M * K * (N * F_SCHUR + (N + 1) * F_PREC)
            fam_flops["schur"] = M * K * F_HESS
            fam_ms["pcg"] += kern_ms["schur"]
            fam_ms["schur"] = kern_ms["hessinv"]
        dominant = max(fam_ms, key=fam_ms.get)
        pcg_kernel = ("k_pcg_q<fused Schur>" if fused else "k_pcg_q") if N <= 64 else "k_pcg"
        names = {"linearize": "k_lin_tangent_iiwa", "schur": "k_hessinv" if fused else "k_schur", "pcg": pcg_kernel,
                 "linesearch": "k_linesearch"}
        achieved = fam_flops[dominant] / (fam_ms[dominant] * 1e-3) / 1e12
        total_flops = float(np.sum([flops_solve_iteration(N, p) for p in P_prof.reshape(-1)]))
        # compulsory HBM bytes of a solve-iteration in the fused-in-L2 design
        alg_bytes = (3 * (N + 1) * 14 + 2 * N * 7 + N * 3 + 441) * 8 * M * K
        total_s = kern_ms["total"] * 1e-3
        return {
            "bound": "fp64", "kernel": names[dominant],
            "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved / fp64_peak,
            "peak_source": "in-run DFMA probe (gato_measure_fp64_peak); MEASURED_PEAKS.json carries no fp64 figure",
            "launch_ms": fam_ms[dominant] / K, "algorithmic_flops_per_launch": fam_flops[dominant] / K,
            "traffic": ncu_traffic(self.name, names[dominant].split("<")[0]),
            "hbm": {"achieved": alg_bytes / total_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
                    "frac": alg_bytes / total_s / 1e9 / hbm_peak, "peak_source": hbm_src,
                    "algorithmic_bytes_per_step": alg_bytes},
            "step": {"achieved": total_flops / total_s / 1e12, "unit": "TFLOP/s",
                     "frac": total_flops / total_s / 1e12 / fp64_peak, "algorithmic_flops_per_step": total_flops},
            "fused_schur_pcg": bool(fused),
            "kernel_ms_per_step": {k: round(v, 5) for k, v in kern_ms.items()},
            "kernel_tflops": {k: fam_flops[k] / (fam_ms[k] * 1e-3) / 1e12 for k in fam_flops},
        }


def hbm_peak():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        try:
            return float(json.loads(f.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def stream_launch_check(name, w, device_index):
    """The same batch once through the default engine (CUDA-graph WHILE node) and once through a plain
    stream-launch engine (loop mode 3): the results must be bitwise identical.  The second run is what makes
    the repo's kernels visible to a profiler that does not enumerate kernels inside conditional graph nodes."""
    M = min(w["M"], 32)
    a = GpuArm(name, w, M, 0, device_index, loop_mode=0)
    b = GpuArm(name, w, M, 0, device_index, loop_mode=3)
    try:
        ra, rb = a.eng.solve(a.batch), b.eng.solve(b.batch)
        same = all(np.array_equal(getattr(ra, f), getattr(rb, f), equal_nan=True) for f in ("X", "U", "trace", "info"))
        return {"bitwise_equal": bool(same), "solves": M, "loop_modes": [a.eng.loop_mode, b.eng.loop_mode],
                "stream_launches": int(b.eng.launch_count())}
    finally:
        a.close()
        b.close()


def measure_config(name, w, M, lo, device_index, steps, warmup, flush, fp64_peak, world=1, barrier=None,
                   reduce_max=None, clocks=None):
    """value / e2e / roofline of one workload on this rank's shard; times are max over ranks."""
    from paper_2510_07625_b200 import _lib
    arm = GpuArm(name, w, M, lo, device_index)
    try:
        dev_ms, wall_s, res_last = arm.device_run(warmup, steps, flush, clocks=clocks, barrier=barrier)
        launches = arm.eng.launch_count()   # the control step's shift / goal window ride in the solve's first kernel
        e2e_s, lat, h2d, d2h = arm.e2e_run(warmup, steps, barrier=barrier)
        kern_ms, P_prof = arm.profile()
        if reduce_max:
            dev_ms, e2e_s, wall_s = reduce_max([dev_ms, e2e_s, wall_s])
        units = world * M * arm.K
        ms_per_step = dev_ms / steps
        peak_hbm, hbm_src = hbm_peak()
        rec = {
            "value": units * steps / (dev_ms * 1e-3), "unit": UNIT, "ms_per_step": ms_per_step, "steps": steps,
            "warmup": warmup,
            "sqp_iteration_rate_hz": arm.K * 1e3 / ms_per_step, "solves_per_sec": world * M * 1e3 / ms_per_step,
            "p50_latency_ms": 1e3 * statistics.median(lat), "p90_latency_ms": 1e3 * sorted(lat)[int(0.9 * (len(lat) - 1))],
            "wall_ms_per_step_incl_flush": 1e3 * wall_s / steps,
            "e2e": {"value": units * steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": 1e3 * e2e_s / steps},
            "gpu_launches": int(launches * steps), "gpu_launches_per_step": int(launches),
            "roofline": arm.roofline(kern_ms, P_prof, fp64_peak, peak_hbm, hbm_src),
            "pcg_iterations_mean": float(np.mean(res_last.trace[:, :arm.K, _lib.TRACE_PCG_ITERATIONS])),
            "all_solves_ok": bool(np.all(res_last.info[:, _lib.INFO_STATUS] == 0)),
            "loop_mode": {1: "cuda-graph WHILE node", 2: "cuda-graph unrolled", 3: "stream launches"}[arm.eng.loop_mode],
        }
        return rec, res_last
    finally:
        arm.close()


def device_only(name, w, M, lo, device_index, steps, warmup, flush):
    arm = GpuArm(name, w, M, lo, device_index)
    try:
        dev_ms, _, _ = arm.device_run(warmup, steps, flush)
        return {"value": M * arm.K * steps / (dev_ms * 1e-3), "unit": UNIT, "ms_per_step": dev_ms / steps,
                "batch": M, "steps": steps}
    finally:
        arm.close()


def run_gpu_arm(args, rank, local_rank, world):
    import torch
    import torch.distributed as dist

    from paper_2510_07625_b200 import sharding
    from paper_2510_07625_b200.engine import measure_fp64_peak

    ndev = torch.cuda.device_count()
    if ndev < 1:
        raise SystemExit("bench.py: no CUDA device (the solve has no CPU path)")
    # fewer GPUs than ranks (or GATO_DIST_BACKEND=gloo): ranks wrap around the visible devices and the
    # collectives go through host memory -- the multi-rank path exercised on a small box
    backend = os.environ.get("GATO_DIST_BACKEND") or ("nccl" if ndev >= world else "gloo")
    device_index = local_rank % ndev
    torch.cuda.set_device(device_index)
    device = torch.device("cuda", device_index)
    coll_device = device if backend == "nccl" else torch.device("cpu")
    if world > 1:
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")          # communicator log: "... nranks N ..." per rank
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(backend)

    def barrier():
        if world > 1:
            dist.barrier()

    def reduce_max(values):
        t = torch.tensor(values, dtype=torch.float64, device=coll_device)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(v) for v in t.tolist()]

    name = workload_name(args)
    w = workload_config(args)
    M = w["M"]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)
    fp64_peak = measure_fp64_peak()
    clocks = ClockSampler(device_index)

    # ---- the headline workload: this rank's contiguous shard [rank*M, (rank+1)*M) of the global batch ----
    rec, res_last = measure_config(name, w, M, rank * M, device_index, args.steps, args.warmup, flush, fp64_peak,
                                   world=world, barrier=barrier, reduce_max=reduce_max, clocks=clocks)
    gathered = sharding.gather_results(res_last, [M] * world, rank, world, device=coll_device) if world > 1 else res_last

    extra = {}
    if world > 1:
        # strong scaling: STRONG_TOTAL solves in total, split into contiguous shards
        sub_steps = max(3, min(args.steps, 10))
        bounds = sharding.shard_bounds(STRONG_TOTAL, world)
        lo, hi = bounds[rank]
        arm = GpuArm(name, w, hi - lo, lo, device_index)
        try:
            dev_ms, _, res_s = arm.device_run(min(args.warmup, 3), sub_steps, flush, barrier=barrier)
        finally:
            arm.close()
        (dev_ms,) = reduce_max([dev_ms])
        g = sharding.gather_results(res_s, [b - a for a, b in bounds], rank, world, device=coll_device)
        extra["strong"] = {"global_batch": STRONG_TOTAL, "batch_per_gpu": hi - lo, "steps": sub_steps,
                           "value": STRONG_TOTAL * arm.K * sub_steps / (dev_ms * 1e-3), "unit": UNIT,
                           "ms_per_step": dev_ms / sub_steps, "scaling": "strong",
                           "gathered_rows": None if g is None else int(g.X.shape[0])}
        # the same two workloads on ONE GPU (rank 0 alone, the other ranks wait at the barrier)
        if rank == 0:
            extra["n1"] = {"weak": device_only(name, w, M, 0, device_index, sub_steps, min(args.warmup, 3), flush),
                           "strong": device_only(name, w, STRONG_TOTAL, 0, device_index, max(3, sub_steps // 2), 2, flush)}
        barrier()

    if rank == 0:
        line = {
            "metric": METRIC, "value": rec["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": rec["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(name, w, world),
        }
        for k in ("sqp_iteration_rate_hz", "solves_per_sec", "p50_latency_ms", "p90_latency_ms",
                  "wall_ms_per_step_incl_flush", "e2e", "gpu_launches", "gpu_launches_per_step", "loop_mode"):
            line[k] = rec[k]
        line["clocks"] = clocks.summary()
        line["roofline"] = {k: v for k, v in rec["roofline"].items() if k not in ("kernel_ms_per_step", "kernel_tflops")}
        line["fused_schur_pcg"] = rec["roofline"]["fused_schur_pcg"]
        line["kernel_ms_per_step"] = rec["roofline"]["kernel_ms_per_step"]
        line["kernel_tflops"] = rec["roofline"]["kernel_tflops"]
        line["pcg_iterations_mean"] = rec["pcg_iterations_mean"]
        line["all_solves_ok"] = rec["all_solves_ok"] and bool(np.all(gathered.info[:, 2] == 0))
        line["dist"] = {"backend": backend if world > 1 else None, "ranks": world, "visible_gpus": ndev,
                        "gathered_rows": int(gathered.X.shape[0])}
        line.update(extra)
        line["stream_launch_check"] = stream_launch_check(name, w, device_index)
        if world == 1 and not args.no_extra_configs and args.workload is None:
            # the throughput configurations, timed in the same process (configs[2] and the per-GPU shard of configs[4])
            line["configs"] = {}
            for sub in ("c3", "c5"):
                ws = workload_config(args, sub)
                sub_steps = max(3, min(args.steps, 20 if sub == "c3" else 10))
                srec, _ = measure_config(sub, ws, ws["M"], 0, device_index, sub_steps, min(args.warmup, 3), flush,
                                         fp64_peak)
                srec["config"] = config_dict(sub, ws, 1)
                if not args.no_cpu_baseline:
                    try:
                        srec["cpu_baseline_c"] = cpu_baseline_c(ws, 4.0)
                        srec["e2e_speedup_vs_cpu_baseline_c"] = srec["e2e"]["value"] / srec["cpu_baseline_c"]["value"]
                    except Exception as exc:  # noqa: BLE001
                        srec["cpu_baseline_c"] = {"unavailable": f"{type(exc).__name__}: {exc}"}
                line["configs"][sub] = srec
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(name, w, args.cpu_budget_s)
            line["e2e_speedup_vs_cpu_baseline"] = rec["e2e"]["value"] / line["cpu_baseline"]["value"]
            try:   # the compiled arm is an extra: never let it take the bench line down
                line["cpu_baseline_c"] = cpu_baseline_c(w, min(args.cpu_budget_s, 10.0))
                line["e2e_speedup_vs_cpu_baseline_c"] = rec["e2e"]["value"] / line["cpu_baseline_c"]["value"]
            except Exception as exc:  # noqa: BLE001
                line["cpu_baseline_c"] = {"unavailable": f"{type(exc).__name__}: {exc}"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def respawn(args):
    """`python bench.py --gpus N` (N > 1) outside torchrun: launch the N ranks ourselves."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse_args()
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":       # CPU arm: rank 0 alone runs and prints it, the other ranks exit 0
        if rank == 0:
            run_reference_arm(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(respawn(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    run_gpu_arm(args, rank, local_rank, world)


if __name__ == "__main__":
    main()
