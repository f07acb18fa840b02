"""Where the host side of one end-to-end control step (BatchEngine.step = gato_solve_host) goes: the call with
and without its copies, and the Python-side input writes.   python scripts/e2e_breakdown.py"""
import ctypes as C
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2510_07625_b200 as gb  # noqa: E402
from paper_2510_07625_b200 import workloads  # noqa: E402

w = bench.WORKLOADS["c2"]
M, N = w["M"], w["N"]
batch = bench.make_batch(w, M)
eng = gb.BatchEngine(gb.Iiwa14(), M, N, w["h"], workloads.fixed_budget_settings(1))
eng.upload(batch)
eng.stream.synchronize()
path = bench.tracking_reference(w, 4096, workloads.SEED)
host_in = eng.host_inputs()
fields = ("x_start", "goal", "force")


def timed(fn, n=300):
    for _ in range(20):
        fn()
    ts = []
    for i in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e6 * statistics.median(ts)


s = [0]


def full():
    host_in["goal"][...] = path[s[0]:s[0] + N + 1][None]
    out = eng.step(None, fields=fields, shift=True, copy=False)
    host_in["x_start"][...] = out.X[:, 1, :]
    s[0] += 1


def call_only():
    eng.step(None, fields=fields, shift=True, copy=False)


def writes_only():
    host_in["goal"][...] = path[s[0]:s[0] + N + 1][None]
    host_in["x_start"][...] = eng.pin_np["X"][:, 1, :]


cin, cout = eng._span("x_start", "force"), eng._span("X", "info")
base_d, base_h = eng.arena.data_ptr(), eng.pinned.data_ptr()


def raw(in_bytes, out_bytes, shift=1):
    eng._check(eng.lib.gato_solve_host(
        eng.handle, C.c_void_p(eng.stream.cuda_stream),
        C.c_void_p(base_d + 8 * cin.start), C.c_void_p(base_h + 8 * cin.start), in_bytes, shift,
        C.c_void_p(base_d + 8 * cout.start), C.c_void_p(base_h + 8 * cout.start), out_bytes), "gato_solve_host")


nin, nout = 8 * (cin.stop - cin.start), 8 * (cout.stop - cout.start)
eng.launch(); eng.stream.synchronize()
dev = []
for _ in range(50):
    eng.launch()
    eng.stream.synchronize()
    dev.append(1e3 * eng.download().device_ms)
print(f"device time of the solve alone (CUDA events)      {statistics.median(dev):7.1f} us")
print(f"full e2e step (writes + call)                      {timed(full):7.1f} us")
print(f"BatchEngine.step call only                         {timed(call_only):7.1f} us")
print(f"Python-side input writes only                      {timed(writes_only):7.1f} us")
print(f"gato_solve_host, both copies ({nin} B in, {nout} B out) {timed(lambda: raw(nin, nout)):7.1f} us")
print(f"gato_solve_host, no copies                         {timed(lambda: raw(0, 0)):7.1f} us")
print(f"gato_solve_host, H2D only                          {timed(lambda: raw(nin, 0)):7.1f} us")
print(f"gato_solve_host, D2H only                          {timed(lambda: raw(0, nout)):7.1f} us")
print(f"gato_solve_host, no copies, no shift               {timed(lambda: raw(0, 0, 0)):7.1f} us")
eng.close()
