"""ORACLE (test infrastructure, never shipped on the product path).

ctypes front end of oracle/trajopt_c.c: the compiled C (POSIX threads) restatement of the reference's
batched SQP solve for the iiwa14 model.  Same algorithm as
oracle/trajopt_np.py (bitwise-pinned to the reference); used as the fast checker for full-size
batches in tests/ and as the second CPU arm of bench.py."""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "lib" / "libtrajopt_c.so"
_LIB = None


class Settings(C.Structure):
    _fields_ = [("max_sqp_iterations", C.c_int32), ("pcg_max_iterations", C.c_int32), ("num_shrinks", C.c_int32),
                ("regularize_r", C.c_int32), ("pcg_retry_limit", C.c_int32), ("pcg_tolerance", C.c_double),
                ("mu", C.c_double), ("beta", C.c_double), ("rho_min", C.c_double), ("rho_max", C.c_double),
                ("rho_factor", C.c_double), ("step_tolerance", C.c_double), ("feasibility_tolerance", C.c_double)]


def build() -> Path:
    subprocess.run(["make", "-C", str(HERE)], check=True, capture_output=True)
    return LIB_PATH


def load():
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            build()
        lib = C.CDLL(str(LIB_PATH))
        dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int32)
        lib.trajopt_c_solve_batch.argtypes = [C.c_int32, C.c_int32, C.c_double, dp, dp, dp, dp, dp, dp, dp, dp, dp,
                                              C.POINTER(Settings), dp, ip, C.c_int32]
        lib.trajopt_c_solve_batch.restype = C.c_int
        lib.trajopt_c_deriv.argtypes = [dp, dp, dp, dp]
        lib.trajopt_c_rk4_jac.argtypes = [dp, dp, dp, C.c_double, dp, dp, dp]
        lib.trajopt_c_threads.restype = C.c_int
        _LIB = lib
    return _LIB


def make_settings(st) -> Settings:
    """From oracle.trajopt_np.Settings (or any object with the reference's SolverSettings fields)."""
    cap = getattr(st, "pcg_max_iterations", None)
    tol = getattr(st, "step_tolerance", None)
    return Settings(int(st.max_sqp_iterations), int(cap) if cap else 0, int(st.num_shrinks), int(bool(st.regularize_r)),
                    int(st.pcg_retry_limit), float(st.pcg_tolerance), float(st.mu), float(st.beta), float(st.rho_min),
                    float(st.rho_max), float(st.rho_factor), float("nan") if tol is None else float(tol),
                    float(st.feasibility_tolerance))


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def solve_batch(x_start, goal, Q, R, QN, force, rho_init, X, U, h, st, threads: int = 0):
    """M iiwa14 solves (arrays as in paper_2510_07625_b200.PackedBatch).  Returns (X, U, trace, info) with
    trace [M, max_it, 8] in the row layout of include/gato_b200.h and info [M, 4] =
    (n_records, converged, status, fail_iteration)."""
    lib = load()
    cs = st if isinstance(st, Settings) else make_settings(st)
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (x_start, goal, Q, R, QN, force, rho_init)]
    M, N = arrs[1].shape[0], arrs[1].shape[1] - 1
    Xo = np.array(X, dtype=np.float64, order="C", copy=True)
    Uo = np.array(U, dtype=np.float64, order="C", copy=True)
    trace = np.full((M, cs.max_sqp_iterations, 8), np.nan)
    info = np.zeros((M, 4), dtype=np.int32)
    rc = lib.trajopt_c_solve_batch(M, N, float(h), *(_p(a) for a in arrs), _p(Xo), _p(Uo), C.byref(cs), _p(trace),
                                   info.ctypes.data_as(C.POINTER(C.c_int32)), int(threads))
    if rc != 0:
        raise RuntimeError(f"trajopt_c_solve_batch failed ({rc})")
    return Xo, Uo, trace, info


def threads() -> int:
    return int(load().trajopt_c_threads())


def deriv(x, u, f):
    lib = load()
    x, u, f = (np.ascontiguousarray(a, dtype=np.float64) for a in (x, u, f))
    out = np.empty(14)
    lib.trajopt_c_deriv(_p(x), _p(u), _p(f), _p(out))
    return out


def rk4_and_jacobians(x, u, f, h):
    lib = load()
    x, u, f = (np.ascontiguousarray(a, dtype=np.float64) for a in (x, u, f))
    out, A, B = np.empty(14), np.empty((14, 14)), np.empty((14, 7))
    lib.trajopt_c_rk4_jac(_p(x), _p(u), _p(f), float(h), _p(out), _p(A), _p(B))
    return out, A, B
