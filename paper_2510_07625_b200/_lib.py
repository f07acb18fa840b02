"""ctypes binding of libgato_b200.so (include/gato_b200.h).  Fails loudly: there is no CPU
fallback anywhere in this package."""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import BackendUnavailableError

ABI_VERSION = 1
FLAG_UNFUSED = 1      # gato_config.flags: keep form_schur in its own kernel, write the plain stage arrays
FLAG_FUSED = 2        # gato_config.flags: Schur formation inside the PCG kernel also for small batches
FLAG_UNTIMED = 4      # gato_config.flags: no CUDA events around the solve's launch (gato_last_solve_ms unavailable)
INFO_WORDS = 8
TRACE_WORDS = 8
(INFO_N_RECORDS, INFO_CONVERGED, INFO_STATUS, INFO_FAIL_ITER, INFO_FAIL_KNOT, INFO_FAIL_BLOCK,
 INFO_FAIL_AUX, INFO_RETRIES) = range(8)
(TRACE_MERIT, TRACE_CONSTRAINT_L1, TRACE_ALPHA, TRACE_RHO, TRACE_PCG_ITERATIONS, TRACE_ACCEPTED,
 TRACE_STEP_INF_NORM, TRACE_ITERATION) = range(8)
STATUS_OK, STATUS_FACTORIZATION, STATUS_PCG_BREAKDOWN = 0, 1, 2
BLOCK_Q, BLOCK_R, BLOCK_S = 0, 1, 2


class GatoConfig(C.Structure):
    _fields_ = [
        ("abi_version", C.c_int32), ("model_id", C.c_int32), ("batch", C.c_int32),
        ("horizon", C.c_int32), ("state_dim", C.c_int32), ("control_dim", C.c_int32),
        ("force_dim", C.c_int32), ("max_sqp_iterations", C.c_int32),
        ("pcg_max_iterations", C.c_int32), ("num_shrinks", C.c_int32),
        ("regularize_r", C.c_int32), ("pcg_retry_limit", C.c_int32), ("loop_mode", C.c_int32),
        ("flags", C.c_int32),
        ("timestep", C.c_double), ("pcg_tolerance", C.c_double), ("mu", C.c_double),
        ("beta", C.c_double), ("rho_min", C.c_double), ("rho_max", C.c_double),
        ("rho_factor", C.c_double), ("step_tolerance", C.c_double),
        ("feasibility_tolerance", C.c_double), ("model_params", C.c_double * 8),
    ]


class GatoBuffers(C.Structure):
    _fields_ = [(name, C.c_void_p) for name in (
        "x_start", "goal", "Q", "R", "QN", "force", "rho_init", "X", "U", "trace", "info")]


EXPORTS = {
    "gato_version": (C.c_char_p, []),
    "gato_create": (C.c_int, [C.POINTER(GatoConfig), C.POINTER(C.c_void_p)]),
    "gato_bind": (C.c_int, [C.c_void_p, C.POINTER(GatoBuffers)]),
    "gato_solve": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gato_solve_mpc": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_int64, C.c_int64]),
    "gato_shift_warm_start": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gato_solve_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                  C.c_void_p, C.c_void_p, C.c_int64]),
    "gato_merit_candidates": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "gato_best_of_batch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "gato_mpc_advance": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64]),
    "gato_pending": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_int32)]),
    "gato_resume": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    "gato_loop_mode": (C.c_int, [C.c_void_p]),
    "gato_fused": (C.c_int, [C.c_void_p]),
    "gato_scratch": (C.c_int, [C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
    "gato_read_scratch": (C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.c_int64]),
    "gato_launch_count": (C.c_int64, [C.c_void_p]),
    "gato_last_solve_ms": (C.c_int, [C.c_void_p, C.POINTER(C.c_float)]),
    "gato_solve_profiled": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_float)]),
    "gato_measure_fp64_peak": (C.c_int, [C.POINTER(C.c_double)]),
    "gato_last_error": (C.c_char_p, [C.c_void_p]),
    "gato_destroy": (None, [C.c_void_p]),
    "gato_step_many": (C.c_int, [C.c_int32, C.POINTER(C.c_double), C.c_int64, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p]),
    "gato_select_hypothesis": (C.c_int, [C.c_int32, C.POINTER(C.c_double), C.c_int32, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_double, C.c_int32, C.c_int32, C.c_void_p,
                                         C.c_void_p, C.c_void_p]),
    "gato_step_jacobians_many": (C.c_int, [C.c_int32, C.POINTER(C.c_double), C.c_int64, C.c_void_p,
                                           C.c_void_p, C.c_void_p, C.c_double, C.c_void_p,
                                           C.c_void_p, C.c_void_p]),
    "gato_btmv_batched": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p]),
    "gato_pcg_batched": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int32,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p]),
}

_LIB = None


def library_path() -> Path:
    override = os.environ.get("GATO_B200_LIB")
    if override:
        return Path(override)
    return Path(__file__).resolve().parent / "lib" / "libgato_b200.so"


def load():
    """Load the shared library and bind every symbol include/gato_b200.h declares."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = library_path()
    if not path.exists():
        raise BackendUnavailableError(
            f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a). This package has no CPU fallback.")
    try:
        lib = C.CDLL(str(path))
    except OSError as exc:
        raise BackendUnavailableError(f"cannot load {path}: {exc}") from exc
    for name, (restype, argtypes) in EXPORTS.items():
        try:
            fn = getattr(lib, name)
        except AttributeError as exc:
            raise BackendUnavailableError(f"{path} does not export {name}") from exc
        fn.restype = restype
        fn.argtypes = argtypes
    _LIB = lib
    return lib
