"""Device engine: one gato handle + its device/pinned buffers for a fixed
(model, M, N, timestep, settings) configuration on one GPU.

torch is used for device memory, pinned host staging and streams only; every kernel runs
behind the C ABI (include/gato_b200.h).  The array-level API here is what an MPC loop uses
(buffers stay resident between control steps); `batch.batch_solve`
is the reference-typed wrapper on top of it.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import BackendUnavailableError
from .models import device_model
from .settings import SolverSettings

# inputs of one batch, in the order they are staged host->device
INPUT_FIELDS = ("x_start", "goal", "Q", "R", "QN", "force", "rho_init", "X", "U")


@dataclass
class PackedBatch:
    """Host arrays of one homogeneous batch (C-contiguous float64).

    x_start (M, n) | goal (M, N+1, n) | Q (M, n, n) | R (M, m, m) | QN (M, n, n) |
    force (M, N, fdim) | rho_init (M,) | X (M, N+1, n) | U (M, N, m)
    """

    x_start: np.ndarray
    goal: np.ndarray
    Q: np.ndarray
    R: np.ndarray
    QN: np.ndarray
    force: np.ndarray
    rho_init: np.ndarray
    X: np.ndarray
    U: np.ndarray

    @property
    def size(self) -> int:
        return self.x_start.shape[0]

    def slice(self, lo: int, hi: int) -> "PackedBatch":
        return PackedBatch(*(getattr(self, f)[lo:hi] for f in INPUT_FIELDS))

    def nbytes(self) -> int:
        return sum(getattr(self, f).nbytes for f in INPUT_FIELDS)


@dataclass
class PackedResult:
    X: np.ndarray         # (M, N+1, n)
    U: np.ndarray         # (M, N, m)
    trace: np.ndarray     # (M, max_it, TRACE_WORDS)
    info: np.ndarray      # (M, INFO_WORDS) int32
    device_ms: float

    def nbytes(self) -> int:
        return self.X.nbytes + self.U.nbytes + self.trace.nbytes + self.info.nbytes


def _torch():
    try:
        import torch
    except ImportError as exc:  # pragma: no cover
        raise BackendUnavailableError("torch is required for device buffers") from exc
    if not torch.cuda.is_available():
        raise BackendUnavailableError(
            "no CUDA device visible: the batched SQP solve runs only on the GPU (no CPU fallback)")
    return torch


def make_config(model, M: int, N: int, timestep: float, settings: SolverSettings,
                loop_mode: int = 0, stage_arrays: bool = False, fused: bool | None = None,
                timing: bool = True) -> _lib.GatoConfig:
    model_id, params = device_model(model)
    cfg = _lib.GatoConfig()
    cfg.abi_version = _lib.ABI_VERSION
    cfg.model_id = model_id
    cfg.batch = M
    cfg.horizon = N
    cfg.state_dim = model.state_dim
    cfg.control_dim = model.control_dim
    cfg.force_dim = model.force_dim
    cfg.max_sqp_iterations = settings.max_sqp_iterations
    cfg.pcg_max_iterations = settings.pcg.max_iterations or 0
    cfg.num_shrinks = settings.line_search.num_shrinks
    cfg.regularize_r = int(settings.regularize_r)
    cfg.pcg_retry_limit = settings.pcg_retry_limit
    cfg.loop_mode = loop_mode
    cfg.flags = _lib.FLAG_UNFUSED if (stage_arrays or fused is False) else (_lib.FLAG_FUSED if fused else 0)
    if not timing:
        cfg.flags |= _lib.FLAG_UNTIMED
    cfg.timestep = float(timestep)
    cfg.pcg_tolerance = settings.pcg.tolerance
    cfg.mu = settings.line_search.mu
    cfg.beta = settings.line_search.beta
    cfg.rho_min = settings.rho_min
    cfg.rho_max = settings.rho_max
    cfg.rho_factor = settings.rho_factor
    cfg.step_tolerance = math.nan if settings.step_tolerance is None else settings.step_tolerance
    cfg.feasibility_tolerance = settings.feasibility_tolerance
    for i in range(8):
        cfg.model_params[i] = float(params[i])
    return cfg


class BatchEngine:
    """gato_create + gato_bind for one configuration; solve() is H2D -> gato_solve -> D2H."""

    def __init__(self, model, M: int, N: int, timestep: float, settings: SolverSettings,
                 device: int | None = None, loop_mode: int = 0, stage_arrays: bool = False,
                 fused: bool | None = None, timing: bool = True):
        """``timing=False``: no CUDA events around the solve's launch (they cost ~5 us of device time per launch);
        ``device_ms`` of the results is then NaN.  ``stage_arrays=True`` keeps the Schur formation in its own kernel so that ``scratch()`` can read
        Sdiag, Soff, Linv, Lfac and the matrix record (stage-by-stage parity tests); by default solves with
        diagonal weights form their Schur system inside the PCG kernel (from batch x horizon ~ 3000 block rows
        on, where it pays; ``fused=True`` / ``False`` forces either path) and those arrays are not written."""
        torch = _torch()
        self.lib = _lib.load()
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.model, self.M, self.N = model, M, N
        self.settings = settings
        n, m, fd = model.state_dim, model.control_dim, model.force_dim
        self.shapes = {
            "x_start": (M, n), "goal": (M, N + 1, n), "Q": (M, n, n), "R": (M, m, m),
            "QN": (M, n, n), "force": (M, N, fd), "rho_init": (M,),
            "X": (M, N + 1, n), "U": (M, N, m),
        }
        max_it = settings.max_sqp_iterations
        # One device arena and one pinned mirror, laid out so that every transfer of the hot loop is
        # ONE copy:  [x_start goal force | Q R QN rho_init | X U | trace info]
        #   per-step MPC inputs = the first three fields, full upload = everything up to U,
        #   download = X .. info.
        self.layout = ("x_start", "goal", "force", "Q", "R", "QN", "rho_init", "X", "U", "trace", "info")
        shapes = dict(self.shapes)
        shapes["trace"] = (M, max_it, _lib.TRACE_WORDS)
        info_doubles = (M * _lib.INFO_WORDS + 1) // 2          # int32 words stored in 8-byte slots
        self.offsets, off = {}, 0
        for name in self.layout:
            count = info_doubles if name == "info" else int(np.prod(shapes[name]))
            self.offsets[name] = (off, count)
            off += count + (count & 1)                         # keep every field 16-byte aligned
        self.arena_doubles = off
        with torch.cuda.device(self.device):
            self.arena = torch.zeros(off, dtype=torch.float64, device=self.device)
            self.pinned = torch.zeros(off, dtype=torch.float64).pin_memory()

            def view(buf, name):
                o, c = self.offsets[name]
                if name == "info":
                    return buf[o:o + c].view(torch.int32)[:M * _lib.INFO_WORDS].view(M, _lib.INFO_WORDS)
                return buf[o:o + c].view(shapes[name])
            self.dev = {name: view(self.arena, name) for name in self.layout}
            self.pin = {name: view(self.pinned, name) for name in self.layout}
            self.pin_np = {name: t.numpy() for name, t in self.pin.items()}
            self.stream = torch.cuda.Stream(device=self.device)
            self._step_calls = {}
            cfg = make_config(model, M, N, timestep, settings, loop_mode, stage_arrays, fused, timing)
            handle = C.c_void_p()
            rc = self.lib.gato_create(C.byref(cfg), C.byref(handle))
            self.handle = handle
            if rc != 0:
                msg = self.lib.gato_last_error(handle).decode() if handle else "gato_create failed"
                if handle:
                    self.lib.gato_destroy(handle)
                self.handle = None
                raise RuntimeError(f"gato_create: {msg} (code {rc})")
            bufs = _lib.GatoBuffers()
            for name in ("x_start", "goal", "Q", "R", "QN", "force", "rho_init", "X", "U", "trace", "info"):
                setattr(bufs, name, self.dev[name].data_ptr())
            self._check(self.lib.gato_bind(self.handle, C.byref(bufs)), "gato_bind")

    # -- plumbing --------------------------------------------------------------- #
    def _check(self, rc: int, what: str):
        if rc != 0:
            raise RuntimeError(f"{what}: {self.lib.gato_last_error(self.handle).decode()} (code {rc})")

    def close(self):
        if getattr(self, "handle", None):
            self.torch.cuda.synchronize(self.device)
            self.lib.gato_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    @property
    def loop_mode(self) -> int:
        return int(self.lib.gato_loop_mode(self.handle))

    @property
    def fused(self) -> bool:
        """True if solves with diagonal weights form their Schur system inside the PCG kernel (gato_fused)."""
        return bool(self.lib.gato_fused(self.handle))

    # -- staged steps (all asynchronous on self.stream) ---------------------------- #
    def _span(self, first: str, last: str) -> slice:
        return slice(self.offsets[first][0], self.offsets[last][0] + self.offsets[last][1])

    def upload(self, batch: PackedBatch, fields=INPUT_FIELDS):
        """Host -> pinned -> device for the named inputs: one contiguous copy when the fields are
        adjacent in the arena (the per-step MPC inputs x_start, goal, force; or everything)."""
        torch = self.torch
        for name in fields:
            src = getattr(batch, name)
            if src.shape != self.shapes[name]:
                raise ValueError(f"{name}: expected shape {self.shapes[name]}, got {src.shape}")
            self.pin_np[name][...] = src
        order = [n for n in self.layout if n in fields]
        with torch.cuda.stream(self.stream):
            i = 0
            while i < len(order):          # maximal runs of adjacent fields
                j = i
                while j + 1 < len(order) and self.layout.index(order[j + 1]) == self.layout.index(order[j]) + 1:
                    j += 1
                span = self._span(order[i], order[j])
                self.arena[span].copy_(self.pinned[span], non_blocking=True)
                i = j + 1

    def launch(self):
        """gato_solve on the engine stream; loops on the device until every solve terminated."""
        self._check(self.lib.gato_solve(self.handle, C.c_void_p(self.stream.cuda_stream)), "gato_solve")

    def finish(self):
        """Loop modes without a device-side WHILE: run extra passes if a PCG retry used one."""
        if self.loop_mode == 1:
            return
        pending = C.c_int32(0)
        stream = C.c_void_p(self.stream.cuda_stream)
        guard = self.settings.max_sqp_iterations * (self.settings.pcg_retry_limit + 1) + 1
        while guard > 0:
            self._check(self.lib.gato_pending(self.handle, stream, C.byref(pending)), "gato_pending")
            if pending.value == 0:
                break
            self._check(self.lib.gato_resume(self.handle, stream, 1), "gato_resume")
            guard -= 1

    def download(self) -> PackedResult:
        """Device -> pinned -> host for X, U, trace, info: one copy."""
        torch = self.torch
        span = self._span("X", "info")
        with torch.cuda.stream(self.stream):
            self.pinned[span].copy_(self.arena[span], non_blocking=True)
        self.stream.synchronize()
        ms = C.c_float(0.0)
        # device time of the last launch()/mpc_step(); step() (gato_solve_host) is timed by its caller
        timed = self.lib.gato_last_solve_ms(self.handle, C.byref(ms)) == 0
        return PackedResult(self.pin_np["X"].copy(), self.pin_np["U"].copy(), self.pin_np["trace"].copy(),
                            self.pin_np["info"].copy(), float(ms.value) if timed else float("nan"))

    def solve(self, batch: PackedBatch) -> PackedResult:
        """The end-to-end call: host inputs in, host results out."""
        self.upload(batch)
        self.launch()
        self.finish()
        return self.download()

    STEP_FIELDS = ("x_start", "goal", "force")

    def input_mirror(self) -> "InputMirror":
        """A second pinned staging buffer for the inputs, laid out like the engine's own.  The engine's mirror
        receives the results, so its X and U are overwritten by every step; a caller that solves from the same
        (or separately prepared) initial iterate again and again keeps it here and passes it to ``step(mirror=)``."""
        return InputMirror(self)

    def step(self, batch: PackedBatch | None, fields=STEP_FIELDS, shift: bool = False,
             copy: bool = True, mirror: "InputMirror | None" = None) -> PackedResult:
        """One control step with host buffers in ONE call across the C ABI (gato_solve_host): the named
        inputs (a contiguous run of the arena; default: the per-step MPC inputs x_start, goal, force) go
        host -> pinned -> device, the warm start is optionally shifted on the device (mpc.py:85-89), the
        solve runs to termination and X, U, trace, info come back.  copy=False returns views of the
        pinned mirror, valid until the next call.  ``mirror``: read the inputs from this staging buffer
        (``input_mirror()``) instead of the engine's own."""
        if mirror is not None:
            return self._step_from(mirror, batch, fields, shift, copy)
        call = self._step_calls.get(fields) if isinstance(fields, tuple) else None
        if call is None:           # the argument list of a field set is built once: this is the control loop's call
            order = [n for n in self.layout if n in fields]
            idx = [self.layout.index(n) for n in order]
            if idx != list(range(idx[0], idx[0] + len(idx))):
                raise ValueError("step(): the uploaded fields must be adjacent in the arena; use upload() + launch()")
            cin, cout = self._span(order[0], order[-1]), self._span("X", "info")
            base_d, base_h = self.arena.data_ptr(), self.pinned.data_ptr()
            head = (self.handle, C.c_void_p(self.stream.cuda_stream), C.c_void_p(base_d + 8 * cin.start),
                    C.c_void_p(base_h + 8 * cin.start), 8 * (cin.stop - cin.start))
            tail = (C.c_void_p(base_d + 8 * cout.start), C.c_void_p(base_h + 8 * cout.start),
                    8 * (cout.stop - cout.start))
            call = (head, tail)
            self._step_calls[tuple(fields)] = call
        if batch is not None:      # None: the caller has written the inputs into host_inputs() already
            for name in fields:
                src = getattr(batch, name)
                if src.shape != self.shapes[name]:
                    raise ValueError(f"{name}: expected shape {self.shapes[name]}, got {src.shape}")
                self.pin_np[name][...] = src
        rc = self.lib.gato_solve_host(*call[0], 1 if shift else 0, *call[1])
        if rc != 0:
            self._check(rc, "gato_solve_host")
        pin = self.pin_np
        if copy:
            return PackedResult(pin["X"].copy(), pin["U"].copy(), pin["trace"].copy(), pin["info"].copy(), float("nan"))
        return PackedResult(pin["X"], pin["U"], pin["trace"], pin["info"], float("nan"))

    def bind_step(self, fields=STEP_FIELDS, shift: bool = False, mirror: "InputMirror | None" = None):
        """The control loop's call, bound once: returns ``f() -> PackedResult`` (views of the pinned mirror, valid
        until the next call) that does exactly ``step(None, fields, shift, copy=False, mirror=mirror)`` without
        rebuilding the argument list -- the inputs are written into ``host_inputs()`` (or the mirror) beforehand."""
        order = [n for n in self.layout if n in fields]
        idx = [self.layout.index(n) for n in order]
        if idx != list(range(idx[0], idx[0] + len(idx))):
            raise ValueError("step(): the uploaded fields must be adjacent in the arena; use upload() + launch()")
        cin, cout = self._span(order[0], order[-1]), self._span("X", "info")
        base_d = self.arena.data_ptr()
        base_in = (self.pinned if mirror is None else mirror.pinned).data_ptr()
        args = (self.handle, C.c_void_p(self.stream.cuda_stream), C.c_void_p(base_d + 8 * cin.start),
                C.c_void_p(base_in + 8 * cin.start), 8 * (cin.stop - cin.start), 1 if shift else 0,
                C.c_void_p(base_d + 8 * cout.start), C.c_void_p(self.pinned.data_ptr() + 8 * cout.start),
                8 * (cout.stop - cout.start))
        fn, check = self.lib.gato_solve_host, self._check
        pin = self.pin_np
        result = PackedResult(pin["X"], pin["U"], pin["trace"], pin["info"], float("nan"))

        def call():
            rc = fn(*args)
            if rc != 0:
                check(rc, "gato_solve_host")
            return result
        return call

    def _step_from(self, mirror, batch, fields, shift, copy):
        order = [n for n in self.layout if n in fields]
        idx = [self.layout.index(n) for n in order]
        if idx != list(range(idx[0], idx[0] + len(idx))):
            raise ValueError("step(): the uploaded fields must be adjacent in the arena; use upload() + launch()")
        if batch is not None:
            mirror.write(batch, fields)
        cin, cout = self._span(order[0], order[-1]), self._span("X", "info")
        base_d = self.arena.data_ptr()
        self._check(self.lib.gato_solve_host(
            self.handle, C.c_void_p(self.stream.cuda_stream), C.c_void_p(base_d + 8 * cin.start),
            C.c_void_p(mirror.pinned.data_ptr() + 8 * cin.start), 8 * (cin.stop - cin.start), 1 if shift else 0,
            C.c_void_p(base_d + 8 * cout.start), C.c_void_p(self.pinned.data_ptr() + 8 * cout.start),
            8 * (cout.stop - cout.start)), "gato_solve_host")
        pin = self.pin_np
        get = (lambda a: a.copy()) if copy else (lambda a: a)
        return PackedResult(get(pin["X"]), get(pin["U"]), get(pin["trace"]), get(pin["info"]), float("nan"))

    def host_inputs(self) -> dict:
        """Writable numpy views of the pinned staging buffers of the inputs (x_start, goal, force, Q, R, QN,
        rho_init, X, U): fill them in place and call ``step(None, fields=...)`` to skip one host copy."""
        return {name: self.pin_np[name] for name in INPUT_FIELDS}

    def merit_candidates(self, dX=None, dU=None):
        """(merits, violations), each (M, num_shrinks + 2): the L1 merit (sqp.py:118-166) of the candidates
        X + beta^-c dX, c = 0..num_shrinks, followed by the merit of the uploaded iterate itself, evaluated
        by the line-search kernel alone (gato_merit_candidates).  dX, dU: host arrays or None (zero step)."""
        torch = self.torch
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            ddx = None if dX is None else torch.as_tensor(np.ascontiguousarray(dX, dtype=float)).to(self.device)
            ddu = None if dU is None else torch.as_tensor(np.ascontiguousarray(dU, dtype=float)).to(self.device)
            if ddx is not None and tuple(ddx.shape) != self.shapes["X"]:
                raise ValueError(f"dX: expected shape {self.shapes['X']}")
            if ddu is not None and tuple(ddu.shape) != self.shapes["U"]:
                raise ValueError(f"dU: expected shape {self.shapes['U']}")
            self._check(self.lib.gato_merit_candidates(
                self.handle, C.c_void_p(self.stream.cuda_stream),
                C.c_void_p(ddx.data_ptr()) if ddx is not None else None,
                C.c_void_p(ddu.data_ptr()) if ddu is not None else None), "gato_merit_candidates")
        self.stream.synchronize()
        width = self.settings.line_search.num_shrinks + 2
        return self.scratch("merits").reshape(self.M, width), self.scratch("viols").reshape(self.M, width)

    def best_of_batch(self) -> tuple[int, float]:
        """(index, final merit) of the best solve of the last batch, selected on the device
        (gato_best_of_batch; mpc.py:283-298): lowest final merit among the solves that did not fail,
        first minimum on ties; index -1 if every solve failed."""
        torch = self.torch
        with torch.cuda.device(self.device):
            if not hasattr(self, "_best"):
                self._best = (torch.zeros(1, dtype=torch.int32, device=self.device),
                              torch.zeros(1, dtype=torch.float64, device=self.device))
            bi, bm = self._best
            self._check(self.lib.gato_best_of_batch(self.handle, C.c_void_p(self.stream.cuda_stream),
                                                    C.c_void_p(bi.data_ptr()), C.c_void_p(bm.data_ptr())),
                        "gato_best_of_batch")
            self.stream.synchronize()
            return int(bi.item()), float(bm.item())

    def _goal_path_args(self, goal_path):
        ptr, plen, stride = None, 0, 0
        if goal_path is not None:
            if not (goal_path.is_cuda and goal_path.dtype == self.torch.float64 and goal_path.is_contiguous()):
                raise ValueError("goal_path must be a contiguous CUDA float64 tensor")
            n = self.shapes["x_start"][1]
            if goal_path.dim() == 2 and goal_path.shape[1] == n:
                plen, stride = goal_path.shape[0], 0
            elif goal_path.dim() == 3 and goal_path.shape[0] == self.M and goal_path.shape[2] == n:
                plen, stride = goal_path.shape[1], goal_path.shape[1] * n
            else:
                raise ValueError(f"goal_path must have shape (T, {n}) or ({self.M}, T, {n})")
            ptr = C.c_void_p(goal_path.data_ptr())
        return ptr, plen, stride

    def mpc_advance(self, goal_path=None, step: int = 0):
        """One control period on the device, in place (gato_mpc_advance): x_start <- X[:, 1], X and U
        shifted (mpc.py:85-89) and, with ``goal_path`` (a CUDA float64 tensor [T, n] shared by all solves or
        [M, T, n]), the goal window advanced to goal_path[step : step + N + 1] (clamped at the end)."""
        ptr, plen, stride = self._goal_path_args(goal_path)
        self._check(self.lib.gato_mpc_advance(self.handle, C.c_void_p(self.stream.cuda_stream), ptr, int(plen),
                                              int(stride), int(step)), "gato_mpc_advance")

    def mpc_step(self, goal_path=None, step: int = 0):
        """One control period AND its solve in one launch (gato_solve_mpc, shift mode 2): what ``mpc_advance`` does
        rides in the first kernel of the solve's graph.  Same arguments as ``mpc_advance``; asynchronous like
        ``launch`` (follow with ``finish`` / ``download``).  ``goal_path=None``: shift and state hand-over only."""
        ptr, plen, stride = self._goal_path_args(goal_path)
        self._check(self.lib.gato_solve_mpc(self.handle, C.c_void_p(self.stream.cuda_stream), 2, ptr, int(plen),
                                            int(stride), int(step)), "gato_solve_mpc")

    def shift_warm_start(self):
        """X, U <- shifted one knot left with the tail duplicated, on the device (mpc.py:85-89)."""
        self._check(self.lib.gato_shift_warm_start(self.handle, C.c_void_p(self.stream.cuda_stream)),
                    "gato_shift_warm_start")

    KERNEL_FAMILIES = ("hessinv", "linearize", "schur", "pcg", "linesearch", "update", "prologue", "total")

    def solve_profiled(self) -> dict:
        """One solve in plain stream-launch mode with CUDA events between the kernels: device
        milliseconds per kernel family, summed over the passes (inputs must be uploaded)."""
        ms = (C.c_float * 8)()
        self._check(self.lib.gato_solve_profiled(self.handle, C.c_void_p(self.stream.cuda_stream), ms),
                    "gato_solve_profiled")
        return dict(zip(self.KERNEL_FAMILIES, (float(v) for v in ms)))

    def launch_count(self) -> int:
        self.stream.synchronize()
        return int(self.lib.gato_launch_count(self.handle))

    def scratch(self, name: str) -> np.ndarray:
        """Copy an internal stage array to the host (parity tests)."""
        torch = self.torch
        ptr, count = C.c_void_p(), C.c_int64()
        self._check(self.lib.gato_scratch(self.handle, name.encode(), C.byref(ptr), C.byref(count)),
                    "gato_scratch")
        self.stream.synchronize()
        is_int = name in ("si", "pcg_iters")
        dtype, width = (np.int32, 4) if is_int else (np.float64, 8)
        if name == "counters":
            dtype, width = np.uint32, 4
        out = np.empty(count.value, dtype=dtype)
        self._check(self.lib.gato_read_scratch(self.handle, name.encode(), C.c_void_p(out.ctypes.data),
                                               count.value * width), "gato_read_scratch")
        return out


# ------------------------------------------------------------------------------------
# stateless operators (dynamics.step_many / step_jacobians_many / blocktri.pcg on the GPU)
# ------------------------------------------------------------------------------------

def _dev(torch, arr, dtype=None):
    arr = np.ascontiguousarray(arr, dtype=dtype or np.float64)
    if arr.size == 0:        # e.g. the off-diagonal stack of a single-block-row system
        return torch.zeros(1, dtype=torch.float64, device="cuda")
    return torch.as_tensor(arr).cuda()


class InputMirror:
    """Pinned host staging of an engine's inputs (same layout as the engine's own mirror); see
    ``BatchEngine.input_mirror``."""

    def __init__(self, eng: "BatchEngine"):
        torch = eng.torch
        self.shapes = eng.shapes
        self.pinned = torch.zeros(eng.offsets["U"][0] + eng.offsets["U"][1] + 1, dtype=torch.float64).pin_memory()
        self.arrays = {}
        for name in INPUT_FIELDS:
            o, c = eng.offsets[name]
            self.arrays[name] = self.pinned[o:o + c].view(eng.shapes[name]).numpy()

    def write(self, batch: PackedBatch, fields=INPUT_FIELDS):
        for name in fields:
            src = getattr(batch, name)
            if src.shape != self.shapes[name]:
                raise ValueError(f"{name}: expected shape {self.shapes[name]}, got {src.shape}")
            self.arrays[name][...] = src


def measure_fp64_peak() -> float:
    """Sustained fp64 FMA TFLOP/s of the current GPU (register-resident DFMA probe)."""
    _torch()
    out = C.c_double(0.0)
    rc = _lib.load().gato_measure_fp64_peak(C.byref(out))
    if rc != 0:
        raise RuntimeError(f"gato_measure_fp64_peak failed ({rc})")
    return float(out.value)


def step_many(model, X, U, h: float, F) -> np.ndarray:
    """Row-wise RK4 steps on the GPU (dynamics.py:805-816)."""
    torch = _torch()
    lib = _lib.load()
    model_id, params = device_model(model)
    X = np.ascontiguousarray(X, dtype=float)
    rows = X.shape[0]
    dX, dU, dF = _dev(torch, X), _dev(torch, U), _dev(torch, F)
    out = torch.empty_like(dX)
    p = (C.c_double * 8)(*params)
    rc = lib.gato_step_many(model_id, p, rows, dX.data_ptr(), dU.data_ptr(), dF.data_ptr(), float(h),
                            out.data_ptr(), C.c_void_p(torch.cuda.current_stream().cuda_stream))
    if rc != 0:
        raise RuntimeError(f"gato_step_many failed ({rc})")
    return out.cpu().numpy()


def select_hypothesis(model, x_prev, u_applied, x_meas, forces, control_period: float, h_plant: float = 0.001,
                      position_only: bool = False, return_errors: bool = False):
    """Index of the candidate force whose one-period plant prediction best matches the measurement
    (mpc.select_hypothesis, mpc.py:130-147; plant = fixed-substep RK4, dynamics.py:820-864), computed on
    the GPU by gato_select_hypothesis.  ``forces``: (M, force_dim) constant candidates (a
    ``HypothesisSet.forces`` array); ties break toward the lowest index."""
    torch = _torch()
    lib = _lib.load()
    model_id, params = device_model(model)
    ratio = control_period / h_plant
    substeps = round(ratio)
    if h_plant <= 0 or substeps < 1 or abs(ratio - substeps) > 1e-9 * max(1.0, abs(ratio)):
        raise ValueError(f"control period {control_period} is not an integer multiple of plant substep {h_plant}")
    forces = np.ascontiguousarray(forces, dtype=float)
    if forces.ndim != 2 or forces.shape[1] != model.force_dim:
        raise ValueError(f"forces must have shape (M, {model.force_dim})")
    xs = [np.ascontiguousarray(v, dtype=float).reshape(-1) for v in (x_prev, u_applied, x_meas)]
    if xs[0].size != model.state_dim or xs[1].size != model.control_dim or xs[2].size != model.state_dim:
        raise ValueError("x_prev, u_applied, x_meas do not match the model dimensions")
    dxp, du, dxm, df = (_dev(torch, v) for v in (*xs, forces))
    M = forces.shape[0]
    err = torch.empty(M, dtype=torch.float64, device="cuda")
    best = torch.empty(1, dtype=torch.int32, device="cuda")
    p = (C.c_double * 8)(*params)
    rc = lib.gato_select_hypothesis(model_id, p, M, dxp.data_ptr(), du.data_ptr(), dxm.data_ptr(), df.data_ptr(),
                                    float(h_plant), int(substeps), 1 if position_only else 0, err.data_ptr(),
                                    best.data_ptr(), C.c_void_p(torch.cuda.current_stream().cuda_stream))
    if rc != 0:
        raise RuntimeError(f"gato_select_hypothesis failed ({rc})")
    idx = int(best.item())
    return (idx, err.cpu().numpy()) if return_errors else idx


def step_jacobians_many(model, X, U, h: float, F):
    """Row-wise exact RK4 Jacobians on the GPU (dynamics.py:774-802)."""
    torch = _torch()
    lib = _lib.load()
    model_id, params = device_model(model)
    X = np.ascontiguousarray(X, dtype=float)
    rows, n = X.shape
    m = model.control_dim
    dX, dU, dF = _dev(torch, X), _dev(torch, U), _dev(torch, F)
    A = torch.empty((rows, n, n), dtype=torch.float64, device="cuda")
    B = torch.empty((rows, n, m), dtype=torch.float64, device="cuda")
    p = (C.c_double * 8)(*params)
    rc = lib.gato_step_jacobians_many(model_id, p, rows, dX.data_ptr(), dU.data_ptr(), dF.data_ptr(),
                                      float(h), A.data_ptr(), B.data_ptr(),
                                      C.c_void_p(torch.cuda.current_stream().cuda_stream))
    if rc != 0:
        raise RuntimeError(f"gato_step_jacobians_many failed ({rc})")
    return A.cpu().numpy(), B.cpu().numpy()


def pcg_batched(S_diag, S_off, gamma, P_diag, P_off, tolerance: float, max_iterations: int | None = None):
    """Batched PCG on explicit block-tridiagonal systems (blocktri.py:123-173).

    S_diag, P_diag: (systems, nb, bd, bd); S_off, P_off: (systems, nb-1, bd, bd);
    gamma: (systems, nb*bd).  Returns (lam, iterations, converged, status, residual)."""
    torch = _torch()
    lib = _lib.load()
    S_diag = np.ascontiguousarray(S_diag, dtype=float)
    systems, nb, bd, _ = S_diag.shape
    d = [_dev(torch, a) for a in (S_diag, S_off, gamma, P_diag, P_off)]
    lam = torch.empty((systems, nb * bd), dtype=torch.float64, device="cuda")
    its = torch.empty(systems, dtype=torch.int32, device="cuda")
    conv = torch.empty(systems, dtype=torch.int32, device="cuda")
    status = torch.empty(systems, dtype=torch.int32, device="cuda")
    res = torch.empty(systems, dtype=torch.float64, device="cuda")
    rc = lib.gato_pcg_batched(systems, nb, bd, *(t.data_ptr() for t in d), float(tolerance),
                              int(max_iterations or 0), lam.data_ptr(), its.data_ptr(), conv.data_ptr(),
                              status.data_ptr(), res.data_ptr(),
                              C.c_void_p(torch.cuda.current_stream().cuda_stream))
    if rc != 0:
        raise RuntimeError(f"gato_pcg_batched failed ({rc})")
    return (lam.cpu().numpy(), its.cpu().numpy(), conv.cpu().numpy().astype(bool), status.cpu().numpy(),
            res.cpu().numpy())
