"""Batch engine: the drop-in for the reference's ``batch_solve`` / ``sqp_solve``
(/root/reference/pkg/src/trajbatch/batch.py:25-124, sqp.py:204-295) on B200.

``batch_solve(spec, workers)`` takes the reference's own types (or the mirrors defined in
this package), runs every solve on the GPU and returns results in input order with the
reference's per-slot error isolation: ``results[i] is None`` exactly when ``errors[i]`` is an
``"ExcType: message"`` string (batch.py:92-99).  ``workers`` is accepted for signature
compatibility; parallelism is over the whole batch on the device(s).
"""

from __future__ import annotations

import dataclasses
import time
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from . import _lib
from .engine import BatchEngine, PackedBatch, PackedResult
from .models import device_model
from .problem import ProblemSpec
from .results import BatchResult, IterationRecord, SqpResult
from .settings import SolverSettings


@dataclass
class BatchSpec:
    """M problems + initial trajectories + settings (batch.py:25-74): homogeneous n, m, N;
    ``overrides[i]`` replaces the shared settings for problem i."""

    problems: list
    inits: list
    settings: SolverSettings
    overrides: list | None = None

    def __post_init__(self):
        if len(self.problems) < 1:
            raise ValueError("batch must contain at least one problem")
        if len(self.inits) != len(self.problems):
            raise ValueError("need one initial trajectory per problem")
        if self.overrides is not None and len(self.overrides) != len(self.problems):
            raise ValueError("overrides must align with problems")
        first = self.problems[0]
        for p in self.problems[1:]:
            if (p.model.state_dim != first.model.state_dim
                    or p.model.control_dim != first.model.control_dim
                    or p.horizon != first.horizon):
                raise ValueError("batch problems must share n, m and horizon")

    @property
    def size(self) -> int:
        return len(self.problems)

    def effective_settings(self, i: int) -> SolverSettings:
        if self.overrides is not None and self.overrides[i] is not None:
            return self.overrides[i]
        return self.settings

    @classmethod
    def with_rho_inits(cls, problems, inits, settings, rho_inits) -> "BatchSpec":
        overrides = [dataclasses.replace(settings, rho_init=float(rho)) for rho in rho_inits]
        return cls(problems, inits, settings, overrides)


# ------------------------------------------------------------------------------------
# packing / unpacking
# ------------------------------------------------------------------------------------

def _settings_key(st) -> tuple:
    """Everything of a SolverSettings except rho_init (which is a per-solve device array)."""
    return (st.max_sqp_iterations, st.pcg.tolerance, st.pcg.max_iterations, st.line_search.mu,
            st.line_search.beta, st.line_search.num_shrinks, st.rho_min, st.rho_max, st.rho_factor,
            st.step_tolerance, st.feasibility_tolerance, bool(st.regularize_r), st.pcg_retry_limit)


def _as_settings(st) -> SolverSettings:
    """Accept the reference package's SolverSettings object as well as ours."""
    if isinstance(st, SolverSettings):
        return st
    from .settings import LineSearchSettings, PcgSettings
    return SolverSettings(
        max_sqp_iterations=st.max_sqp_iterations,
        pcg=PcgSettings(st.pcg.tolerance, st.pcg.max_iterations),
        line_search=LineSearchSettings(st.line_search.mu, st.line_search.beta, st.line_search.num_shrinks),
        rho_init=st.rho_init, rho_min=st.rho_min, rho_max=st.rho_max, rho_factor=st.rho_factor,
        step_tolerance=st.step_tolerance, feasibility_tolerance=st.feasibility_tolerance,
        regularize_r=st.regularize_r, pcg_retry_limit=st.pcg_retry_limit)


def _force_rows(problem) -> np.ndarray:
    """Assumed force at knot start times k*h (qpform.py:113-123)."""
    N, fd = problem.horizon, problem.model.force_dim
    force = problem.force
    if force is None:
        return np.zeros((N, fd))
    if force.profile is None:
        value = np.asarray(force.value, dtype=float)
        if value.shape != (fd,):
            raise ValueError(f"force dimension {value.shape} does not match the model's ({fd},)")
        return np.broadcast_to(value, (N, fd))
    return np.stack([np.asarray(force.profile(k * problem.timestep), dtype=float) for k in range(N)])


def pack_problems(problems, inits, rho_inits) -> PackedBatch:
    M = len(problems)
    p0 = problems[0]
    N, n, m, fd = p0.horizon, p0.model.state_dim, p0.model.control_dim, p0.model.force_dim
    out = PackedBatch(
        x_start=np.empty((M, n)), goal=np.empty((M, N + 1, n)), Q=np.empty((M, n, n)),
        R=np.empty((M, m, m)), QN=np.empty((M, n, n)), force=np.empty((M, N, fd)),
        rho_init=np.asarray(rho_inits, dtype=float).copy(), X=np.empty((M, N + 1, n)),
        U=np.empty((M, N, m)))
    for i, (p, (X0, U0)) in enumerate(zip(problems, inits)):
        out.x_start[i] = p.x_start
        out.goal[i] = p.cost.goal          # (n,) broadcasts over the N+1 knots
        out.Q[i], out.R[i], out.QN[i] = p.cost.Q, p.cost.R, p.cost.QN
        out.force[i] = _force_rows(p)
        out.X[i] = np.asarray(X0, dtype=float).reshape(N + 1, n)   # sqp.py:222-223
        out.U[i] = np.asarray(U0, dtype=float).reshape(N, m)
    return out


_CHOLESKY_TEXT = None


def _cholesky_failure_text(k: int) -> str:
    """The text scipy.linalg.cho_factor puts into its LinAlgError for a failing pivot k -- the reference
    embeds it verbatim (qpform.py:264-266), and it depends on the installed scipy ("{k}-th leading minor of the
    array is not positive definite" up to 1.15, "Internal potrf return info = [{k}] for slices [0]." later).
    Probed once from the scipy that is installed; the classic wording is the fallback."""
    global _CHOLESKY_TEXT
    if _CHOLESKY_TEXT is None:
        template = "{k}-th leading minor of the array is not positive definite"
        try:
            import scipy.linalg
            try:
                scipy.linalg.cho_factor(np.diag([1.0, -1.0]), lower=True, check_finite=False)
            except scipy.linalg.LinAlgError as exc:   # failing pivot 2
                msg = str(exc)
                if msg.count("2") == 1:
                    template = msg.replace("2", "{k}")
        except ImportError:
            pass
        _CHOLESKY_TEXT = template
    return _CHOLESKY_TEXT.format(k=k)


_BLOCK_LABEL = {_lib.BLOCK_Q: "Q_{k}", _lib.BLOCK_R: "R_{k}", _lib.BLOCK_S: "S diagonal block {k}"}


def render_error(info_row) -> str | None:
    """Status words -> the reference's "ExcType: message" strings (batch.py:99, sqp.py:242-250,
    qpform.py:264-266, 352)."""
    status = int(info_row[_lib.INFO_STATUS])
    if status == _lib.STATUS_OK:
        return None
    it = int(info_row[_lib.INFO_FAIL_ITER])
    aux = int(info_row[_lib.INFO_FAIL_AUX])
    if status == _lib.STATUS_FACTORIZATION:
        label = _BLOCK_LABEL[int(info_row[_lib.INFO_FAIL_BLOCK])].format(k=int(info_row[_lib.INFO_FAIL_KNOT]))
        return (f"FactorizationError: SQP iteration {it}: {label} is not positive definite: "
                f"{_cholesky_failure_text(aux)}")
    retries = int(info_row[_lib.INFO_RETRIES])
    return (f"PcgBreakdownError: SQP iteration {it}: PCG broke down {retries} times "
            f"(last at inner iteration {aux})")


def unpack_results(res: PackedResult):
    results, errors = [], []
    for i in range(res.X.shape[0]):
        err = render_error(res.info[i])
        errors.append(err)
        if err is not None:
            results.append(None)
            continue
        records = []
        for row in res.trace[i, :int(res.info[i, _lib.INFO_N_RECORDS])]:
            alpha = float(row[_lib.TRACE_ALPHA])
            records.append(IterationRecord(
                iteration=int(row[_lib.TRACE_ITERATION]), merit=float(row[_lib.TRACE_MERIT]),
                constraint_l1=float(row[_lib.TRACE_CONSTRAINT_L1]),
                alpha=None if alpha != alpha else alpha, rho=float(row[_lib.TRACE_RHO]),
                pcg_iterations=int(row[_lib.TRACE_PCG_ITERATIONS]),
                accepted=bool(row[_lib.TRACE_ACCEPTED]),
                step_inf_norm=float(row[_lib.TRACE_STEP_INF_NORM])))
        results.append(SqpResult(res.X[i].copy(), res.U[i].copy(), records,
                                 bool(res.info[i, _lib.INFO_CONVERGED])))
    return results, errors


# ------------------------------------------------------------------------------------
# engines are cached per configuration so repeated calls (MPC loops, benchmarks) reuse the
# device buffers and the instantiated CUDA graph
# ------------------------------------------------------------------------------------

_ENGINES: OrderedDict = OrderedDict()  # key -> BatchEngine, least recently used first
_ENGINE_CACHE_SIZE = 16


def _engine_for(model, M, N, timestep, settings, device, in_use=(), shard: int = 0) -> BatchEngine:
    """Cached engine of one configuration.  Eviction is least-recently-used and never closes an engine
    that the running call still has work on (``in_use``); if every cached engine is busy the cache
    grows for the duration of the call."""
    model_id, params = device_model(model)
    # `shard` keeps two shards of one call apart when they land on the same device with the same shape
    key = (model_id, tuple(params), M, N, float(timestep), _settings_key(settings), device, shard)
    eng = _ENGINES.get(key)
    if eng is not None:
        _ENGINES.move_to_end(key)
        return eng
    if len(_ENGINES) >= _ENGINE_CACHE_SIZE:
        busy = {id(e) for e in in_use}
        for old_key in list(_ENGINES):
            if len(_ENGINES) < _ENGINE_CACHE_SIZE:
                break
            if id(_ENGINES[old_key]) not in busy:
                _ENGINES.pop(old_key).close()
    eng = BatchEngine(model, M, N, timestep, settings, device=device)
    _ENGINES[key] = eng
    return eng


def clear_engine_cache():
    while _ENGINES:
        _, eng = _ENGINES.popitem()
        eng.close()


def _check_problem(p, init) -> None:
    """Everything pack_problems would trip over for ONE problem, raised as the exception the reference's
    sqp_solve would raise for it (sqp.py:222-225, qpform.py:113-123), so that batch_solve can isolate the
    slot (batch.py:92-99) instead of losing the batch."""
    N, n, m = p.horizon, p.model.state_dim, p.model.control_dim
    X0 = np.asarray(init[0], dtype=float)
    U0 = np.asarray(init[1], dtype=float)
    if X0.size != (N + 1) * n:
        raise ValueError(f"cannot reshape array of size {X0.size} into shape ({N + 1},{n})")
    if U0.size != N * m:
        raise ValueError(f"cannot reshape array of size {U0.size} into shape ({N},{m})")
    _force_rows(p)


def shard_bounds(M: int, shards: int) -> list[tuple[int, int]]:
    """Contiguous batch-index ranges [g*M/G, (g+1)*M/G)."""
    return [((g * M) // shards, ((g + 1) * M) // shards) for g in range(shards)]


def batch_solve(spec, workers: int = 1, devices: list[int] | None = None) -> BatchResult:
    """Solve every problem of the batch on the GPU(s); results in input order."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    M = spec.size
    start = time.perf_counter()
    settings = [_as_settings(spec.effective_settings(i)) for i in range(M)]
    # homogeneous device batches: same model + timestep + settings (rho_init is per solve)
    groups: dict = {}
    for i, p in enumerate(spec.problems):
        model_id, params = device_model(p.model)
        key = (model_id, tuple(params), float(p.timestep), _settings_key(settings[i]))
        groups.setdefault(key, []).append(i)

    results: list = [None] * M
    errors: list = [None] * M
    device_ms = 0.0
    pending = []
    for idx in groups.values():
        good = []
        for i in idx:   # a problem that cannot be packed fails alone (batch.py:92-99)
            try:
                _check_problem(spec.problems[i], spec.inits[i])
                good.append(i)
            except Exception as exc:  # noqa: BLE001 - isolate the failing slot
                errors[i] = f"{type(exc).__name__}: {exc}"
        idx = good
        if not idx:
            continue
        problems = [spec.problems[i] for i in idx]
        packed = pack_problems(problems, [spec.inits[i] for i in idx],
                               [settings[i].rho_init for i in idx])
        devs = devices if devices else [None]
        for shard, ((lo, hi), dev) in enumerate(zip(shard_bounds(len(idx), len(devs)), devs)):
            if hi == lo:
                continue
            eng = _engine_for(problems[0].model, hi - lo, problems[0].horizon, problems[0].timestep,
                              settings[idx[0]], dev, in_use=[e for e, _ in pending], shard=shard)
            eng.upload(packed.slice(lo, hi))
            eng.launch()
            pending.append((eng, idx[lo:hi]))
    for eng, members in pending:       # every device is already busy; now drain in order
        eng.finish()
        res = eng.download()
        device_ms = max(device_ms, res.device_ms)
        r, e = unpack_results(res)
        for slot, ri, ei in zip(members, r, e):
            results[slot], errors[slot] = ri, ei
    wall = time.perf_counter() - start
    return BatchResult(results, errors, wall, [1e-3 * device_ms / M] * M, device_time=1e-3 * device_ms)


def sqp_solve(problem: ProblemSpec, X_init, U_init, settings: SolverSettings | None = None) -> SqpResult:
    """Single solve with the reference's signature and error behaviour (sqp.py:204-295):
    solver failures raise FactorizationError / PcgBreakdownError."""
    from .errors import FactorizationError, PcgBreakdownError
    settings = _as_settings(settings) if settings is not None else SolverSettings()
    packed = pack_problems([problem], [(X_init, U_init)], [settings.rho_init])
    eng = _engine_for(problem.model, 1, problem.horizon, problem.timestep, settings, None)
    res = eng.solve(packed)
    err = render_error(res.info[0])
    if err is not None:
        kind, _, msg = err.partition(": ")
        if kind == "FactorizationError":
            raise FactorizationError(msg, int(res.info[0, _lib.INFO_FAIL_KNOT]))
        raise PcgBreakdownError(msg, int(res.info[0, _lib.INFO_FAIL_AUX]))
    return unpack_results(res)[0][0]


def bench_scaling(problem_template: ProblemSpec, M_list, N_list, workers: int = 1, repeats: int = 3,
                  budget_iterations: int = 5, devices: list[int] | None = None) -> list[dict]:
    """Median/p90 wall times over an (M, N) grid of fixed-budget batches: the reference's
    ``bench_scaling`` (batch.py:127-169) with the same protocol -- M copies of the template resized
    to horizon N, zero initialisation, exactly ``budget_iterations`` SQP iterations, one warm-up per
    cell discarded -- and the same row schema (M, N, median_ms, p90_ms, workers), so the reference's
    table / heat-map tooling (cli.py:264-280) consumes the rows unchanged.  Extra columns:
    ``device_ms`` (CUDA-event time of the batch), ``sqp_iteration_rate_hz`` and
    ``solve_iterations_per_s`` derived from it."""
    import dataclasses
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if repeats < 1:
        raise ValueError("repeats must be >= 1")
    if np.asarray(problem_template.cost.goal).ndim != 1:
        raise ValueError("bench_scaling needs a template with a single-state goal")
    settings = SolverSettings(max_sqp_iterations=budget_iterations, step_tolerance=None)
    rows = []
    for N in N_list:
        problem = dataclasses.replace(problem_template, horizon=int(N))
        n, m = problem.model.state_dim, problem.model.control_dim
        init = (np.zeros((N + 1, n)), np.zeros((N, m)))
        for M in M_list:
            spec = BatchSpec([problem] * M, [init] * M, settings)
            batch_solve(spec, workers=workers, devices=devices)          # warm-up discarded
            runs = [batch_solve(spec, workers=workers, devices=devices) for _ in range(repeats)]
            times = sorted(r.wall_time for r in runs)
            median = times[len(times) // 2] if repeats % 2 else 0.5 * (times[len(times) // 2 - 1] + times[len(times) // 2])
            p90 = times[min(len(times) - 1, int(np.ceil(0.9 * len(times))) - 1)]
            dev = float(np.median([r.device_time for r in runs]))
            rows.append({
                "M": M, "N": N, "median_ms": 1e3 * median, "p90_ms": 1e3 * p90, "workers": workers,
                "device_ms": 1e3 * dev,
                "sqp_iteration_rate_hz": budget_iterations / dev if dev > 0 else float("nan"),
                "solve_iterations_per_s": M * budget_iterations / dev if dev > 0 else float("nan"),
            })
    return rows
