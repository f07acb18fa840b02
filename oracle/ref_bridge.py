"""ORACLE-SIDE BRIDGE to the unmodified reference package (test infrastructure, never shipped on the
product path).

`__graft_entry__.build()` installs /root/reference/pkg into baseline/_ref (git-ignored, travels to the GPU
box) with pip.  This module imports it from there -- or, in the build container, straight from
/root/reference/pkg/src -- and plugs oracle/iiwa14_np.py into the reference's own DynamicsModel interface
(dynamics.py:94-142), exactly as tests/golden/make_golden.py does, so that the reference *solver*
(`trajbatch.batch_solve`, `trajbatch.sqp_solve`, `trajbatch.mpc`) can be run unmodified on the iiwa14
workloads: as the CPU arm of bench.py (`kind: "reference"`) and as the caller in tests/test_gpu_reference_callers.py.
Only tests/, smoke() and bench.py's CPU legs may import this.
"""

from __future__ import annotations

import importlib
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
CANDIDATES = (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src"))

_tb = None
_where = None


def load():
    """The reference package (module `trajbatch`) or None when it is not installed here."""
    global _tb, _where
    if _tb is not None:
        return _tb
    for base in CANDIDATES:
        if (base / "trajbatch" / "__init__.py").exists():
            if str(base) not in sys.path:
                sys.path.insert(0, str(base))
            try:
                _tb = importlib.import_module("trajbatch")
                _where = str(base)
                return _tb
            except Exception:   # noqa: BLE001 - a broken install reads as "not available"
                if str(base) in sys.path:
                    sys.path.remove(str(base))
    return None


def where() -> str | None:
    load()
    return _where


def iiwa14_model():
    """oracle/iiwa14_np.py behind the reference's DynamicsModel base class (module-level class so that
    problems survive the reference's forked process pool, batch.py:115-118)."""
    tb = load()
    if tb is None:
        raise RuntimeError("the reference package is not installed (baseline/_ref)")
    global RefIiwa14
    if RefIiwa14 is None:
        from oracle.iiwa14_np import Iiwa14 as OracleIiwa14

        class _RefIiwa14(OracleIiwa14, tb.DynamicsModel):
            name = "iiwa14"
            state_dim = 14
            control_dim = 7
            force_dim = 3

        _RefIiwa14.__name__ = _RefIiwa14.__qualname__ = "RefIiwa14"
        _RefIiwa14.__module__ = __name__
        RefIiwa14 = _RefIiwa14
    return RefIiwa14()


RefIiwa14 = None


def problems_from_arrays(batch, h, rows=None):
    """Reference ProblemSpec objects + initial trajectories for the solves `rows` of a PackedBatch
    (constant force per solve, as in the workloads)."""
    tb = load()
    model = iiwa14_model()
    rows = range(batch.size) if rows is None else rows
    problems, inits = [], []
    for b in rows:
        cost = tb.CostSpec(batch.Q[b], batch.R[b], batch.QN[b], np.array(batch.goal[b]))
        problems.append(tb.ProblemSpec(model=model, cost=cost, horizon=batch.X.shape[1] - 1, timestep=h,
                                       x_start=np.array(batch.x_start[b]),
                                       force=tb.ExternalForce.constant(batch.force[b, 0])))
        inits.append((np.array(batch.X[b]), np.array(batch.U[b])))
    return problems, inits


def fixed_budget_settings(iterations, pcg_tolerance=1e-6, pcg_max_iterations=200):
    tb = load()
    return tb.SolverSettings(max_sqp_iterations=iterations,
                             pcg=tb.PcgSettings(tolerance=pcg_tolerance, max_iterations=pcg_max_iterations),
                             step_tolerance=None)
