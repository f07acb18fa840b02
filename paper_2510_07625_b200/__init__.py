"""gato-b200: B200-native batched SQP trajectory optimisation (GATO, arXiv 2510.07625).

Public surface mirrors the hot-path names of the reference package ``trajbatch``
(/root/reference/pkg/src/trajbatch/__init__.py): problem and settings types, ``batch_solve``,
``sqp_solve`` and the row-wise dynamics / PCG operators, all executed by hand-written CUDA
kernels behind the C ABI in include/gato_b200.h.  There is no CPU execution path.
"""

from .batch import BatchSpec, batch_solve, bench_scaling, clear_engine_cache, shard_bounds, sqp_solve
from .blocktri import BlockTriMatrix, PcgResult, btmv, densify, pcg, step, step_jacobians
from .engine import (BatchEngine, PackedBatch, PackedResult, pcg_batched, select_hypothesis, step_jacobians_many,
                     step_many)
from .errors import (BackendUnavailableError, ConfigError, DimensionError, FactorizationError,
                     PcgBreakdownError)
from .merit import adapt_rho, constraint_l1, line_search, merit, merit_many
from .models import Cartpole, DoubleIntegrator, DynamicsModel, Iiwa14, Pendulum, TwoLinkArm
from .mpc import best_of_batch, rho_grid, sample_hypotheses, shift_warm_start
from .problem import CostSpec, ExternalForce, ProblemSpec
from .results import BatchResult, IterationRecord, SqpResult
from .settings import LineSearchSettings, PcgSettings, SolverSettings
from .stages import KnotLinearization, SchurSystem, StageDump, StepDirection, first_iteration_stages

__version__ = "0.1.0"

__all__ = [
    "BlockTriMatrix", "PcgResult", "btmv", "densify", "pcg", "step", "step_jacobians",
    "best_of_batch", "rho_grid", "sample_hypotheses", "shift_warm_start",
    "adapt_rho", "constraint_l1", "line_search", "merit", "merit_many",
    "KnotLinearization", "SchurSystem", "StageDump", "StepDirection", "first_iteration_stages",
    "BackendUnavailableError", "BatchEngine", "BatchResult", "BatchSpec", "Cartpole", "ConfigError",
    "CostSpec", "DimensionError", "DoubleIntegrator", "DynamicsModel", "ExternalForce",
    "FactorizationError", "Iiwa14", "IterationRecord", "LineSearchSettings", "PackedBatch",
    "PackedResult", "PcgBreakdownError", "PcgSettings", "Pendulum", "ProblemSpec", "SolverSettings",
    "SqpResult", "TwoLinkArm", "batch_solve", "bench_scaling", "clear_engine_cache", "pcg_batched", "shard_bounds",
    "select_hypothesis", "sqp_solve", "step_jacobians_many", "step_many",
]
