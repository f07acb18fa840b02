"""Reference-named block-tridiagonal operators on the GPU (blocktri.py:19-173): ``BlockTriMatrix``,
``btmv``, ``pcg`` / ``PcgResult``, ``densify``, and the scalar ``step`` / ``step_jacobians`` of
dynamics.py:716-772.  Thin host wrappers over gato_btmv_batched, gato_pcg_batched, gato_step_many and
gato_step_jacobians_many with the reference's argument checks and error types; ``pcg`` keeps the
reference's formulation (explicit preconditioner, true-residual stop test)."""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .engine import _dev, _torch, pcg_batched, step_jacobians_many, step_many
from .errors import DimensionError, PcgBreakdownError
from .problem import ExternalForce
from .settings import PcgSettings


@dataclass
class BlockTriMatrix:
    """Symmetric block-tridiagonal matrix (blocktri.py:19-58): diag_blocks (n_blockrows, d, d),
    offdiag_blocks (n_blockrows - 1, d, d), block k at block position (k + 1, k)."""

    diag_blocks: np.ndarray
    offdiag_blocks: np.ndarray

    def __post_init__(self):
        self.diag_blocks = np.ascontiguousarray(self.diag_blocks, dtype=float)
        self.offdiag_blocks = np.ascontiguousarray(self.offdiag_blocks, dtype=float)
        if self.diag_blocks.ndim != 3 or self.diag_blocks.shape[1] != self.diag_blocks.shape[2]:
            raise DimensionError("diag_blocks must have shape (n_blockrows, d, d)")
        nb, bd = self.n_blockrows, self.block_dim
        if self.offdiag_blocks.shape != (max(nb - 1, 0), bd, bd):
            raise DimensionError(f"expected {nb - 1} off-diagonal blocks of shape ({bd}, {bd}), "
                                 f"got {self.offdiag_blocks.shape}")

    @property
    def n_blockrows(self) -> int:
        return self.diag_blocks.shape[0]

    @property
    def block_dim(self) -> int:
        return self.diag_blocks.shape[1]

    @property
    def size(self) -> int:
        return self.n_blockrows * self.block_dim

    @classmethod
    def identity(cls, n_blockrows: int, block_dim: int) -> "BlockTriMatrix":
        eye = np.broadcast_to(np.eye(block_dim), (n_blockrows, block_dim, block_dim))
        return cls(np.array(eye), np.zeros((n_blockrows - 1, block_dim, block_dim)))


@dataclass
class PcgResult:
    solution: np.ndarray
    iterations: int
    converged: bool
    final_residual_norm: float


def densify(mat: BlockTriMatrix) -> np.ndarray:
    """Dense symmetric expansion (blocktri.py:92-102; host bookkeeping, not a hot path)."""
    nb, bd = mat.n_blockrows, mat.block_dim
    dense = np.zeros((nb * bd, nb * bd))
    for i in range(nb):
        dense[i * bd:(i + 1) * bd, i * bd:(i + 1) * bd] = mat.diag_blocks[i]
    for k in range(nb - 1):
        dense[(k + 1) * bd:(k + 2) * bd, k * bd:(k + 1) * bd] = mat.offdiag_blocks[k]
        dense[k * bd:(k + 1) * bd, (k + 1) * bd:(k + 2) * bd] = mat.offdiag_blocks[k].T
    return dense


def btmv(mat: BlockTriMatrix, v) -> np.ndarray:
    """densify(mat) @ v on the GPU, terms in the reference's order (blocktri.py:105-120)."""
    v = np.asarray(v, dtype=float)
    nb, bd = mat.n_blockrows, mat.block_dim
    if v.shape != (nb * bd,):
        raise DimensionError(f"vector length {v.shape} does not match system size {nb * bd}")
    torch = _torch()
    lib = _lib.load()
    d, o, dv = _dev(torch, mat.diag_blocks), _dev(torch, mat.offdiag_blocks), _dev(torch, v)
    y = torch.empty(nb * bd, dtype=torch.float64, device="cuda")
    rc = lib.gato_btmv_batched(1, nb, bd, d.data_ptr(), o.data_ptr(), dv.data_ptr(), y.data_ptr(),
                               C.c_void_p(torch.cuda.current_stream().cuda_stream))
    if rc != 0:
        raise RuntimeError(f"gato_btmv_batched failed ({rc})")
    return y.cpu().numpy()


def pcg(S: BlockTriMatrix, gamma, phi_inv: BlockTriMatrix, settings: PcgSettings) -> PcgResult:
    """blocktri.pcg (blocktri.py:123-173) for one system on the GPU; PcgBreakdownError on non-positive
    curvature."""
    gamma = np.asarray(gamma, dtype=float)
    if gamma.shape != (S.size,):
        raise DimensionError(f"rhs length {gamma.shape} does not match system size {S.size}")
    if phi_inv.n_blockrows != S.n_blockrows or phi_inv.block_dim != S.block_dim:
        raise DimensionError("preconditioner dimensions do not match the system")
    lam, its, conv, status, res = pcg_batched(S.diag_blocks[None], S.offdiag_blocks[None], gamma[None],
                                              phi_inv.diag_blocks[None], phi_inv.offdiag_blocks[None],
                                              settings.tolerance, settings.iteration_cap(S.size))
    if int(status[0]) == _lib.STATUS_PCG_BREAKDOWN:
        raise PcgBreakdownError(f"non-positive curvature at PCG iteration {int(its[0])}", int(its[0]))
    return PcgResult(lam[0], int(its[0]), bool(conv[0]), float(res[0]))


def _force_vector(model, f_ext) -> np.ndarray:
    if f_ext is None:
        return np.zeros(model.force_dim)
    vec = f_ext.at(0.0) if isinstance(f_ext, ExternalForce) or hasattr(f_ext, "at") else np.asarray(f_ext, dtype=float)
    vec = np.asarray(vec, dtype=float)
    if vec.shape != (model.force_dim,):
        raise DimensionError(f"force dimension {vec.shape} does not match {model.name}'s force channel "
                             f"({model.force_dim},)")
    return vec


def _check_point(model, x, u):
    x, u = np.asarray(x, dtype=float), np.asarray(u, dtype=float)
    if x.shape != (model.state_dim,):
        raise DimensionError(f"state shape {x.shape} != ({model.state_dim},)")
    if u.shape != (model.control_dim,):
        raise DimensionError(f"control shape {u.shape} != ({model.control_dim},)")
    if not (np.all(np.isfinite(x)) and np.all(np.isfinite(u))):
        raise ValueError("non-finite state or control")
    return x, u


def step(model, x, u, h: float, f_ext=None) -> np.ndarray:
    """One RK4 step with u and f_ext held constant (dynamics.py:716-728), on the GPU."""
    x, u = _check_point(model, x, u)
    if h <= 0:
        raise ValueError("timestep must be positive")
    return step_many(model, x[None], u[None], h, _force_vector(model, f_ext)[None])[0]


def step_jacobians(model, x, u, h: float, f_ext=None):
    """Exact Jacobians (A, B) of the RK4 map at (x, u) (dynamics.py:731-772), on the GPU."""
    x, u = _check_point(model, x, u)
    A, B = step_jacobians_many(model, x[None], u[None], h, _force_vector(model, f_ext)[None])
    return A[0], B[0]
