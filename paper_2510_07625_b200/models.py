"""Model descriptors: which device dynamics a problem uses, and its parameters.

Host-side mirror of the reference's ``DynamicsModel`` family
(/root/reference/pkg/src/trajbatch/dynamics.py:94-703).  These objects carry dimensions and
parameters only -- the dynamics themselves run on the GPU (csrc/models.cuh,
csrc/model_iiwa14.cuh); there is deliberately no host evaluation path here.
Objects of the reference package itself are accepted wherever a descriptor is expected
(duck-typed on ``name`` and the public parameter attributes).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

MODEL_DOUBLE_INTEGRATOR = 0
MODEL_PENDULUM = 1
MODEL_CARTPOLE = 2
MODEL_TWO_LINK_ARM = 3
MODEL_IIWA14 = 4


@dataclass(frozen=True)
class DynamicsModel:
    """Dimension contract of dynamics.py:94-107."""

    @property
    def state_dim(self) -> int:
        raise NotImplementedError

    @property
    def control_dim(self) -> int:
        raise NotImplementedError

    @property
    def force_dim(self) -> int:
        raise NotImplementedError

    @property
    def position_dim(self) -> int:
        return self.state_dim // 2

    def zero_force(self):
        from .problem import ExternalForce
        return ExternalForce.zero(self.force_dim)


@dataclass(frozen=True)
class DoubleIntegrator(DynamicsModel):
    """dynamics.py:145-163.  Device instantiations exist for dims = 1..7."""

    dims: int = 1
    mass: float = 1.0
    name: str = "double_integrator"

    @property
    def state_dim(self):
        return 2 * self.dims

    @property
    def control_dim(self):
        return self.dims

    @property
    def force_dim(self):
        return self.dims


@dataclass(frozen=True)
class Pendulum(DynamicsModel):
    """dynamics.py:190-214."""

    mass: float = 1.0
    length: float = 1.0
    gravity: float = 9.81
    damping: float = 0.1
    name: str = "pendulum"
    state_dim = 2
    control_dim = 1
    force_dim = 1


@dataclass(frozen=True)
class Cartpole(DynamicsModel):
    """dynamics.py:255-279."""

    cart_mass: float = 1.0
    pole_mass: float = 0.2
    pole_length: float = 0.5
    gravity: float = 9.81
    name: str = "cartpole"
    state_dim = 4
    control_dim = 1
    force_dim = 2


@dataclass(frozen=True)
class TwoLinkArm(DynamicsModel):
    """dynamics.py:387-414."""

    m1: float = 1.0
    m2: float = 1.0
    l1: float = 0.5
    l2: float = 0.5
    gravity: float = 0.0
    joint_damping: float = 0.05
    name: str = "two_link_arm"
    state_dim = 4
    control_dim = 2
    force_dim = 2


@dataclass(frozen=True)
class Iiwa14(DynamicsModel):
    """KUKA LBR iiwa 14 R820, 7 revolute joints, world-frame flange force channel
    (parameter table frozen in csrc/model_iiwa14.cuh)."""

    name: str = "iiwa14"
    state_dim = 14
    control_dim = 7
    force_dim = 3


def device_model(model) -> tuple[int, np.ndarray]:
    """(model id, 8-double parameter block) of gato_config for a descriptor or a
    reference-package model object."""
    name = getattr(model, "name", None)
    params = np.zeros(8)
    if name == "double_integrator":
        if not 1 <= model.dims <= 7:
            raise ValueError("double_integrator is instantiated on the device for dims 1..7")
        params[:2] = [model.dims, model.mass]
        return MODEL_DOUBLE_INTEGRATOR, params
    if name == "pendulum":
        params[:4] = [model.mass, model.length, model.gravity, model.damping]
        return MODEL_PENDULUM, params
    if name == "cartpole":
        params[:4] = [model.cart_mass, model.pole_mass, model.pole_length, model.gravity]
        return MODEL_CARTPOLE, params
    if name == "two_link_arm":
        params[:6] = [model.m1, model.m2, model.l1, model.l2, model.gravity, model.joint_damping]
        return MODEL_TWO_LINK_ARM, params
    if name == "iiwa14":
        return MODEL_IIWA14, params
    raise ValueError(f"model {name!r} has no device implementation")
