"""Collision-model parameters (API mirror of reference mechanics.py:47-75).

The CUDA force kernel consumes the same 7-slot parameter vector the reference
kernels do (kernels.py:44-52): kappa, gamma, timestep, max_displacement,
adherence_scale, 0, 1 -- cast to the pool dtype before use.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

DEFAULT_ADHERENCE = 0.4

PAR_KAPPA, PAR_GAMMA, PAR_TIMESTEP, PAR_MAX_DISP, PAR_ADHERENCE_SCALE, PAR_ZERO, PAR_ONE = range(7)
PARAM_COUNT = 7

# Reference cost model (mechanics.py:34-40): 11 flops for the separation +
# overlap test of every candidate, 25 in total for an evaluated pair.
FLOPS_PER_CANDIDATE = 11
FLOPS_PER_FORCE_EVAL = 25


@dataclass(frozen=True)
class ForceParams:
    kappa: float = 2.0
    gamma: float = 1.0
    timestep: float = 0.01
    max_displacement: float = 3.0
    adherence_scale: float = 1.0

    def __post_init__(self):
        if min(self.kappa, self.gamma, self.adherence_scale) < 0:
            raise ValueError("force coefficients must be nonnegative")
        if not self.timestep > 0:
            raise ValueError("timestep must be positive")
        if not self.max_displacement > 0:
            raise ValueError("max_displacement must be positive")

    def as_array(self, dtype):
        vec = [self.kappa, self.gamma, self.timestep, self.max_displacement,
               self.adherence_scale, 0.0, 1.0]
        return np.asarray(vec, dtype=np.float64).astype(dtype)
