"""B200-native mechanical-interaction step for spherical agents (arXiv 2105.00039).

Drop-in for the reference ``cellgrid`` operator API on its hot path:
``AgentPool`` + ``SimulationConfig(strategy=Gpu())`` + ``step`` / ``run``,
executed by hand-written sm_100a kernels behind a C ABI
(include/cellgrid_b200.h, libcellgrid_b200.so).
"""

from .engine import (AgentParallel, GrowthParams, Gpu, RunReport, Serial, SimulationConfig, StepStats,
                     TileCapacityError, VoxelTiled, as_gpu, grow_and_divide, run, step, strategy_label)
from .geometry import FP32, FP64, Aabb
from .mechanics import DEFAULT_ADHERENCE, FLOPS_PER_FORCE_EVAL, ForceParams
from .pool import AgentPool, PoolCapacityError, PrecisionMode
from .spatial import (DEFAULT_BOX_CAP, GridOverflowError, StencilTooSmallError, UniformGrid,
                      build_grid)
from .workloads import box_side_for_density

__version__ = "0.1.0"

__all__ = ["AgentParallel", "Serial", "VoxelTiled", "as_gpu", "Aabb", "AgentPool", "DEFAULT_ADHERENCE", "DEFAULT_BOX_CAP", "FLOPS_PER_FORCE_EVAL",
           "FP32", "FP64", "ForceParams", "Gpu", "GridOverflowError", "GrowthParams",
           "PoolCapacityError", "PrecisionMode", "RunReport", "SimulationConfig",
           "StencilTooSmallError", "StepStats", "TileCapacityError", "UniformGrid",
           "box_side_for_density", "build_grid", "grow_and_divide", "run", "step", "strategy_label"]
