"""Synthetic inputs of BASELINE.json's configurations.

Every pool is built with the reference's own constructors' semantics
(pool.py:145-190, bench.py:137-172), so the CPU oracle and the GPU path see
identical data:

  C1  spawn_grid(32, 8.0, 10.0, 0.4)                          32,768 agents
  C2  spawn_random(1M, cube(L27), 10.0, 0.4, seed 0)          L27 = box_side_for_density(1M, 10, 27)
  C3  spawn_random(2M, cube(Lc), 10.0, 0.4, seed 0), frozen    c in {4, 12, 27, 50, 100}
  C4  256^3 lattice, spacing 8, diameter 10, + U(-1, 1) jitter (spawn_generator(0)), 16,777,216
  C5  per-rank x-slab of a (256 G) x 256 x 256 jittered lattice (jitter seed = rank)
"""

from __future__ import annotations

import numpy as np

from .geometry import Aabb
from .pool import AgentPool, PrecisionMode
from .rng import spawn_generator

C3_DENSITIES = (4.0, 12.0, 27.0, 50.0, 100.0)


def box_side_for_density(agent_count, radius, target_mean_neighbors):
    """Cube side L with (n - 1) * (4/3) pi r^3 / L^3 = target (bench.py:137-148)."""
    if agent_count < 2:
        raise ValueError("agent_count must be >= 2")
    if not (radius > 0 and target_mean_neighbors > 0):
        raise ValueError("radius and target must be positive")
    ball = (4.0 / 3.0) * np.pi * float(radius) ** 3
    return ((agent_count - 1) * ball / float(target_mean_neighbors)) ** (1.0 / 3.0)


def c1(precision=PrecisionMode.FP64):
    return AgentPool.spawn_grid(32, 8.0, 10.0, 0.4, precision=precision)


def random_pool(n, density, precision=PrecisionMode.FP64, seed=0):
    side = box_side_for_density(n, 10.0, density)
    return AgentPool.spawn_random(n, Aabb.cube(side), 10.0, 0.4, seed, precision=precision)


def c2(precision=PrecisionMode.FP64, n=1_000_000):
    return random_pool(n, 27.0, precision)


def c3(density, precision=PrecisionMode.FP64, n=2_000_000):
    return random_pool(n, density, precision)


def jittered_lattice_positions(side, spacing=8.0, jitter=1.0, seed=0, x_planes=None, x0=0):
    """(n, 3) float64 lattice positions + U(-jitter, jitter) per coordinate.

    x_planes/x0 select a slab of lattice planes (C5 shards); the default is the
    full side^3 cube in the reference's x-major uid order (pool.py:162-173)."""
    nx = side if x_planes is None else x_planes
    ticks_x = (np.arange(nx, dtype=np.float64) + x0) * spacing
    ticks = np.arange(side, dtype=np.float64) * spacing
    gx, gy, gz = np.meshgrid(ticks_x, ticks, ticks, indexing="ij")
    pos = np.column_stack([gx.reshape(-1), gy.reshape(-1), gz.reshape(-1)])
    pos += (2.0 * spawn_generator(seed).random(pos.shape) - 1.0) * jitter
    return pos


def c4(precision=PrecisionMode.FP64, side=256):
    return AgentPool.from_arrays(jittered_lattice_positions(side), 10.0, 0.4, precision)


def c5_shard(rank, world, precision=PrecisionMode.FP64, side=256):
    """Rank's slab of the weak-scaling lattice: 256 x-planes per rank; uids are
    globally unique (x-major over the global lattice)."""
    pos = jittered_lattice_positions(side, seed=rank, x_planes=side, x0=rank * side)
    n = pos.shape[0]
    dt = precision.dtype
    uid = np.arange(n, dtype=np.uint64) + np.uint64(rank * n)
    return AgentPool(position_x=pos[:, 0].astype(dt), position_y=pos[:, 1].astype(dt),
                     position_z=pos[:, 2].astype(dt), diameter=np.full(n, 10.0, dt),
                     adherence=np.full(n, 0.4, dt), uid=uid, next_uid=world * n)
