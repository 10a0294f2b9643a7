"""Per-step driver with a ``Gpu`` execution strategy (API mirror of reference
engine.py:56-353).

The operator API is the reference's: ``SimulationConfig`` + ``step(pool,
config, step_index) -> StepStats`` + ``run(pool, config) -> RunReport``, with a
new strategy type ``Gpu`` standing where ``Serial`` / ``AgentParallel`` /
``VoxelTiled`` stand in the reference (engine.py:56-97).  Each step follows the
reference contract (engine.py:12-14): Z-order re-sort if due -> grid rebuild ->
force phase -> apply, executed by libcellgrid_b200.so on one B200.  There is
no CPU path: an unavailable device raises.

``step`` is the drop-in for one call: it uploads the pool, steps on the
device and writes positions, displacements and the new storage order back into
the pool.  ``run`` keeps the population resident in HBM for all steps and
synchronises the host pool once at the end.

The behaviour phase (growth then division, reference engine.py:191-232) runs
on the device too (cg_behavior, csrc/behavior.cuh), bit for bit: numpy's SVML
cube root and its Philox + ziggurat daughter directions are restated in
csrc/behavior_math.h.  A run with growth keeps the pool resident.
"""

from __future__ import annotations

import atexit
import csv
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native
from .mechanics import ForceParams
from .pool import PrecisionMode

RECORD_SCALARS = 5      # reference engine.py:38-39 (bytes_modeled record)
DEFAULT_BOX_CAP = 1 << 24


class TileCapacityError(RuntimeError):
    """Reference engine.py:44-54.  The Gpu strategy stages no fixed-capacity
    tile, so it never raises this; the class exists for API compatibility."""

    def __init__(self, box, needed, capacity):
        super().__init__("stencil of box %d holds %d agents, exceeding tile capacity %d"
                         % (box, needed, capacity))
        self.box, self.needed, self.capacity = box, needed, capacity


SUMMATIONS = {"uid": 0, "stencil": 1}


@dataclass(frozen=True)
class Gpu:
    """B200 strategy: grid rebuild + 27-box sweep as sm_100a kernels.

    summation -- "uid": colliding pairs accumulated in ascending uid order
                 (bit-identical to the reference kernels, kernels.py:206-257);
                 "stencil": accumulated in stencil order (deterministic, within
                 a few ulp of the reference, fewer passes).
    relayout_every -- the device moves agent records into its box-sorted
                 slot order on every k-th sort step (the paper's Z-order
                 locality, GPU v2); the reference's (Morton code, uid) storage
                 order is always what the host sees (kept as a permutation).
    """

    device: int = 0
    summation: str = "uid"
    relayout_every: int = 1

    def __post_init__(self):
        if self.device < 0:
            raise ValueError("device must be >= 0")
        if self.summation not in SUMMATIONS:
            raise ValueError("summation must be one of %s" % sorted(SUMMATIONS))
        if self.relayout_every < 1:
            raise ValueError("relayout_every must be >= 1")


@dataclass(frozen=True)
class Serial:
    """Reference engine.py:57-59.  The reference states that Serial,
    AgentParallel and VoxelTiled produce bit-identical pools (engine.py:5);
    here every one of them is executed by the B200 path in uid summation,
    which is bit-identical to them (tests/test_gpu_parity.py), so a reference
    configuration runs unchanged.  The label stays the reference's."""


@dataclass(frozen=True)
class AgentParallel:
    """Reference engine.py:62-70 (same validation); executed on the B200 (see Serial)."""

    thread_count: int

    def __post_init__(self):
        if self.thread_count < 1:
            raise ValueError("thread_count must be >= 1")


@dataclass(frozen=True)
class VoxelTiled:
    """Reference engine.py:73-87 (same validation); executed on the B200 (see
    Serial).  The B200 path stages no fixed-capacity tile, so an explicit
    ``tile_stencil_capacity`` -- whose overflow the reference reports as
    TileCapacityError -- is not supported and is rejected when the
    configuration is built."""

    thread_count: int
    tile_stencil_capacity: Optional[int] = None

    def __post_init__(self):
        if self.thread_count < 1:
            raise ValueError("thread_count must be >= 1")
        if self.tile_stencil_capacity is not None and self.tile_stencil_capacity < 1:
            raise ValueError("tile_stencil_capacity must be >= 1")


def strategy_label(strategy):
    """Reference engine.py:90-97, plus ``gpu(<device>)`` for Gpu."""
    if isinstance(strategy, Gpu):
        return "gpu(%d)" % strategy.device
    if isinstance(strategy, Serial):
        return "serial"
    if isinstance(strategy, AgentParallel):
        return "parallel(%d)" % strategy.thread_count
    if isinstance(strategy, VoxelTiled):
        return "voxel(%d)" % strategy.thread_count
    raise TypeError("unknown strategy %r" % (strategy,))


def as_gpu(strategy):
    """The Gpu strategy that executes ``strategy``: a reference CPU strategy
    maps to device 0 in uid summation (bit-identical to it)."""
    if isinstance(strategy, Gpu):
        return strategy
    if isinstance(strategy, VoxelTiled) and strategy.tile_stencil_capacity is not None:
        raise NotImplementedError("VoxelTiled with an explicit tile_stencil_capacity: the B200 path stages no "
                                  "fixed-capacity tile; use tile_stencil_capacity=None or Gpu()")
    strategy_label(strategy)
    return Gpu(device=0, summation="uid")


@dataclass(frozen=True)
class GrowthParams:
    """Reference engine.py:100-112: volume growth per step and the diameter
    gate for division (the behaviour phase, ``grow_and_divide``)."""

    volume_growth_rate: float
    division_diameter: float
    division_enabled: bool = True

    def __post_init__(self):
        if not self.volume_growth_rate > 0:
            raise ValueError("volume_growth_rate must be positive")
        if not self.division_diameter > 0:
            raise ValueError("division_diameter must be positive")


@dataclass(frozen=True)
class SimulationConfig:
    force_params: ForceParams = field(default_factory=ForceParams)
    strategy: object = field(default_factory=Gpu)
    precision: PrecisionMode = PrecisionMode.FP64
    morton_sort_every: int = 1
    steps: int = 10
    growth: Optional[GrowthParams] = None
    freeze_displacement: bool = False
    interaction_radius: Optional[float] = None

    def __post_init__(self):
        if self.steps < 0:
            raise ValueError("steps must be >= 0")
        if self.morton_sort_every < 0:
            raise ValueError("morton_sort_every must be >= 0 (0 = never)")
        as_gpu(self.strategy)


@dataclass
class StepStats:
    step_index: int
    agent_count: int
    divisions: int
    force_evals: int
    candidates: int
    degenerate_pairs: int
    bytes_modeled: int
    t_behavior: float
    t_sort: float
    t_grid: float
    t_force: float
    t_apply: float
    t_total: float
    grid_dims: tuple
    grid_occupied_boxes: int
    grid_max_occupancy: int


@dataclass
class RunReport:
    strategy: str
    precision: str
    initial_count: int
    final_count: int
    steps: list
    final_state_hash: str
    wall_time: float

    @property
    def force_evals(self):
        return sum(s.force_evals for s in self.steps)

    @property
    def candidates(self):
        return sum(s.candidates for s in self.steps)

    @property
    def bytes_modeled(self):
        return sum(s.bytes_modeled for s in self.steps)

    @property
    def divisions(self):
        return sum(s.divisions for s in self.steps)

    def write_step_log(self, path):
        cols = ("step_index", "agent_count", "divisions", "force_evals", "candidates",
                "degenerate_pairs", "bytes_modeled", "t_behavior", "t_sort", "t_grid",
                "t_force", "t_apply", "t_total")
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(cols)
            for s in self.steps:
                w.writerow([getattr(s, c) for c in cols])


# -------------------------------------------------------------------- contexts
_contexts = {}


def _context(strategy, dtype):
    strategy = as_gpu(strategy)
    key = (strategy.device, np.dtype(dtype).str, strategy.summation, strategy.relayout_every)
    ctx = _contexts.get(key)
    if ctx is None:
        ctx = _native.Context(strategy.device, dtype)
        ctx.set_option(_native.CG_OPT_SUMMATION, SUMMATIONS[strategy.summation])
        ctx.set_option(_native.CG_OPT_RELAYOUT_EVERY, strategy.relayout_every)
        _contexts[key] = ctx
    return ctx


@atexit.register
def _release_contexts():
    for ctx in _contexts.values():
        ctx.close()
    _contexts.clear()


def grow_and_divide(pool, growth: GrowthParams, step_index=0, strategy=None):
    """Behaviour phase (reference engine.py:191-232) on the device: every
    agent's volume pi/6 d^3 grows by ``volume_growth_rate`` (pool dtype);
    agents whose diameter reached ``division_diameter`` split, mothers in
    ascending uid: the mother keeps half the volume, the daughter (the other
    half, same adherence) is appended at mother_radius / 4 along
    ``unit_vector(uid, step_index)``.  The pool is updated in place (the
    daughters appended, next_uid advanced); returns the number of divisions."""
    if pool.count == 0:
        return 0
    ctx = _context(strategy or Gpu(), pool.dtype)
    _upload(ctx, pool)
    k = ctx.behavior(step_index, growth.volume_growth_rate, growth.division_diameter,
                     growth.division_enabled, pool.next_uid)
    _assign(pool, ctx.download())
    pool.next_uid += k
    return k


def params_vector(fp: ForceParams):
    return np.array([fp.kappa, fp.gamma, fp.timestep, fp.max_displacement,
                     fp.adherence_scale], np.float64)


def step_flags(config, step_index, record=False):
    flags = 0
    every = config.morton_sort_every
    if every > 0 and step_index % every == 0:
        flags |= _native.CG_STEP_SORT
    if config.freeze_displacement:
        flags |= _native.CG_STEP_FREEZE
    if record:
        flags |= _native.CG_STEP_RECORD
    return flags


def _check(pool, config):
    if pool.dtype != config.precision.dtype:
        raise ValueError("pool dtype %s does not match configured precision %s"
                         % (pool.dtype, config.precision.value))


def _upload(ctx, pool):
    ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter,
               pool.adherence, pool.uid)


_POOL_KEYS = ("px", "py", "pz", "diameter", "adherence", "uid", "dx", "dy", "dz")
_POOL_COLS = (("px", "position_x"), ("py", "position_y"), ("pz", "position_z"),
              ("diameter", "diameter"), ("adherence", "adherence"), ("uid", "uid"),
              ("dx", "displacement_x"), ("dy", "displacement_y"), ("dz", "displacement_z"))


def _reusable(ctx, pool):
    """The host pool's own arrays where a download can write in place
    (contiguous, writeable, right dtype/length) -- so pinned host columns
    stay pinned."""
    into = {}
    for key, attr in _POOL_COLS:
        a = getattr(pool, attr, None)
        want = np.uint64 if key == "uid" else ctx.dtype
        if (isinstance(a, np.ndarray) and a.dtype == want and a.shape == (ctx.n,)
                and a.flags.c_contiguous and a.flags.writeable):
            into[key] = a
    return into


def _assign(pool, cols):
    pool.position_x, pool.position_y, pool.position_z = cols["px"], cols["py"], cols["pz"]
    pool.diameter, pool.adherence, pool.uid = cols["diameter"], cols["adherence"], cols["uid"]
    pool.displacement_x, pool.displacement_y, pool.displacement_z = cols["dx"], cols["dy"], cols["dz"]


def _download(ctx, pool):
    """Write the device pool back into the host pool (in place where possible)."""
    _assign(pool, ctx.download(into=_reusable(ctx, pool)))


def _empty_stats(step_index):
    return StepStats(step_index=step_index, agent_count=0, divisions=0, force_evals=0,
                     candidates=0, degenerate_pairs=0, bytes_modeled=0, t_behavior=0.0,
                     t_sort=0.0, t_grid=0.0, t_force=0.0, t_apply=0.0, t_total=0.0,
                     grid_dims=(0, 0, 0), grid_occupied_boxes=0, grid_max_occupancy=0)


def _to_stats(st, step_index, itemsize):
    n = int(st.agent_count)
    return StepStats(step_index=step_index, agent_count=n, divisions=0,
                     force_evals=int(st.force_evals), candidates=int(st.candidates),
                     degenerate_pairs=int(st.degenerate_pairs),
                     bytes_modeled=(int(st.candidates) + n) * RECORD_SCALARS * itemsize,
                     t_behavior=0.0, t_sort=st.t_sort_ms * 1e-3, t_grid=st.t_grid_ms * 1e-3,
                     t_force=st.t_force_ms * 1e-3, t_apply=0.0, t_total=st.t_total_ms * 1e-3,
                     grid_dims=tuple(int(d) for d in st.grid_dims),
                     grid_occupied_boxes=int(st.grid_occupied_boxes),
                     grid_max_occupancy=int(st.grid_max_occupancy))


def step(pool, config: SimulationConfig, step_index=0):
    """Advance ``pool`` by one step: the behaviour phase (if configured), then
    the mechanical step, both on the GPU; returns StepStats."""
    _check(pool, config)
    if pool.count == 0:
        return _empty_stats(step_index)
    ctx = _context(config.strategy, pool.dtype)
    _upload(ctx, pool)
    divisions, t_behavior = 0, 0.0
    if config.growth is not None:
        t0 = time.perf_counter()
        g = config.growth
        divisions = ctx.behavior(step_index, g.volume_growth_rate, g.division_diameter, g.division_enabled,
                                 pool.next_uid)
        pool.next_uid += divisions
        t_behavior = time.perf_counter() - t0
    # the step and the download of its result, transfers overlapped with the sweep;
    # a step without the Z-order sort (and without growth) keeps the storage
    # order and the diameters, so diameter, adherence and uid on the host are
    # already the device's
    flags = step_flags(config, step_index)
    sorted_step = bool(flags & _native.CG_STEP_SORT)
    whole = sorted_step or config.growth is not None
    wanted = _POOL_KEYS if whole else ("px", "py", "pz", "dx", "dy", "dz")
    st, cols = ctx.step_download(params_vector(config.force_params), config.interaction_radius,
                                 DEFAULT_BOX_CAP, flags, into=_reusable(ctx, pool), columns=wanted)
    if not whole:
        cols.update(diameter=pool.diameter, adherence=pool.adherence, uid=pool.uid)
    _assign(pool, cols)
    out = _to_stats(st, step_index, pool.precision.itemsize)
    out.divisions = divisions
    out.t_behavior = t_behavior
    out.t_total += t_behavior
    return out


def run(pool, config: SimulationConfig):
    """``config.steps`` steps with the pool resident on the device (behaviour
    phase included); the host pool is synchronised once, at the end."""
    _check(pool, config)
    t0 = time.perf_counter()
    initial = pool.count
    stats = []
    if pool.count == 0:
        stats = [_empty_stats(k) for k in range(config.steps)]
    elif config.steps:
        ctx = _context(config.strategy, pool.dtype)
        _upload(ctx, pool)
        pv = params_vector(config.force_params)
        g = config.growth
        ids, raw, divs, tbeh = [], [], [], []
        for k in range(config.steps):
            d, tb = 0, 0.0
            if g is not None:
                tb0 = time.perf_counter()
                d = ctx.behavior(k, g.volume_growth_rate, g.division_diameter, g.division_enabled, pool.next_uid)
                pool.next_uid += d
                tb = time.perf_counter() - tb0
            divs.append(d)
            tbeh.append(tb)
            ids.append(ctx.step(pv, config.interaction_radius, DEFAULT_BOX_CAP,
                                step_flags(config, k), wait=False))
            if len(ids) > 16:                     # the device stats ring holds 64 steps
                raw.append(ctx.fetch_stats(ids.pop(0)))
        raw.extend(ctx.fetch_stats(i) for i in ids)
        stats = [_to_stats(st, k, pool.precision.itemsize) for k, st in enumerate(raw)]
        for s_, d, tb in zip(stats, divs, tbeh):
            s_.divisions = d
            s_.t_behavior = tb
            s_.t_total += tb
        _download(ctx, pool)
    return RunReport(strategy=strategy_label(config.strategy), precision=config.precision.value,
                     initial_count=initial, final_count=pool.count, steps=stats,
                     final_state_hash=pool.state_hash(), wall_time=time.perf_counter() - t0)
