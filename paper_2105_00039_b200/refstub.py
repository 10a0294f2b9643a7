"""The Gpu strategy installed into the reference package.

``install(cellgrid)`` is the ctypes stub a maintainer would add to the reference
(``cellgrid/gpu.py`` plus the three ``isinstance`` branches), applied at run time
to an imported, unmodified ``cellgrid``:

* ``cellgrid.engine.step`` (engine.py:279-341): a ``Gpu`` strategy runs the
  step through this package's C ABI (``engine.step``: behaviour phase and
  mechanical step on the device, the pool synchronised back into the
  reference's ``AgentPool`` columns); every other strategy runs the reference's
  own step, untouched.
* ``cellgrid.engine.strategy_label`` (engine.py:90-97) and the copy
  ``cellgrid.bench`` imported by name: ``Gpu`` rows are labelled ``gpu(k)``;
  ``SimulationConfig.__post_init__`` (engine.py:126-131) then accepts ``Gpu``.
* ``cellgrid.engine.Gpu``: the strategy class, next to ``Serial`` /
  ``AgentParallel`` / ``VoxelTiled``.

``engine.run`` and the benchmark harness (``cellgrid.bench.run_benchmark_a/b``,
bench.py:210-262) call ``step`` / ``strategy_label`` through the module, so
after ``install`` they emit ``gpu(k)`` rows beside the reference's CPU rows in
the same CSV (``cellgrid.bench.write_report``).  Nothing here re-implements the
harness; ``report.py`` is the thin entry point over it.
"""

from __future__ import annotations

import dataclasses

from . import engine as _eng
from .mechanics import ForceParams
from .pool import AgentPool, PrecisionMode

Gpu = _eng.Gpu

_COLUMNS = ("position_x", "position_y", "position_z", "diameter", "adherence", "uid",
            "displacement_x", "displacement_y", "displacement_z")


def _pool_view(ref_pool):
    """This package's AgentPool over the reference pool's arrays (no copy)."""
    return AgentPool(**{c: getattr(ref_pool, c) for c in _COLUMNS}, next_uid=int(ref_pool.next_uid))


def _config(ref_config):
    """The reference SimulationConfig restated with this package's types
    (same field names and meaning, engine.py:115-131)."""
    fp = ref_config.force_params
    growth = ref_config.growth
    return _eng.SimulationConfig(
        force_params=ForceParams(**{f.name: getattr(fp, f.name) for f in dataclasses.fields(ForceParams)}),
        strategy=ref_config.strategy,
        precision=PrecisionMode(ref_config.precision.value),
        morton_sort_every=ref_config.morton_sort_every,
        steps=ref_config.steps,
        growth=None if growth is None else _eng.GrowthParams(growth.volume_growth_rate, growth.division_diameter,
                                                            growth.division_enabled),
        freeze_displacement=ref_config.freeze_displacement,
        interaction_radius=ref_config.interaction_radius)


def gpu_step(ref_engine, ref_pool, ref_config, step_index=0):
    """engine.py:279-341 for a Gpu strategy: the device step on the reference
    pool (its columns replaced by the step's result, next_uid advanced), and
    the reference's StepStats."""
    if ref_pool.dtype != ref_config.precision.dtype:
        raise ValueError("pool dtype %s does not match configured precision %s"
                         % (ref_pool.dtype, ref_config.precision.value))
    view = _pool_view(ref_pool)
    st = _eng.step(view, _config(ref_config), step_index)
    for c in _COLUMNS:
        setattr(ref_pool, c, getattr(view, c))
    ref_pool.next_uid = view.next_uid
    names = [f.name for f in dataclasses.fields(ref_engine.StepStats)]
    return ref_engine.StepStats(**{k: getattr(st, k) for k in names})


def install(cellgrid=None):
    """Add the Gpu strategy to an imported reference package; idempotent.
    Returns the package."""
    if cellgrid is None:
        import cellgrid  # noqa: F811 -- the reference package on sys.path
    ref = cellgrid.engine
    if getattr(ref, "_b200_stub", None) is not None:
        return cellgrid
    ref_step, ref_label = ref.step, ref.strategy_label

    def step(pool, config, step_index=0):
        if isinstance(config.strategy, Gpu):
            return gpu_step(ref, pool, config, step_index)
        return ref_step(pool, config, step_index)

    def strategy_label(strategy):
        if isinstance(strategy, Gpu):
            return _eng.strategy_label(strategy)
        return ref_label(strategy)

    step.__doc__ = ref_step.__doc__
    ref.step = step
    ref.strategy_label = strategy_label
    ref.Gpu = Gpu
    bench = getattr(cellgrid, "bench", None)
    if bench is None:
        import importlib
        bench = importlib.import_module(cellgrid.__name__ + ".bench")
    if getattr(bench, "strategy_label", None) is ref_label:
        bench.strategy_label = strategy_label
    ref._b200_stub = (ref_step, ref_label)
    return cellgrid


def uninstall(cellgrid):
    """Restore the reference's own step / strategy_label."""
    ref = cellgrid.engine
    saved = getattr(ref, "_b200_stub", None)
    if saved is None:
        return
    ref.step, ref.strategy_label = saved
    bench = getattr(cellgrid, "bench", None)
    if bench is not None and getattr(bench, "strategy_label", None) is not None:
        bench.strategy_label = saved[1]
    del ref.Gpu
    ref._b200_stub = None
