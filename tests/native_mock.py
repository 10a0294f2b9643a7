"""CPU stand-in for paper_2105_00039_b200._native.Context (TEST INFRASTRUCTURE).

The engine calls upload / behavior / step_download on its context; this mock
answers them with the C oracle (oracle.step: the reference step restated,
pinned to reference fixtures) and oracle.behavior, so host-side plumbing above
the C ABI -- the engine, the reference stub (refstub) -- runs without a GPU.
Only the contract is mocked: same columns, same counters, same storage order.
"""

from __future__ import annotations

from types import SimpleNamespace

import numpy as np

import oracle
from paper_2105_00039_b200.engine import GrowthParams
from paper_2105_00039_b200.mechanics import ForceParams
from paper_2105_00039_b200.pool import AgentPool

_KEYS = (("px", "position_x"), ("py", "position_y"), ("pz", "position_z"), ("diameter", "diameter"),
         ("adherence", "adherence"), ("uid", "uid"), ("dx", "displacement_x"), ("dy", "displacement_y"),
         ("dz", "displacement_z"))


class MockContext:
    def __init__(self, device=0, dtype=np.float64):
        self.dtype = np.dtype(dtype)
        self.n = 0
        self.pool = None
        self.steps = 0

    def set_option(self, *_):
        pass

    def upload(self, px, py, pz, diameter, adherence, uid):
        uid = np.array(uid, np.uint64)
        self.pool = AgentPool(position_x=np.array(px, self.dtype), position_y=np.array(py, self.dtype),
                              position_z=np.array(pz, self.dtype), diameter=np.array(diameter, self.dtype),
                              adherence=np.array(adherence, self.dtype), uid=uid,
                              next_uid=int(uid.max()) + 1 if uid.size else 0)
        self.n = uid.shape[0]

    def behavior(self, step_index, volume_growth_rate, division_diameter, division_enabled, next_uid):
        self.pool.next_uid = int(next_uid)
        k = oracle.behavior.grow_and_divide(
            self.pool, GrowthParams(volume_growth_rate, division_diameter, division_enabled), step_index)
        self.n = self.pool.count
        return int(k)

    def _cols(self, columns):
        return {k: getattr(self.pool, a).copy() for k, a in _KEYS if k in columns}

    def step_download(self, params5, interaction_radius=None, box_cap=1 << 24, flags=0, into=None,
                      columns=tuple(k for k, _ in _KEYS)):
        p = [float(v) for v in params5]
        fp = ForceParams(kappa=p[0], gamma=p[1], timestep=p[2], max_displacement=p[3], adherence_scale=p[4])
        r = oracle.step(self.pool, fp, sort=bool(flags & 1), freeze=bool(flags & 2),
                        interaction_radius=interaction_radius, box_cap=box_cap)
        st = SimpleNamespace(agent_count=self.n, force_evals=r.force_evals, candidates=r.candidates,
                             degenerate_pairs=r.degenerate_pairs, t_sort_ms=0.0, t_grid_ms=0.0, t_force_ms=0.0,
                             t_total_ms=0.0, grid_dims=tuple(int(d) for d in r.dims),
                             grid_occupied_boxes=int(np.count_nonzero(r.box_count)),
                             grid_max_occupancy=int(r.box_count.max(initial=0)))
        self.steps += 1
        return st, self._cols(columns)

    def download(self, into=None):
        return self._cols(tuple(k for k, _ in _KEYS))
