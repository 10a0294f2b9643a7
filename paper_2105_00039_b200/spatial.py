"""Uniform grid built on the GPU (API mirror of reference spatial.py:43-127).

``build_grid`` runs the device grid rebuild (K1-K4 of csrc/grid.cuh) on the
pool and returns a ``UniformGrid`` with the reference's fields.  The device
keeps the grid as a box-sorted CSR (counts + offsets); the reference's
linked-cell view (``box_head`` / ``successors``, kernels.py:132-145) is derived
from it on demand and is identical to what reference ``link_chains`` builds.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from ._native import GridOverflowError, StencilTooSmallError  # noqa: F401  (re-export)

DEFAULT_BOX_CAP = 1 << 24
SENTINEL = -1


@dataclass
class UniformGrid:
    box_length: float
    origin: np.ndarray
    dims: np.ndarray
    box_count: np.ndarray
    box_index: np.ndarray

    @property
    def num_boxes(self):
        return int(self.box_count.shape[0])

    @property
    def occupied_box_count(self):
        return int(np.count_nonzero(self.box_count))

    @property
    def max_occupancy(self):
        return int(self.box_count.max()) if self.num_boxes else 0

    def occupancy_histogram(self):
        return np.bincount(self.box_count)

    def box_coords(self):
        dy, dz = int(self.dims[1]), int(self.dims[2])
        return self.box_index // (dy * dz), (self.box_index // dz) % dy, self.box_index % dz

    def stencil_candidate_cap(self):
        return 27 * self.max_occupancy

    @property
    def box_offsets(self):
        """CSR offsets: exclusive prefix sum of box_count (num_boxes + 1 entries)."""
        off = np.zeros(self.num_boxes + 1, np.int64)
        np.cumsum(self.box_count, out=off[1:])
        return off

    def _chains(self):
        n = self.box_index.shape[0]
        order = np.lexsort((np.arange(n), self.box_index))
        succ = np.full(n, SENTINEL, np.int64)
        same = self.box_index[order[1:]] == self.box_index[order[:-1]]
        succ[order[1:][same]] = order[:-1][same]
        head = np.full(self.num_boxes, SENTINEL, np.int64)
        head[self.box_index[order]] = order      # last write per box = highest index
        return head, succ

    @property
    def box_head(self):
        """Agent added to each box last (kernels.py:141-143 insertion order)."""
        return self._chains()[0]

    @property
    def successors(self):
        return self._chains()[1]


def build_grid(pool, interaction_radius=None, parallel=False, box_cap=DEFAULT_BOX_CAP, device=0):
    """Index ``pool`` with box_length = max(interaction_radius, max diameter)."""
    if pool.count == 0:
        raise ValueError("cannot build a grid over an empty pool")
    if interaction_radius is not None and not float(interaction_radius) > 0:
        raise ValueError("interaction_radius must be positive, got %r" % (interaction_radius,))
    ctx = _native.Context(device, pool.dtype)
    try:
        ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter,
                   pool.adherence, pool.uid)
        st = ctx.build_grid(interaction_radius, box_cap)
        dims = np.array(list(st.grid_dims), np.int64)
        bi, bc = ctx.grid_export(int(np.prod(dims)))
        return UniformGrid(box_length=float(st.box_length), origin=np.array(list(st.origin)),
                           dims=dims, box_count=bc, box_index=bi)
    finally:
        ctx.close()
