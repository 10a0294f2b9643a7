"""Uniform grid built on the GPU (API mirror of reference spatial.py:43-127).

``build_grid`` runs the device grid rebuild (K1-K4 of csrc/grid.cuh) on the
pool and returns a ``UniformGrid`` with the reference's fields.  The device
keeps the grid as a box-sorted CSR (counts + offsets); the reference's
linked-cell view (``box_head`` / ``successors``, kernels.py:132-145) is derived
from it on demand and is identical to what reference ``link_chains`` builds.
"""

from __future__ import annotations

import hashlib
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


def _query_context(grid, pool, radius, device):
    """Device context holding ``pool`` indexed by ``grid``'s geometry: the grid
    is re-derived on the device from the same pool (spatial.py:99-116 is a pure
    function of the pool and box_length, so the geometry is identical); a pool
    that no longer matches ``grid`` is rejected rather than queried on a stale
    index."""
    radius = float(radius)
    if not radius > 0:
        raise ValueError("radius must be positive, got %r" % radius)
    if radius > grid.box_length:
        raise StencilTooSmallError("radius %g exceeds box_length %g" % (radius, grid.box_length))
    ctx = _native.Context(device, pool.dtype)
    try:
        ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter,
                   pool.adherence, pool.uid)
        st = ctx.build_grid(grid.box_length, DEFAULT_BOX_CAP)
        if (list(st.grid_dims) != [int(d) for d in grid.dims]
                or float(st.box_length) != float(grid.box_length)
                or list(st.origin) != [float(o) for o in grid.origin]):
            raise ValueError("pool does not match the grid it is queried with (rebuild the grid)")
    except BaseException:
        ctx.close()
        raise
    return ctx, radius


def neighbor_counts(grid, pool, radius, device=0):
    """Number of other agents within ``radius`` of each agent (closed ball,
    f64 d^2 <= r^2), in storage order -- reference spatial.py:148-155 /
    kernels.grid_neighbor_counts (kernels.py:427-468) on the device
    (csrc/query.cuh)."""
    if pool.count == 0:
        return np.zeros(0, np.int64)
    ctx, radius = _query_context(grid, pool, radius, device)
    try:
        return ctx.neighbor_counts(radius)
    finally:
        ctx.close()


def neighbor_csr(grid, pool, radius, device=0):
    """(indptr, indices) neighbour table in storage order; each row ascends by
    neighbour uid -- reference spatial.py:158-169 / kernels.grid_neighbor_fill
    (kernels.py:471-520) on the device."""
    if pool.count == 0:
        return np.zeros(1, np.int64), np.zeros(0, np.int64)
    ctx, radius = _query_context(grid, pool, radius, device)
    try:
        return ctx.neighbor_csr(radius)
    finally:
        ctx.close()


def neighbor_table_hash(pool, indptr, indices):
    """Digest of a CSR neighbour table in uid space (reference
    spatial.py:217-232): rows in ascending owner uid, each hashed as
    owner uid, row length, neighbour uids.  One SHA-256 over the concatenated
    little-endian words, which is the same digest as the reference's
    per-row updates."""
    h = hashlib.sha256()
    h.update(b"cellgrid-neighbors-v1")
    uid = np.ascontiguousarray(pool.uid, dtype=np.uint64)
    indptr = np.asarray(indptr, np.int64)
    indices = np.asarray(indices, np.int64)
    n = uid.shape[0]
    order = np.argsort(uid, kind="stable")
    lens = (indptr[1:] - indptr[:-1])[order]
    starts = np.zeros(n + 1, np.int64)
    np.cumsum(lens + 2, out=starts[1:])
    buf = np.empty(int(starts[-1]), np.uint64)
    buf[starts[:-1]] = uid[order]
    buf[starts[:-1] + 1] = lens.astype(np.uint64)
    if indices.shape[0]:
        # entry k of owner row r (r-th smallest uid) goes to starts[r] + 2 + k
        row_of = np.repeat(np.arange(n), lens)
        k = np.arange(row_of.shape[0]) - np.repeat(np.cumsum(lens) - lens, lens)
        src = indptr[:-1][order][row_of] + k
        buf[starts[:-1][row_of] + 2 + k] = uid[indices[src]]
    h.update(buf.astype("<u8", copy=False).tobytes())
    return h.hexdigest()
