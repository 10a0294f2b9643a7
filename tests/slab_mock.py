"""CPU stand-in for the slab half of the C ABI (TEST INFRASTRUCTURE).

Implements the cg_slab_* contract of include/cellgrid_b200.h with numpy and
the C oracle, so tests can drive paper_2105_00039_b200.distributed.SlabRunner
over gloo without a GPU: same record layout (8 pool-dtype scalars + uid),
same ownership rule (global box plane in [X_r, X_r+1)), same ghost planes
(X_r - 1, X_r+1) and the same one-round exchange layout, ghosts as
candidates only.
"""

from __future__ import annotations

import ctypes
from types import SimpleNamespace

import numpy as np

import oracle

COLS = ("position_x", "position_y", "position_z", "diameter", "adherence",
        "displacement_x", "displacement_y", "displacement_z")


def _view(ptr, nbytes):
    return np.ctypeslib.as_array((ctypes.c_uint8 * max(nbytes, 1)).from_address(ptr))[:nbytes]


class MockSlabContext:
    def __init__(self, pool, params7):
        self.dt = pool.dtype
        self.rec_dtype = np.dtype([("v", self.dt, 8), ("uid", np.uint64)])
        self.cols = {c: getattr(pool, c).copy() for c in COLS}
        self.uid = pool.uid.copy()
        self.params7 = params7
        self.ghosts = None

    @property
    def record_bytes(self):
        return self.rec_dtype.itemsize

    @property
    def n(self):
        return self.uid.shape[0]

    def local_bbox(self):
        if self.n == 0:
            return np.array([np.inf] * 3 + [-np.inf] * 3 + [float(self.cols["diameter"].max(initial=0.0)), 0, 0,
                                                            -np.inf, 0.0])
        p = [self.cols[c].astype(np.float64) for c in COLS[:3]]
        d = self.cols["diameter"].astype(np.float64)
        return np.array([q.min() for q in p] + [q.max() for q in p] +
                        [float(d.max()), 0, 0, -float(d.min()), float(self.uid.max())])

    def _ix(self, x):
        return np.clip(np.floor((x.astype(np.float64) - self.origin[0]) / self.L).astype(np.int64), 0,
                       self.dims[0] - 1)

    def slab_plan(self, bb, world, rank, interaction_radius=None, box_cap=1 << 24):
        L = float(bb[6]) if interaction_radius is None else max(float(interaction_radius), float(bb[6]))
        self.L = L
        self.origin = np.asarray(bb[:3], np.float64) - L
        self.dims = (np.floor((np.asarray(bb[3:6]) - np.asarray(bb[:3])) / L).astype(np.int64) + 3)
        B = [(k * int(self.dims[0])) // world for k in range(world + 1)]
        self.bounds = B
        self.rank, self.world = rank, world
        ix = self._ix(self.cols["position_x"])
        q = np.searchsorted(B, ix, side="right") - 1
        Bn = np.asarray(B)
        self.q = q
        self.up = (q + 1 < world) & (ix == Bn[np.minimum(q + 1, world)] - 1)
        self.down = (q > 0) & (ix == Bn[q])
        counts = np.zeros(3 * world, np.int64)
        for d in range(world):
            counts[3 * d] = np.count_nonzero(q == d) if d != rank else 0
            counts[3 * d + 1] = np.count_nonzero(self.up & (q + 1 == d))
            counts[3 * d + 2] = np.count_nonzero(self.down & (q - 1 == d))
        return counts, np.array(B[rank:rank + 2], np.int64)

    def _records(self, idx):
        rec = np.empty(idx.shape[0], self.rec_dtype)
        rec["v"] = np.stack([self.cols[c][idx] for c in COLS], 1)
        rec["uid"] = self.uid[idx]
        return rec

    def _write(self, ptr, rec):
        _view(ptr, rec.nbytes)[:] = rec.view(np.uint8)

    def _read(self, ptr, count):
        return _view(ptr, count * self.record_bytes).view(self.rec_dtype).copy()

    def slab_pack(self, ptr):
        q, r = self.q, self.rank
        runs = []
        for d in range(self.world):
            runs.append(np.nonzero((q == d) & (d != r))[0])
            runs.append(np.nonzero(self.up & (q + 1 == d))[0])
            runs.append(np.nonzero(self.down & (q - 1 == d))[0])
        self._write(ptr, self._records(np.concatenate(runs)))
        keep = q == r
        for c in COLS:
            self.cols[c] = self.cols[c][keep]
        self.uid = self.uid[keep]

    def slab_unpack(self, ptr, recv_counts):
        rc = np.asarray(recv_counts, np.int64).reshape(self.world, 3)
        rec = self._read(ptr, int(rc.sum()))
        starts = np.concatenate([[0], np.cumsum(rc.ravel())])
        seg = [rec[starts[k]:starts[k + 1]] for k in range(3 * self.world)]
        mig = np.concatenate(seg[0::3])
        for k, c in enumerate(COLS):
            self.cols[c] = np.concatenate([self.cols[c], mig["v"][:, k]])
        self.uid = np.concatenate([self.uid, mig["uid"]])
        self.ghosts = np.concatenate(seg[1::3] + seg[2::3])

    def slab_step(self, params5, flags=0):
        from paper_2105_00039_b200.pool import AgentPool
        g = self.ghosts
        n = self.n
        cols = {c: np.concatenate([self.cols[c], g["v"][:, k]]) for k, c in enumerate(COLS)}
        pool = AgentPool(position_x=cols["position_x"], position_y=cols["position_y"],
                         position_z=cols["position_z"], diameter=cols["diameter"],
                         adherence=cols["adherence"], uid=np.concatenate([self.uid, g["uid"]]))
        nb = int(np.prod(self.dims))
        bidx = oracle.box_ids(pool, self.L, self.origin, self.dims)
        count, start, members = oracle.csr(bidx, nb)
        (dx, dy, dz), m, nk, _ = oracle.force_phase(pool, bidx, self.dims, start, members, self.params7)
        self.cols["displacement_x"], self.cols["displacement_y"], self.cols["displacement_z"] = dx[:n], dy[:n], dz[:n]
        if not flags & 2:
            for c, d in zip(COLS[:3], (dx, dy, dz)):
                self.cols[c] = self.cols[c] + d[:n]
        self.ghosts = None
        return SimpleNamespace(force_evals=int(nk[:n].sum()), candidates=int(m[:n].sum()),
                               degenerate_pairs=0, agent_count=n)
