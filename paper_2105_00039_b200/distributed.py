"""x-slab decomposition of the mechanical step over several GPUs.

The reference is single-process (no distributed layer).  Here one process per
GPU owns the agents whose global box plane ix lies in its slab
[X_r, X_r+1), X_k = floor(k * dimx / world), of the GLOBAL grid -- the grid
every rank derives, bit for bit, from the all-reduced bounding box
(spatial.py:99-116).  Per step:

  1. all-reduce of the 7-double local bbox (min xyz, max xyz, max diameter);
  2. cg_slab_plan: geometry, owner rank of every owned agent, and whether it
     lies in a neighbour's ghost plane (X_q - 1 or X_q+1 of its owner q+-1);
  3. ONE exchange round: all-to-all of 3 counts per rank pair, then of the
     packed records -- per destination [migrants][lo ghosts][hi ghosts];
     migrants leave / join the owned sets (the whole agent row moves),
     ghosts are this step's candidates only;
  4. cg_slab_step: grid rebuild over owned + ghosts on the slab's sub-grid
     (planes X_r - 1 .. X_r+1), sweep, gate, cap, apply for owned agents;
  5. all-reduce of the counters.

An owned agent's candidate set (its 27 global boxes) and its uid-ordered pair
sum are exactly those of a single-GPU step over the global pool, so
positions/displacements are bit-identical to it.  Exchanges go through
``torch.distributed``: NCCL on device buffers (production), or gloo through
host staging (CPU tests, several ranks sharing one GPU).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class TorchExchange:
    """Collectives for the slab step over an initialised torch.distributed
    process group.  ``device_buffers``: NCCL exchanges device tensors directly;
    otherwise records are staged through host memory (gloo)."""

    def __init__(self, device="cuda", device_buffers=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.device = device
        backend = dist.get_backend()
        self.device_buffers = (backend == "nccl") if device_buffers is None else device_buffers
        self.coll_device = device if self.device_buffers else "cpu"

    # -- buffers the context packs into / reads from (device memory)
    def buffer(self, nbytes):
        return self.torch.empty(max(int(nbytes), 1), dtype=self.torch.uint8, device=self.device)

    @staticmethod
    def ptr(buf):
        return buf.data_ptr()

    def _to_coll(self, t):
        return t if self.device_buffers else t.cpu()

    def _from_coll(self, t):
        return t if self.device_buffers else t.to(self.device)

    def allreduce_bbox(self, bb):
        """min over bb[0:3], max over bb[3:7]."""
        torch = self.torch
        v = torch.tensor(np.concatenate([-bb[:3], bb[3:]]), dtype=torch.float64, device=self.coll_device)
        self.dist.all_reduce(v, op=self.dist.ReduceOp.MAX)
        v = v.cpu().numpy()
        return np.concatenate([-v[:3], v[3:]])

    def allreduce_sum(self, arr):
        t = self.torch.tensor(np.asarray(arr, np.int64), device=self.coll_device)
        self.dist.all_reduce(t)
        return t.cpu().numpy()

    def allreduce_max(self, arr):
        t = self.torch.tensor(np.asarray(arr, np.float64), device=self.coll_device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t.cpu().numpy()

    def alltoall_counts(self, counts):
        torch = self.torch
        send = torch.tensor(np.asarray(counts, np.int64), device=self.coll_device)
        recv = torch.empty_like(send)
        self.dist.all_to_all_single(recv, send)
        return recv.cpu().numpy()

    def alltoall_bytes(self, send, send_bytes, recv_bytes):
        """send: buffer holding the per-destination byte runs in rank order."""
        torch = self.torch
        total_in, total_out = int(np.sum(send_bytes)), int(np.sum(recv_bytes))
        src = self._to_coll(send[:total_in]) if total_in else torch.empty(0, dtype=torch.uint8,
                                                                              device=self.coll_device)
        dst = torch.empty(total_out, dtype=torch.uint8, device=self.coll_device)
        self.dist.all_to_all_single(dst, src, [int(b) for b in recv_bytes], [int(b) for b in send_bytes])
        if self.device_buffers and self.device != "cpu":
            torch.cuda.synchronize()
        return self._from_coll(dst) if total_out else self.buffer(0)


@dataclass
class SlabStats:
    """Global counters of one slab step (StepStats fields of engine.py:134-151)."""
    force_evals: int
    candidates: int
    degenerate_pairs: int
    agents: int
    migrated_in: int
    migrated_out: int
    ghosts: int
    planes: tuple


class SlabRunner:
    """Drives cg_slab_* on one rank.  ``ctx`` is a _native.Context (or any
    object with the same slab methods, e.g. the CPU mock in tests/).

    ``sync_counters=False`` defers the counter all-reduce: ``step`` returns
    this rank's counters and ``collect()`` all-reduces every pending step's
    counters in one collective (one host round trip per step fewer)."""

    def __init__(self, ctx, exchange, sync_counters=True):
        self.ctx, self.ex = ctx, exchange
        self.rank, self.world = exchange.rank, exchange.world
        self.rec = ctx.record_bytes
        self.sync_counters = sync_counters
        self._pending = []
        self._epoch = None           # (list epoch, cached receive counts)

    def step(self, params5, flags=0, interaction_radius=None, box_cap=1 << 24):
        ctx, ex, r, W, R = self.ctx, self.ex, self.rank, self.world, self.rec
        bb = ex.allreduce_bbox(ctx.local_bbox())
        counts, planes = ctx.slab_plan(bb, W, r, interaction_radius, box_cap)
        epoch = ctx.slab_list_epoch() if hasattr(ctx, "slab_list_epoch") else -1
        if epoch >= 0 and self._epoch is not None and self._epoch[0] == epoch:
            recv_counts = self._epoch[1]                  # refresh sizes are fixed within an epoch
        else:
            recv_counts = ex.alltoall_counts(counts)      # 3 per rank pair
            self._epoch = (epoch, recv_counts) if epoch >= 0 else None
        send_bytes = counts.reshape(W, 3).sum(1) * R
        recv_bytes = recv_counts.reshape(W, 3).sum(1) * R
        send = ex.buffer(int(send_bytes.sum()))
        ctx.slab_pack(ex.ptr(send))
        recv = ex.alltoall_bytes(send, send_bytes, recv_bytes)
        ctx.slab_unpack(ex.ptr(recv), recv_counts)
        st = ctx.slab_step(params5, flags)
        local = [st.force_evals, st.candidates, st.degenerate_pairs, st.agent_count]
        rc = recv_counts.reshape(W, 3)
        stats = SlabStats(force_evals=local[0], candidates=local[1], degenerate_pairs=local[2],
                          agents=local[3], migrated_in=int(rc[:, 0].sum()),
                          migrated_out=int(counts.reshape(W, 3)[:, 0].sum()), ghosts=int(rc[:, 1:].sum()),
                          planes=(int(planes[0]), int(planes[1])))
        if not self.sync_counters:
            self._pending.append(stats)
            return stats
        tot = ex.allreduce_sum(local)
        stats.force_evals, stats.candidates, stats.degenerate_pairs, stats.agents = (int(v) for v in tot)
        return stats

    def collect(self):
        """Global counters of the steps whose all-reduce was deferred."""
        if not self._pending:
            return []
        loc = np.array([[s.force_evals, s.candidates, s.degenerate_pairs, s.agents] for s in self._pending],
                       np.int64)
        tot = np.asarray(self.ex.allreduce_sum(loc.ravel())).reshape(loc.shape)
        out = self._pending
        for s, t in zip(out, tot):
            s.force_evals, s.candidates, s.degenerate_pairs, s.agents = (int(v) for v in t)
        self._pending = []
        return out
