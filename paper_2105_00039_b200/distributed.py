"""x-slab decomposition of the mechanical step over several GPUs.

The reference is single-process (no distributed layer).  Here one process per
GPU owns the agents whose global box plane ix lies in its slab
[X_r, X_r+1), X_k = floor(k * dimx / world), of the GLOBAL grid -- the grid
every rank derives, bit for bit, from the all-reduced bounding box
(spatial.py:99-116).  Per step:

  1. all-reduce of the 11-double local bbox (min xyz, max xyz, max diameter,
     largest displacement, list veto, min diameter, max uid);
  2. cg_slab_plan: geometry, owner rank of every owned agent, and whether it
     lies in a neighbour's ghost plane (X_q - 1 or X_q+1 of its owner q+-1);
  3. ONE exchange round: all-to-all of 3 counts per rank pair (skipped inside
     a neighbour-list epoch, whose run sizes are fixed), then the packed
     records -- per destination [migrants][lo ghosts][hi ghosts] -- as
     send/recv pairs with the ranks that have records for each other (x +-1
     in practice), all-to-all only if a run goes further;
     migrants leave / join the owned sets (the whole agent row moves),
     ghosts are this step's candidates only;
  4. cg_slab_step: grid rebuild over owned + ghosts on the slab's sub-grid
     (planes X_r - 1 .. X_r+1), sweep, gate, cap, apply for owned agents;
  5. all-reduce of the counters.

An owned agent's candidate set (its 27 global boxes) and its uid-ordered pair
sum are exactly those of a single-GPU step over the global pool, so
positions/displacements are bit-identical to it.  Exchanges go through
``torch.distributed``: NCCL on device buffers (production), or gloo through
host staging (CPU tests, several ranks sharing one GPU).  Every collective is
issued on the context's own CUDA stream (``stream=ctx.stream``), so pack ->
exchange -> unpack -> step are stream-ordered on the device: no host waits
besides the bbox all-reduce (the host derives the geometry from it) and the
plan's counts on rebuild steps.  World size 1 skips the collectives.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class TorchExchange:
    """Collectives for the slab step over an initialised torch.distributed
    process group.  ``device_buffers``: NCCL exchanges device tensors directly;
    otherwise records are staged through host memory (gloo)."""

    def __init__(self, device="cuda", device_buffers=None, stream=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.device = device
        backend = dist.get_backend()
        self.device_buffers = (backend == "nccl") if device_buffers is None else device_buffers
        self.coll_device = device if self.device_buffers else "cpu"
        # the context's stream (a cudaStream_t handle): collectives and staging
        # copies are issued on it, behind the context's own kernels
        self.stream = None
        if stream is not None:
            self.bind_stream(stream)

    def bind_stream(self, handle):
        """Issue the collectives and staging copies on this cudaStream_t."""
        if str(self.device).startswith("cuda"):
            self.stream = self.torch.cuda.ExternalStream(int(handle), device=self.torch.device(self.device))

    def _on_stream(self):
        import contextlib
        return self.torch.cuda.stream(self.stream) if self.stream is not None else contextlib.nullcontext()

    # -- buffers the context packs into / reads from (device memory)
    def buffer(self, nbytes):
        if int(nbytes) <= 0:   # nothing to send or receive: one persistent placeholder
            if getattr(self, "_empty", None) is None:
                with self._on_stream():
                    self._empty = self.torch.empty(1, dtype=self.torch.uint8, device=self.device)
            return self._empty
        with self._on_stream():
            return self.torch.empty(int(nbytes), dtype=self.torch.uint8, device=self.device)

    @staticmethod
    def ptr(buf):
        return buf.data_ptr()

    def _to_coll(self, t):
        return t if self.device_buffers else t.cpu()

    def _from_coll(self, t):
        return t if self.device_buffers else t.to(self.device)

    def record_event(self):
        """An event on the context stream (behind what is enqueued so far)."""
        ev = self.torch.cuda.Event()
        ev.record(self.stream)
        return ev

    def wait_event(self, ev):
        """The context stream waits for ``ev``."""
        self.stream.wait_event(ev)

    def exchange_async(self, send, send_bytes, recv_bytes, after):
        """alltoall_bytes on a side stream that starts at ``after`` (an event
        behind the pack on the context stream), so the context stream can run
        other work meanwhile; returns (recv, an event when recv is complete)."""
        torch = self.torch
        if getattr(self, "_comm", None) is None:
            self._comm = torch.cuda.Stream(device=torch.device(self.device))
        comm, ctx_stream = self._comm, self.stream
        comm.wait_event(after)
        send.record_stream(comm)
        self.stream = comm
        try:
            recv = self.alltoall_bytes(send, send_bytes, recv_bytes)
        finally:
            self.stream = ctx_stream
        recv.record_stream(ctx_stream)
        done = torch.cuda.Event()
        done.record(comm)
        return recv, done

    def _allreduce(self, values, dtype, op):
        torch = self.torch
        with self._on_stream():
            t = torch.tensor(values, dtype=dtype, device=self.coll_device)
            self.dist.all_reduce(t, op=op)
            return t.cpu().numpy()

    def allreduce_bbox(self, bb):
        """min over bb[0:3], max over bb[3:] (bb[9] is already negated)."""
        bb = np.asarray(bb, np.float64)
        if self.world == 1:
            return bb.copy()
        v = self._allreduce(np.concatenate([-bb[:3], bb[3:]]), self.torch.float64, self.dist.ReduceOp.MAX)
        return np.concatenate([-v[:3], v[3:]])

    def allreduce_sum(self, arr):
        if self.world == 1:
            return np.asarray(arr, np.int64).copy()
        return self._allreduce(np.asarray(arr, np.int64), self.torch.int64, self.dist.ReduceOp.SUM)

    def allreduce_max(self, arr):
        if self.world == 1:
            return np.asarray(arr, np.float64).copy()
        return self._allreduce(np.asarray(arr, np.float64), self.torch.float64, self.dist.ReduceOp.MAX)

    def alltoall_counts(self, counts):
        if self.world == 1:
            return np.asarray(counts, np.int64).copy()
        torch = self.torch
        with self._on_stream():
            send = torch.tensor(np.asarray(counts, np.int64), device=self.coll_device)
            recv = torch.empty_like(send)
            self.dist.all_to_all_single(recv, send)
            return recv.cpu().numpy()

    def alltoall_bytes(self, send, send_bytes, recv_bytes):
        """send: buffer holding the per-destination byte runs in rank order;
        returns the runs received from every source rank, in rank order.
        Only the ranks that exchange records are paired (send/recv, the x +-1
        neighbours of a slab step); the transfer is ordered on the context
        stream, so nothing waits for it on the host."""
        torch, dist = self.torch, self.dist
        send_bytes = np.asarray(send_bytes, np.int64)
        recv_bytes = np.asarray(recv_bytes, np.int64)
        total_in, total_out = int(send_bytes.sum()), int(recv_bytes.sum())
        if total_in == 0 and total_out == 0:
            return self.buffer(0)
        so = np.concatenate([[0], np.cumsum(send_bytes)])
        ro = np.concatenate([[0], np.cumsum(recv_bytes)])
        with self._on_stream():
            src = self._to_coll(send[:total_in]) if total_in else None
            dst = torch.empty(max(total_out, 1), dtype=torch.uint8, device=self.coll_device)
            r = self.rank
            if send_bytes[r]:   # a run to itself (never planned by a slab step, kept for generality)
                dst[ro[r]:ro[r + 1]].copy_(src[so[r]:so[r + 1]])
            ops = []
            for q in range(self.world):
                if q == r:
                    continue
                if send_bytes[q]:
                    ops.append(dist.P2POp(dist.isend, src[so[q]:so[q + 1]], q))
                if recv_bytes[q]:
                    ops.append(dist.P2POp(dist.irecv, dst[ro[q]:ro[q + 1]], q))
            if ops:
                for req in dist.batch_isend_irecv(ops):
                    req.wait()   # NCCL: the current (context) stream waits; gloo: the host does
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
        # pack / unpack / step do not wait for the host: the exchange must run
        # on the context's stream
        if getattr(exchange, "stream", None) is None and hasattr(ctx, "stream") and hasattr(exchange, "bind_stream"):
            exchange.bind_stream(ctx.stream)
        self.rank, self.world = exchange.rank, exchange.world
        self.rec = ctx.record_bytes
        self.sync_counters = sync_counters
        self._pending = []
        self._epoch = None           # per list epoch: sizes, counters and the send buffer (fixed within it)
        self._has_epoch = hasattr(ctx, "slab_list_epoch")
        self._overlap = hasattr(ctx, "slab_step_interior") and getattr(exchange, "stream", None) is not None
        self._deferred = not sync_counters and hasattr(ctx, "fetch_stats")

    def _sizes(self, counts, recv_counts):
        W, R = self.world, self.rec
        c3, r3 = counts.reshape(W, 3), recv_counts.reshape(W, 3)
        send_bytes, recv_bytes = c3.sum(1) * R, r3.sum(1) * R
        return {"recv_counts": recv_counts, "send_bytes": send_bytes, "recv_bytes": recv_bytes,
                "send": self.ex.buffer(int(send_bytes.sum())), "migrated_in": int(r3[:, 0].sum()),
                "migrated_out": int(c3[:, 0].sum()), "ghosts": int(r3[:, 1:].sum()),
                "recv_any": bool(recv_bytes.sum() > 0)}

    def step(self, params5, flags=0, interaction_radius=None, box_cap=1 << 24):
        ctx, ex, r, W = self.ctx, self.ex, self.rank, self.world
        bb = ex.allreduce_bbox(ctx.local_bbox())
        counts, planes = ctx.slab_plan(bb, W, r, interaction_radius, box_cap)
        epoch = ctx.slab_list_epoch() if self._has_epoch else -1
        if epoch >= 0 and self._epoch is not None and self._epoch[0] == epoch:
            z = self._epoch[1]          # refresh sizes (and the send buffer) are fixed within an epoch
        else:
            z = self._sizes(counts, ex.alltoall_counts(counts))   # 3 counts per rank pair
            self._epoch = (epoch, z) if epoch >= 0 else None
        send = z["send"]
        ctx.slab_pack(ex.ptr(send))
        if epoch >= 0 and z["recv_any"] and self._overlap:
            # list step: the interior agents' sweep runs while the ghost refresh
            # is in flight (side stream); the boundary agents follow the unpack
            after = ex.record_event()
            ctx.slab_step_interior(params5, flags)
            recv, done = ex.exchange_async(send, z["send_bytes"], z["recv_bytes"], after)
            ex.wait_event(done)
        else:
            recv = ex.alltoall_bytes(send, z["send_bytes"], z["recv_bytes"])
        ctx.slab_unpack(ex.ptr(recv), z["recv_counts"])
        stats = SlabStats(force_evals=0, candidates=0, degenerate_pairs=0, agents=0,
                          migrated_in=z["migrated_in"], migrated_out=z["migrated_out"], ghosts=z["ghosts"],
                          planes=(int(planes[0]), int(planes[1])))
        if self._deferred:
            # enqueue only: the counters are fetched (and all-reduced) in collect()
            self._pending.append((stats, ctx.slab_step(params5, flags, wait=False)))
            return stats
        st = ctx.slab_step(params5, flags)
        local = [st.force_evals, st.candidates, st.degenerate_pairs, st.agent_count]
        stats.force_evals, stats.candidates, stats.degenerate_pairs, stats.agents = (int(v) for v in local)
        if not self.sync_counters:
            self._pending.append((stats, None))
            return stats
        tot = ex.allreduce_sum(local)
        stats.force_evals, stats.candidates, stats.degenerate_pairs, stats.agents = (int(v) for v in tot)
        return stats

    def collect(self):
        """Global counters of the steps whose all-reduce was deferred."""
        if not self._pending:
            return []
        for s_, sid in self._pending:
            if sid is not None:
                st = self.ctx.fetch_stats(sid)
                s_.force_evals, s_.candidates = int(st.force_evals), int(st.candidates)
                s_.degenerate_pairs, s_.agents = int(st.degenerate_pairs), int(st.agent_count)
        loc = np.array([[s_.force_evals, s_.candidates, s_.degenerate_pairs, s_.agents] for s_, _ in self._pending],
                       np.int64)
        tot = np.asarray(self.ex.allreduce_sum(loc.ravel())).reshape(loc.shape)
        out = [s_ for s_, _ in self._pending]
        for s_, t in zip(out, tot):
            s_.force_evals, s_.candidates, s_.degenerate_pairs, s_.agents = (int(v) for v in t)
        self._pending = []
        return out
