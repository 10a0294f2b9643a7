"""Per-phase host timing of one slab step (world size from torchrun, or 1 with
NCCL): where the slab driver spends its time beyond the single-context step.

usage: python tools/slab_probe.py [steps]   (or under torchrun)
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2105_00039_b200 import _native, workloads  # noqa: E402
from paper_2105_00039_b200.distributed import TorchExchange  # noqa: E402
from paper_2105_00039_b200.pool import PrecisionMode  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29541"), ("RANK", "0"), ("WORLD_SIZE", "1")):
        os.environ.setdefault(k, v)
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    r, W = dist.get_rank(), dist.get_world_size()
    pool = workloads.c4(PrecisionMode.FP64) if W == 1 else workloads.c5_shard(r, W, PrecisionMode.FP64)
    ctx = _native.Context(local, pool.dtype)
    ctx.set_option(_native.CG_OPT_SUMMATION, 1)
    ctx.reserve(int(pool.count * 1.05) + 4 * 256 * 256 * 2 + 4096)
    ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
    ex = TorchExchange(device="cuda", stream=ctx.stream)
    R = ctx.record_bytes
    params = np.array([2.0, 1.0, 0.01, 3.0, 1.0])
    stream = torch.cuda.ExternalStream(ctx.stream)
    names = ["bbox", "allreduce", "plan", "a2a_counts", "pack", "a2a_bytes", "unpack", "slab_step", "counters"]
    acc = {k: [] for k in names}
    with torch.cuda.stream(stream):
        for it in range(steps + 2):
            t = {}
            last = [time.perf_counter()]

            def mark(name):
                torch.cuda.synchronize()
                now = time.perf_counter()
                t[name] = (now - last[0]) * 1e3
                last[0] = now
            bb = ctx.local_bbox(); mark("bbox")
            bb = ex.allreduce_bbox(bb); mark("allreduce")
            counts, planes = ctx.slab_plan(bb, W, r); mark("plan")
            rc = ex.alltoall_counts(counts); mark("a2a_counts")
            sb = counts.reshape(W, 3).sum(1) * R
            rb = rc.reshape(W, 3).sum(1) * R
            send = ex.buffer(int(sb.sum()))
            ctx.slab_pack(ex.ptr(send)); mark("pack")
            recv = ex.alltoall_bytes(send, sb, rb); mark("a2a_bytes")
            ctx.slab_unpack(ex.ptr(recv), rc); mark("unpack")
            st = ctx.slab_step(params, 0); mark("slab_step")
            ex.allreduce_sum([st.force_evals, st.candidates, st.degenerate_pairs, st.agent_count]); mark("counters")
            if it >= 2:
                for k in names:
                    acc[k].append(t[k])
    tg = [ctx.fetch_stats(ctx.steps - 1 - k) for k in range(min(steps, 8))]
    if r == 0:
        for k in names:
            print("%-12s %8.3f ms" % (k, float(np.median(acc[k]))))
        print("total        %8.3f ms" % sum(float(np.median(acc[k])) for k in names))
        print("device: t_grid %.3f t_force %.3f ms" % (np.median([s.t_grid_ms for s in tg]),
                                                      np.median([s.t_force_ms for s in tg])))
    # the single-context step on the same pool for comparison
    c2 = _native.Context(local, pool.dtype)
    c2.set_option(_native.CG_OPT_SUMMATION, 1)
    c2.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
    ts = []
    for it in range(steps + 2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s2 = c2.step(params, None, 1 << 24, _native.CG_STEP_SORT)
        torch.cuda.synchronize()
        if it >= 2:
            ts.append((time.perf_counter() - t0) * 1e3)
    if r == 0:
        print("single ctx step %.3f ms (t_grid %.3f t_force %.3f)" % (np.median(ts), s2.t_grid_ms, s2.t_force_ms))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
