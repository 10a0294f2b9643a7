"""x-slab decomposition host logic on CPU: world-size 2 and 3 over gloo, each rank a
numpy/oracle mock of the slab C ABI (tests/slab_mock.py), driven by the real
SlabRunner.  The union of the ranks' pools after several steps (with agents
crossing slab boundaries) must equal a single-process oracle run bit for bit,
uid by uid, and the per-step global counters must agree."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

PARAMS5 = np.array([2.0, 1.0, 0.01, 3.0, 1.0])
PARAMS7 = np.array([2.0, 1.0, 0.01, 3.0, 1.0, 0.0, 1.0])


def _pool(jitter, big_steps=True):
    from paper_2105_00039_b200.pool import AgentPool
    from paper_2105_00039_b200.workloads import jittered_lattice_positions
    pos = jittered_lattice_positions(8, spacing=7.0, jitter=jitter, seed=3)
    pos[:, 0] *= 1.5      # elongated in x: several planes per slab
    return AgentPool.from_arrays(pos, 10.0, 0.4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, steps, params5, out_q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch.distributed as dist
    from slab_mock import MockSlabContext
    from paper_2105_00039_b200.distributed import SlabRunner, TorchExchange
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=rank, world_size=world)
    full = _pool(1.0, True)
    # initial distribution ignores the slab rule (uid parity): the first step
    # migrates about half of each rank's agents
    mine = (full.uid % world) == rank
    from paper_2105_00039_b200.pool import AgentPool
    sub = AgentPool(position_x=full.position_x[mine], position_y=full.position_y[mine],
                    position_z=full.position_z[mine], diameter=full.diameter[mine],
                    adherence=full.adherence[mine], uid=full.uid[mine])
    ctx = MockSlabContext(sub, np.concatenate([params5, [0.0, 1.0]]))
    runner = SlabRunner(ctx, TorchExchange(device="cpu", device_buffers=False))
    stats = [runner.step(params5) for _ in range(steps)]
    out_q.put((rank, ctx.uid, {c: v for c, v in ctx.cols.items()},
               [(s.force_evals, s.candidates, s.migrated_in + s.migrated_out) for s in stats]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,params5", [(2, PARAMS5), (2, np.array([2.0, 1.0, 2.0, 3.0, 0.1])),
                                           (3, PARAMS5)])
def test_slab_ranks_match_single_process(world, params5):
    import multiprocessing as mp
    import oracle
    from paper_2105_00039_b200.mechanics import ForceParams
    steps = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, steps, params5, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    uid = np.concatenate([r[1] for r in res])
    assert np.unique(uid).shape[0] == uid.shape[0]
    # single-process reference run (the oracle restates engine.step)
    ref = _pool(1.0, True)
    fp = ForceParams(kappa=params5[0], gamma=params5[1], timestep=params5[2],
                     max_displacement=params5[3], adherence_scale=params5[4])
    ref_counters = []
    for _ in range(steps):
        r = oracle.step(ref, fp, sort=False)
        ref_counters.append((r.force_evals, r.candidates))
    order_ref = np.argsort(ref.uid)
    order = np.argsort(uid)
    assert np.array_equal(uid[order], ref.uid[order_ref])
    for col in ("position_x", "position_y", "position_z", "displacement_x", "displacement_y",
                "displacement_z"):
        mine = np.concatenate([r[2][col] for r in res])[order]
        assert np.array_equal(mine, getattr(ref, col)[order_ref]), col
    # global counters of every step agree on both ranks and with the oracle
    for k in range(steps):
        assert all(r[3][k][:2] == ref_counters[k] for r in res)
    # agents did cross slab boundaries
    assert sum(x[2] for r in res for x in r[3]) > 0
