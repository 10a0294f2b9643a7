"""Benchmark: agent-updates/s of the fp64 mechanical-interaction step on B200.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W`` prints ONE
JSON line on rank 0.  A "step" is one full reference step (engine.py:279-341):
Z-order re-sort, grid rebuild, 27-box force sweep, adherence gate, capped
displacement, apply -- on the device-resident population.

* value    -- agent-updates/s over all ranks, inputs resident in HBM, CUDA
              events on the context stream, max over ranks.
* e2e      -- the same metric through the public drop-in API
              (engine.step(pool, SimulationConfig(strategy=Gpu()))) with the
              pool in pinned host memory: H2D of the pool + step + D2H of the
              updated pool inside the timed region, every step.
* roofline -- the dominant kernel (the force sweep) against MEASURED_PEAKS.json
              hbm_gbs, algorithmic bytes 64 B/agent (fp64).
* cpu_baseline -- the C oracle (restatement of the reference path, OpenMP on
              all host cores) on rank 0, bounded sample of the same workload.

``--impl reference`` times the reference CPU path (the oracle port, all host
threads) on the same config and prints the same line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "agent-updates/s per mechanical step (fp64) at 1/2/4/8 B200; % HBM roofline"
UNIT = "agent-updates/s"
B_ALG = {"fp64": 64, "fp32": 32}     # 5 scalars read + 3 written per agent


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", help="c4 (default), c2, c1, c3_<density>")
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"])
    ap.add_argument("--summation", default="uid", choices=["uid", "stencil"],
                    help="dense pools only (sparse pools always sum each agent's pairs in uid order, "
                         "the reference's order)")
    ap.add_argument("--relayout-every", type=int, default=1,
                    help="move records into slot order on every k-th sort step")
    ap.add_argument("--sort-every", type=int, default=1)
    ap.add_argument("--list-skin", type=int, default=-1,
                    help="CG_OPT_LIST_SKIN: -1 auto (0.07 box lengths), 0 off, k > 0 = k/1000 length units")
    ap.add_argument("--freeze", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "gloo"],
                    help="multi-GPU exchange (gloo: host-staged, e.g. several ranks on one GPU)")
    ap.add_argument("--same-device", action="store_true", help="all ranks on cuda:0 (testing)")
    ap.add_argument("--force-slab", action="store_true",
                    help="run the slab (multi-GPU) driver even at world size 1 (exercises the exchange)")
    ap.add_argument("--side", type=int, default=256,
                    help="lattice side of C4 (and of each rank's C5 slab): 256 = the BASELINE config")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the other BASELINE configs (C4 lists off, C2, C3 sweep) in the N=1 line")
    ap.add_argument("--launch-check", action="store_true",
                    help="start the N ranks, initialise the process group, print world and exit (no GPU work)")
    return ap.parse_args()


def free_port():
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_relaunch(args):
    """``bench.py --gpus N`` (N > 1) outside torchrun: re-run this command as N
    ranks under torch.distributed.run on 127.0.0.1, one process per GPU."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")     # the communicator lines show N ranks
    env.setdefault("OMP_NUM_THREADS", "1")
    raise SystemExit(subprocess.call(cmd, env=env))


def make_pool(name, precision, rank=0, world=1, side=256):
    from paper_2105_00039_b200 import workloads
    from paper_2105_00039_b200.pool import PrecisionMode
    pm = PrecisionMode.FP64 if precision == "fp64" else PrecisionMode.FP32
    if name == "c4":
        return (workloads.c4(pm, side) if world == 1 else workloads.c5_shard(rank, world, pm, side)), \
            "C4: %d^3 jittered lattice (spacing 8, diameter 10, jitter +-1), %s agents" % (side, format(side ** 3, ",")) + \
            ("" if world == 1 else " per rank (C5 slab %d of %d)" % (rank, world))
    if name == "c2":
        return workloads.c2(pm), "C2: 1M uniform random, ref-density 27"
    if name == "c1":
        return workloads.c1(pm), "C1: 32^3 lattice spacing 8"
    if name.startswith("c3_"):
        c = float(name[3:])
        return workloads.c3(c, pm), "C3: 2M uniform random, %g colliding neighbours/agent" % c
    raise SystemExit("unknown config %s" % name)


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.lines = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        busy = [v for v in sm if mx and v > 0.5 * mx] or sm
        return {"sm_mhz": float(np.median(busy)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def profiled_kernel(config, precision, kernel):
    """ncu --set full figures of ``kernel`` from the committed capture
    (profiles/kernel_metrics.json, written by tools/kernel_metrics.py): DRAM
    bytes read + written per launch and the FP64 pipe's busy fraction."""
    try:
        with open(os.path.join(ROOT, "profiles", "kernel_metrics.json")) as fh:
            return json.load(fh).get("%s_%s" % (config, precision), {}).get(kernel) or {}
    except (OSError, ValueError, AttributeError):
        return {}


def fp64_view(cands, evals, ms):
    """Secondary roofline (diagnostic): the reference's cost model
    F = 11 flops per stencil candidate + 14 per kept pair (mechanics.py:34-40)
    per step, against the measured FP64 DFMA rate (profiles/r1_fp64_peak.json,
    tools/fp64_peak.cu)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r1_fp64_peak.json")) as fh:
            peak = float(json.load(fh)["dfma_tflops"])
    except (OSError, KeyError, ValueError):
        return None
    flops = 11.0 * cands + 14.0 * evals
    achieved = flops / (ms * 1e-3) / 1e12
    return {"alg_gflop_per_step": flops / 1e9, "achieved_tflops": achieved, "peak_tflops": peak,
            "frac": achieved / peak, "peak_source": "measured DFMA (profiles/r1_fp64_peak.json)"}


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_port_run(pool, precision, steps, sort_every, freeze):
    """The oracle (C restatement of the reference step) on all host threads;
    returns (median seconds per step, threads)."""
    import oracle
    from paper_2105_00039_b200.mechanics import ForceParams
    th = cpu_threads()
    oracle.lib()
    ts = []
    for k in range(steps):
        t0 = time.perf_counter()
        oracle.step(pool, ForceParams(), sort=(sort_every > 0 and k % sort_every == 0),
                    freeze=freeze, threads=th)
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)), th


def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.same_device:
        local = 0
    if world != args.gpus and rank == 0:
        print("bench.py: --gpus %d but WORLD_SIZE=%d; running %d rank(s)" % (args.gpus, world, world),
              file=sys.stderr)
    if world > 1 or (args.force_slab and args.impl == "ours"):
        import torch
        import torch.distributed as dist
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(free_port()))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        if args.exchange == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            if torch.cuda.is_available() and not args.launch_check:
                torch.cuda.set_device(local)
            dist.init_process_group("gloo")
    return rank, world, local


def reduce_max(v, world):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def run_reference(args, rank, world):
    if rank != 0:
        return
    pool, desc = make_pool(args.config, args.precision, side=args.side)
    n = pool.count
    # bounded sample: the full workload for as many of the K steps as fit in ~1 min of CPU time
    t_one, th = cpu_port_run(pool, args.precision, 1, args.sort_every, args.freeze)
    k_total = args.steps + args.warmup
    k_run = max(1, min(args.steps, int(60.0 / max(t_one, 1e-3)) - 1))
    t_med, th = cpu_port_run(pool, args.precision, k_run, args.sort_every, args.freeze)
    v = n / t_med
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": k_run, "warmup": 1, "ms_per_step": t_med * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
            "config": {"workload": desc, "agents": n, "sort_every": args.sort_every,
                       "freeze": args.freeze, "cpu_threads": th},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": th, "kind": "port", "cpu_model": cpu_model(),
                             "sample": "%d full step(s) of the %d-agent workload (requested K+W=%d)"
                                       % (k_run, n, k_total)},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main_slab(args, rank, world, local):
    """N > 1: C5 weak scaling -- each rank starts with its 256-plane x-slab of the
    (256 G) x 256 x 256 jittered lattice; x-slab decomposition: migration and
    ghost exchange on rebuild steps, ghost refresh on neighbour-list steps
    (paper_2105_00039_b200/distributed.py)."""
    import torch
    from paper_2105_00039_b200 import _native
    from paper_2105_00039_b200.distributed import SlabRunner, TorchExchange
    torch.cuda.set_device(local)
    pool, desc = make_pool(args.config, args.precision, rank, world, args.side)
    n0 = pool.count
    ctx = _native.Context(local, pool.dtype)
    ctx.set_option(_native.CG_OPT_SUMMATION, {"uid": 0, "stencil": 1}[args.summation])
    ctx.reserve(int(n0 * 1.05) + 4 * 256 * 256 * 2 + 4096)
    ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
    ex = TorchExchange(device="cuda", device_buffers=args.exchange == "nccl", stream=ctx.stream)
    # counters all-reduced once for the timed steps (inside the timed region)
    runner = SlabRunner(ctx, ex, sync_counters=False)
    params = np.array([2.0, 1.0, 0.01, 3.0, 1.0])
    flags = _native.CG_STEP_FREEZE if args.freeze else 0
    stream = torch.cuda.ExternalStream(ctx.stream)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            runner.step(params, flags)
        runner.collect()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        launches0 = ctx.launches
        barrier(world)
        torch.cuda.synchronize()
        with Clocks(local) as clk:
            ev0.record(stream)
            for _ in range(args.steps):
                runner.step(params, flags)
            stats = runner.collect()
            ev1.record(stream)
            torch.cuda.synchronize()
        launches = ctx.launches - launches0
        barrier(world)
    ms = reduce_max(ev0.elapsed_time(ev1) / args.steps, world)
    total = stats[-1].agents
    value = total / (ms * 1e-3)
    # the dominant sweep kernel over the timed steps still in the stats ring
    kinds, totals = {}, {}
    for k in range(min(args.steps, 60)):
        s_ = ctx.fetch_stats(ctx.steps - 1 - k)
        kinds.setdefault(int(s_.sweep_kind), []).append(float(s_.t_force_ms))
        totals.setdefault(int(s_.sweep_kind), []).append(float(s_.t_total_ms))
    dom = max(kinds, key=lambda k: sum(kinds[k]))
    names = {0: "grid_sweep", 1: "grid_sweep_list_build", 2: "list_sweep"}
    sweep_mix = {names[k]: {"steps": len(v), "mean_ms": float(np.mean(v)), "mean_step_device_ms": float(np.mean(totals[k]))}
                 for k, v in sorted(kinds.items())}
    t_force = reduce_max(float(np.mean(kinds[dom])), world)
    kernel_name = {0: "sweep7_kernel", 1: "sweep7_kernel_list_build", 2: "list_sweep_kernel"}[dom]
    n_local = ctx.n
    # e2e: each rank's shard crosses the host boundary every step (pinned
    # host -> device upload, slab step, device -> pinned host download)
    e2e = None
    if args.e2e_steps > 0:
        import time as _t
        cap = int(n0 * 1.05) + 4 * 256 * 256 * 2 + 4096
        pin = {k: _native.PinnedArray.empty(cap, np.uint64 if k == "uid" else pool.dtype)
               for k in ("px", "py", "pz", "diameter", "adherence", "uid", "dx", "dy", "dz")}
        cols = ctx.download()
        n = ctx.n
        for k in pin:
            pin[k][:n] = cols[k]
        barrier(world)
        torch.cuda.synchronize()
        t0 = _t.perf_counter()
        h2d = d2h = 0
        with torch.cuda.stream(stream):
            for _ in range(args.e2e_steps):
                ctx.upload(pin["px"][:n], pin["py"][:n], pin["pz"][:n], pin["diameter"][:n],
                           pin["adherence"][:n], pin["uid"][:n])
                h2d += n * (5 * np.dtype(pool.dtype).itemsize + 8)
                runner.step(params, flags)
                n = ctx.n
                ctx.download(into={k: v[:n] for k, v in pin.items()})
                d2h += n * (8 * np.dtype(pool.dtype).itemsize + 8)
            runner.collect()
        torch.cuda.synchronize()
        t_e2e = reduce_max((_t.perf_counter() - t0) / args.e2e_steps, world)
        e2e = {"value": total / t_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d // args.e2e_steps,
               "d2h_bytes_per_step": d2h // args.e2e_steps, "ms_per_step": t_e2e * 1e3,
               "scope": "rank 0's bytes; every rank moves its own shard",
               "api": "distributed.SlabRunner.step between cg_upload / cg_download of the shard"}
    ctx.close()
    if rank != 0:
        return
    peak, peak_src = measured_hbm_peak()
    bal = B_ALG[args.precision]
    achieved = n_local * bal / (t_force * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "config": {"workload": "C5: (%d x %d) x %d x %d jittered lattice, %d agents (%d per GPU at start)"
                               % (args.side, world, args.side, args.side, total, n0),
                   "agents_total": total, "summation": args.summation, "freeze": args.freeze,
                   "l2": "inputs larger than L2 (%.0f MB of agent state per GPU)" % (n0 * 64 / 1e6),
                   "parallelism": "x-slabs x%d over %s: migration + ghost exchange on rebuild steps, ghost refresh on "
                                  "neighbour-list steps" % (world, args.exchange)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None, "kernel": kernel_name + " (per GPU)",
                     "alg_bytes_per_agent": bal, "kernel_ms": t_force, "peak_source": peak_src,
                     "sweep_mix": sweep_mix},
        "step_roofline_frac": total / world * bal / (ms * 1e-3) / 1e9 / peak,
        "pair_interactions_per_s": stats[-1].force_evals / (ms * 1e-3),
        "candidates_per_s": stats[-1].candidates / (ms * 1e-3),
        "migrated_last_step": stats[-1].migrated_in, "ghosts_last_step": stats[-1].ghosts,
        "gpu_launches": launches,
        "e2e": e2e,
        "cpu_baseline": None,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


EXTRAS = (   # (key, config, precision, summation, list skin, sort_every, freeze) -- BASELINE.json configs
    ("c4_lists_off", "c4", "fp64", "uid", 0, 1, False),     # the literal "grid rebuild each step"
    ("c1_fp64", "c1", "fp64", "uid", -1, 1, False),         # the reference's own CPU-runnable case (32^3)
    ("c2_fp64", "c2", "fp64", "uid", -1, 1, False),
    ("c2_fp32", "c2", "fp32", "uid", -1, 1, False),
    ("c3_4_sorted", "c3_4", "fp64", "uid", -1, 1, True),
    ("c3_4_unsorted", "c3_4", "fp64", "uid", -1, 0, True),
    ("c3_27_sorted", "c3_27", "fp64", "uid", -1, 1, True),
    ("c3_27_unsorted", "c3_27", "fp64", "uid", -1, 0, True),
    ("c3_100_sorted", "c3_100", "fp64", "uid", -1, 1, True),
    ("c3_100_unsorted", "c3_100", "fp64", "uid", -1, 0, True),
)


def measure_resident(pool, precision, summation, skin, sort_every, freeze, steps, warmup, local=0):
    """Device time per resident step (CUDA events on the context stream) of one
    configuration; counters and step kinds of the timed steps."""
    import torch
    from paper_2105_00039_b200 import _native
    ctx = _native.Context(local, pool.dtype)
    ctx.set_option(_native.CG_OPT_SUMMATION, {"uid": 0, "stencil": 1}[summation])
    ctx.set_option(_native.CG_OPT_LIST_SKIN, skin)
    ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
    flags_for = lambda k: ((_native.CG_STEP_SORT if sort_every > 0 and k % sort_every == 0 else 0)
                           | (_native.CG_STEP_FREEZE if freeze else 0))
    params = np.array([2.0, 1.0, 0.01, 3.0, 1.0])
    for k in range(warmup):
        ctx.step(params, None, 1 << 24, flags_for(k))
    stream = torch.cuda.ExternalStream(ctx.stream)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.synchronize()
    ev0.record(stream)
    ids = [ctx.step(params, None, 1 << 24, flags_for(warmup + k), wait=False) for k in range(steps)]
    ev1.record(stream)
    ctx.synchronize()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / steps
    stats = [ctx.fetch_stats(i) for i in ids]
    ctx.close()
    kinds = {}
    for s_ in stats:
        kinds.setdefault(int(s_.sweep_kind), []).append(float(s_.t_force_ms))
    mix = {{0: "grid_sweep", 1: "grid_sweep_list_build", 2: "list_sweep"}[k]:
           {"steps": len(v), "mean_ms": float(np.mean(v))} for k, v in sorted(kinds.items())}
    evals = float(np.mean([s.force_evals for s in stats]))
    cands = float(np.mean([s.candidates for s in stats]))
    return ms, evals, cands, mix


def run_extras(args, c4_pool, local):
    peak, _ = measured_hbm_peak()
    out = {}
    pools = {}
    for key, cfg, prec, summ, skin, sort_every, freeze in EXTRAS:
        if args.precision != "fp64" and cfg == "c4":
            continue
        if cfg == "c4" and prec == args.precision and args.side == 256:
            pool, desc = c4_pool, "C4"
        else:
            if (cfg, prec) not in pools:
                pools = {(cfg, prec): make_pool(cfg, prec, side=args.side)}   # keep one host pool at a time
            pool, desc = pools[(cfg, prec)]
        ms, evals, cands, mix = measure_resident(pool, prec, summ, skin, sort_every, freeze, 10, 3, local)
        n = pool.count
        fv = fp64_view(cands, evals, ms)
        out[key] = {"workload": desc, "agents": n, "precision": prec, "summation": summ,
                    "lists": "off" if skin == 0 else "auto", "sort_every": sort_every, "freeze": freeze,
                    "ms_per_step": ms, "agent_updates_per_s": n / (ms * 1e-3),
                    "pair_interactions_per_s": evals / (ms * 1e-3),
                    "step_roofline_frac": n * B_ALG[prec] / (ms * 1e-3) / 1e9 / peak,
                    "fp64_view_frac": fv["frac"] if fv and prec == "fp64" else None,
                    "sweep_mix": mix}
    return out


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def main():
    args = parse()
    maybe_relaunch(args)
    rank, world, local = dist_init(args)
    if args.launch_check:
        barrier(world)
        if rank == 0:
            print(json.dumps({"launch_check": True, "n_gpus": world, "impl": args.impl,
                              "parallelism": "x-slabs x%d over %s" % (world, args.exchange) if world > 1
                              else "single GPU"}), flush=True)
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1 or args.force_slab:
        main_slab(args, rank, world, local)
        return
    import torch
    from paper_2105_00039_b200 import _native
    from paper_2105_00039_b200 import engine as eng
    from paper_2105_00039_b200.pool import PrecisionMode

    torch.cuda.set_device(local)
    pool, desc = make_pool(args.config, args.precision, rank, world, args.side)
    n = pool.count
    flags_for = lambda k: ((_native.CG_STEP_SORT if args.sort_every > 0 and k % args.sort_every == 0 else 0)
                           | (_native.CG_STEP_FREEZE if args.freeze else 0))
    ctx = _native.Context(local, pool.dtype)
    ctx.set_option(_native.CG_OPT_SUMMATION, {"uid": 0, "stencil": 1}[args.summation])
    ctx.set_option(_native.CG_OPT_RELAYOUT_EVERY, args.relayout_every)
    ctx.set_option(_native.CG_OPT_LIST_SKIN, args.list_skin)
    ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence,
               pool.uid)
    params = np.array([2.0, 1.0, 0.01, 3.0, 1.0])
    for k in range(args.warmup):
        ctx.step(params, None, 1 << 24, flags_for(k))
    stream = torch.cuda.ExternalStream(ctx.stream)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launches
    barrier(world)
    torch.cuda.synchronize()
    ctx.synchronize()
    with Clocks(local) as clk:
        ev0.record(stream)
        ids = [ctx.step(params, None, 1 << 24, flags_for(args.warmup + k), wait=False)
               for k in range(args.steps)]
        ev1.record(stream)
        ctx.synchronize()
        torch.cuda.synchronize()
    launches = ctx.launches - launches0
    barrier(world)
    ms = ev0.elapsed_time(ev1) / args.steps
    ms = reduce_max(ms, world)
    stats = [ctx.fetch_stats(i) for i in ids[-min(len(ids), 60):]]
    # the dominant sweep kernel of the timed region (most total time): the
    # grid sweep (kind 0), the grid sweep that also builds neighbour lists
    # (kind 1) or the list sweep (kind 2, csrc/list.cuh)
    kinds = {}
    for s_ in stats:
        kinds.setdefault(int(s_.sweep_kind), []).append(float(s_.t_force_ms))
    dom = max(kinds, key=lambda k: sum(kinds[k]))
    t_force = float(np.mean(kinds[dom]))
    kernel_name = {0: "sweep7_kernel", 1: "sweep7_kernel_list_build", 2: "list_sweep_kernel"}[dom]
    sweep_mix = {{0: "grid_sweep", 1: "grid_sweep_list_build", 2: "list_sweep"}[k]:
                 {"steps": len(v), "mean_ms": float(np.mean(v))} for k, v in sorted(kinds.items())}
    evals = float(np.mean([s.force_evals for s in stats]))
    cands = float(np.mean([s.candidates for s in stats]))
    value = n * world / (ms * 1e-3)
    ctx.close()

    # e2e: the public drop-in API with pinned host columns, H2D + step + D2H every step
    e2e = None
    if args.e2e_steps > 0:
        pin = _native.PinnedArray.copy_of
        from paper_2105_00039_b200.pool import AgentPool
        hp = AgentPool(position_x=pin(pool.position_x), position_y=pin(pool.position_y),
                       position_z=pin(pool.position_z), diameter=pin(pool.diameter),
                       adherence=pin(pool.adherence), uid=pin(pool.uid),
                       displacement_x=pin(pool.displacement_x), displacement_y=pin(pool.displacement_y),
                       displacement_z=pin(pool.displacement_z))
        cfg = eng.SimulationConfig(strategy=eng.Gpu(device=local, summation=args.summation,
                                                    relayout_every=args.relayout_every),
                                   precision=PrecisionMode.FP64 if args.precision == "fp64" else PrecisionMode.FP32,
                                   morton_sort_every=args.sort_every, freeze_displacement=args.freeze)
        eng.step(hp, cfg, 0)                       # warm the context
        barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(args.e2e_steps):
            eng.step(hp, cfg, k + 1)
        torch.cuda.synchronize()
        t_e2e = reduce_max((time.perf_counter() - t0) / args.e2e_steps, world)
        es = np.dtype(pool.dtype).itemsize
        # a sort step brings every column back (new storage order); an unsorted
        # one only positions and displacements (engine.step)
        sorted_steps = sum(1 for k in range(args.e2e_steps)
                           if args.sort_every > 0 and (k + 1) % args.sort_every == 0)
        d2h = (sorted_steps * n * (8 * es + 8) + (args.e2e_steps - sorted_steps) * n * 6 * es) // args.e2e_steps
        e2e = {"value": n * world / t_e2e, "unit": UNIT,
               "h2d_bytes_per_step": n * (5 * es + 8), "d2h_bytes_per_step": d2h,
               "ms_per_step": t_e2e * 1e3, "api": "engine.step(pool, SimulationConfig(strategy=Gpu()))"}

    extras = None
    if world == 1 and args.config == "c4" and not args.no_extras:
        extras = run_extras(args, pool, local)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cp, _ = make_pool(args.config, args.precision, side=args.side)
        t_med, th = cpu_port_run(cp, args.precision, args.cpu_steps, args.sort_every, args.freeze)
        cpu = {"value": cp.count / t_med, "unit": UNIT, "cores": th, "kind": "port", "cpu_model": cpu_model(),
               "sample": "%d full step(s) of the same %d-agent workload, median" % (args.cpu_steps, cp.count)}

    if rank != 0:
        return
    peak, peak_src = measured_hbm_peak()
    bal = B_ALG[args.precision]
    achieved = n * bal / (t_force * 1e-3) / 1e9
    prof = profiled_kernel(args.config, args.precision, kernel_name)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "config": {"workload": desc, "agents_per_gpu": n, "sort_every": args.sort_every,
                   "freeze": args.freeze, "summation": args.summation, "relayout_every": args.relayout_every,
                   "l2": "inputs larger than L2 (%.0f MB of agent state per GPU)" % (n * (6 * np.dtype(pool.dtype).itemsize + 8) / 1e6),
                   "parallelism": "single GPU" if world == 1 else "replicas x%d (no halo exchange)" % world},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": prof.get("traffic"),
                     "fp64_pipe_frac": prof.get("fp64_pipe_frac"), "profile": prof.get("source"),
                     "kernel": kernel_name, "alg_bytes_per_agent": bal,
                     "kernel_ms": t_force, "peak_source": peak_src, "sweep_mix": sweep_mix},
        "step_roofline_frac": n * bal / (ms * 1e-3) / 1e9 / peak,
        "fp64_view": fp64_view(cands, evals, ms),
        "pair_interactions_per_s": evals * world / (ms * 1e-3),
        "candidates_per_s": cands * world / (ms * 1e-3),
        "gpu_launches": launches,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "extra": extras,
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
