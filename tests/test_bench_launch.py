"""bench.py --gpus N launches N ranks by itself when it is not already under
torchrun (the driver's scaling run may call it either way): the process group
comes up with N ranks and rank 0 reports them.  The CPU test stops after the
rendezvous (gloo, no device); the GPU test runs the slab path for real with
both ranks on cuda:0 (gloo exchange) on a small C5 lattice."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    env.pop("LOCAL_RANK", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-3000:]     # rank 0 alone prints
    return json.loads(lines[0])


def test_gpus_2_relaunches_two_ranks():
    out = _run(["--gpus", "2", "--exchange", "gloo", "--launch-check"], 180)
    assert out["n_gpus"] == 2
    assert out["parallelism"] == "x-slabs x2 over gloo"


@pytest.mark.gpu
def test_gpus_2_slab_bench_same_device(cuda_required):
    out = _run(["--gpus", "2", "--same-device", "--exchange", "gloo", "--side", "32", "--steps", "4",
                "--warmup", "3", "--e2e-steps", "1"], 600)
    assert out["n_gpus"] == 2 and out["value"] > 0
    assert out["config"]["parallelism"].startswith("x-slabs x2")
    assert out["config"]["agents_total"] == 2 * 32 ** 3
    assert out["e2e"]["h2d_bytes_per_step"] > 0
