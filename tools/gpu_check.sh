#!/bin/bash
# One GPU session: parity tests, smoke, per-phase probe, short bench.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --maxfail=8 -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
tail -2 gpurun_out/smoke.log
SUMS=${SUMS:-1,0} RELAYOUT=${RELAYOUT:-1} timeout 600 python tools/probe.py ${PROBE:-c1 c2 c4 c3_4 c3_100} > gpurun_out/probe.log 2>&1
cat gpurun_out/probe.log | cut -c1-220
[ -n "$NOBENCH" ] || timeout 600 python bench.py --steps 10 --warmup 3 --cpu-steps 1 > gpurun_out/bench.log 2>&1
tail -c 600 gpurun_out/bench.log
