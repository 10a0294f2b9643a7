#!/bin/bash
# ncu --set full of ten consecutive C4 list-sweep launches (sub-list sweeps and
# refreshes: tools/kernel_metrics.py picks per template), then the step-gap probe.
mkdir -p gpurun_out
TAG=${TAG:-r2bb}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:list_sweep_kernel -s 20 -c 10 \
  -o gpurun_out/prof_${TAG}_list python tools/ab_steps.py c4 40 prof > gpurun_out/prof_${TAG}.log 2>&1
echo "ncu rc $?"
timeout 300 python tools/gap_probe.py > gpurun_out/gap_${TAG}.log 2>&1; cat gpurun_out/gap_${TAG}.log | tail -2
