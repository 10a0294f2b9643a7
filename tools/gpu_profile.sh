#!/bin/bash
# ncu evidence for the C4 step: launch list (cold, serialised) + one full capture
# of the sweep kernel.  usage: bash tools/gpu_profile.sh <tag> [config] [sum] [order]
TAG=${1:-r1}; CFG=${2:-c4}; SUM=${3:-1}; ORD=${4:-1}
mkdir -p gpurun_out
./tools/fp64_peak > gpurun_out/fp64_peak.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}_${CFG}.csv python tools/one_step.py $CFG $SUM $ORD 3 > gpurun_out/launches_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep -s 2 -c 1 \
  -o gpurun_out/prof_${TAG}_${CFG}_sweep python tools/one_step.py $CFG $SUM $ORD 3 > gpurun_out/prof_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"box_keys|order_in_box|scan_tiles|place|gather|make_proxy|bbox" -s 8 -c 8 \
  -o gpurun_out/prof_${TAG}_${CFG}_grid python tools/one_step.py $CFG $SUM $ORD 2 >> gpurun_out/prof_${TAG}.log 2>&1
ls -la gpurun_out
