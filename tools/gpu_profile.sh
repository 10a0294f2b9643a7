#!/bin/bash
# ncu evidence for one config: launch list (cold, serialised) over STEPS steps,
# then one full capture of each sweep kernel: the grid sweep that builds the
# neighbour lists (first launch) and the list sweep (second launch).
# usage: bash tools/gpu_profile.sh <tag> [config] [sum] [relayout] [steps]
TAG=${1:-r1}; CFG=${2:-c4}; SUM=${3:-1}; ORD=${4:-1}; STEPS=${5:-12}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}_${CFG}.csv python tools/one_step.py $CFG $SUM $ORD $STEPS > gpurun_out/launches_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep7_kernel|sweep_warp" -s 1 -c 1 \
  -o gpurun_out/prof_${TAG}_${CFG}_sweep python tools/one_step.py $CFG $SUM $ORD 3 > gpurun_out/prof_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"list_sweep_kernel" -s 1 -c 1 \
  -o gpurun_out/prof_${TAG}_${CFG}_list python tools/one_step.py $CFG $SUM $ORD 5 >> gpurun_out/prof_${TAG}.log 2>&1
if [ -n "$GRID" ]; then
timeout 900 ncu --set full --clock-control none -k regex:"box_keys|scan_|place" -s 3 -c 4 \
  -o gpurun_out/prof_${TAG}_${CFG}_grid python tools/one_step.py $CFG $SUM $ORD 2 >> gpurun_out/prof_${TAG}.log 2>&1
fi
ls -la gpurun_out
