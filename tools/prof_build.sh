#!/bin/bash
# ncu --set full of the C4 list build (second sweep7 launch of a resident run)
# and of the C2 dense grid sweep, at the current defaults.
mkdir -p gpurun_out
TAG=${TAG:-r2bc}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep7_kernel -s 1 -c 1 \
  -o gpurun_out/prof_${TAG}_build python tools/ab_steps.py c4 4 prof > gpurun_out/prof_${TAG}_build.log 2>&1
echo "build rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep7_kernel -s 3 -c 1 \
  -o gpurun_out/prof_${TAG}_c2 python tools/ab_steps.py c2 6 prof > gpurun_out/prof_${TAG}_c2.log 2>&1
echo "c2 rc $?"
