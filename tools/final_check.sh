#!/bin/bash
# Round-end verification on one B200: GPU tests, smoke, the bench line, the
# reference arm, and the launch list of a short bench (cold, serialised).
mkdir -p gpurun_out
bash tools/verify_head.sh
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.jsonl 2> gpurun_out/bench_ref.err; tail -c 600 gpurun_out/bench_ref.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv \
  python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-extras > gpurun_out/launches_final.log 2>&1
echo "ncu rc $?"
