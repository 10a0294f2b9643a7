#!/bin/bash
# A/B of library variants on one GPU: every build/<variant>.so named in $VARIANTS
# over the configs in $CONFIGS (tools/ab_steps.py), interleaved twice; optional
# parity run of the GPU tests against one variant ($TESTLIB, $TESTS).
# usage: VARIANTS="base seeded" CONFIGS="c4:120 c2:40" TAG=r2x bash tools/ab_run.sh
mkdir -p gpurun_out
OUT=gpurun_out/ab_${TAG:-x}.jsonl
: > $OUT
if [ -n "$TESTLIB" ]; then
  CG_LIB=build/$TESTLIB.so timeout 1500 python -m pytest ${TESTS:-tests} -m gpu -q -x > gpurun_out/pytest_${TESTLIB}.log 2>&1
  echo "pytest $TESTLIB rc $?"; tail -2 gpurun_out/pytest_${TESTLIB}.log
fi
for rep in 1 2; do
  for cfg in $CONFIGS; do
    for v in $VARIANTS; do
      CG_LIB=build/$v.so timeout 300 python tools/ab_steps.py ${cfg%%:*} ${cfg##*:} $v >> $OUT 2>>gpurun_out/ab_err.log
    done
  done
done
python - "$OUT" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    d = json.loads(l)
    print(d["tag"], d["config"], round(d["mean_ms"], 4), {k: round(d[k]["total_ms"], 4) for k in ("grid", "build", "list") if k in d}, d["evals_hash"], d["pos_hash"])
PY
