#!/bin/bash
# A/B of list options through tools/ab_steps.py environment knobs (SKIN, MID,
# INNER in 1/1000 units) on one library; each setting twice, interleaved.
# usage: SETTINGS="2600:385:173 3000:385:173" CFG=c4:180 TAG=skin bash tools/ab_env.sh
mkdir -p gpurun_out
OUT=gpurun_out/ab_${TAG:-env}.jsonl
: > $OUT
for rep in 1 2; do
  for s in $SETTINGS; do
    IFS=: read SK MI IN <<< "$s"
    SKIN=$SK MID=$MI INNER=$IN timeout 300 python tools/ab_steps.py ${CFG%%:*} ${CFG##*:} "$s" >> $OUT 2>>gpurun_out/ab_err.log
  done
done
python - "$OUT" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    d = json.loads(l)
    print(d["tag"], round(d["mean_ms"], 4), {k: (d[k]["n"], round(d[k]["total_ms"], 4)) for k in ("build", "list") if k in d}, d["evals_hash"])
PY
