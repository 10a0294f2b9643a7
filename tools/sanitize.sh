#!/bin/bash
# compute-sanitizer over the library's kernels on small pools (GPU box):
# memcheck on every step kind (grid sweep, list build, whole-list / sub-list
# sweeps, deferred slow path, dense thread and warp sweeps, behaviour phase),
# racecheck + synccheck on the shared-memory kernels.  Logs -> gpurun_out/sanitize_*.txt
set -u
mkdir -p gpurun_out
CS="compute-sanitizer --error-exitcode 17 --print-limit 20"
run() { local tag=$1; shift; echo "== $tag: $*" ; timeout 1200 $CS "$@" > gpurun_out/sanitize_$tag.txt 2>&1; echo "rc=$?"; tail -2 gpurun_out/sanitize_$tag.txt; }
run smoke_memcheck --tool memcheck python -c "import __graft_entry__ as g; g.smoke()"
run lists_memcheck --tool memcheck python -m pytest tests/test_gpu_lists.py -x -q -k "long_run or coincident"
run dense_memcheck --tool memcheck python tools/dense_probe.py 12000 216 0
run dense27_memcheck --tool memcheck python tools/dense_probe.py 20000 27 0
run behaviour_memcheck --tool memcheck python -m pytest tests/test_behaviour.py -x -q -k "run"
run dense_racecheck --tool racecheck python tools/dense_probe.py 6000 27 0
run dense_synccheck --tool synccheck python tools/dense_probe.py 6000 216 0
run lists_racecheck --tool racecheck python -m pytest tests/test_gpu_lists.py -x -q -k "coincident"
run slab_memcheck --tool memcheck --target-processes all python -m pytest tests/test_slab_gpu.py -x -q -k "test_slab_ranks_match_single_context and 2-0--1"
run uid64_memcheck --tool memcheck python -m pytest tests/test_gpu_uid64.py -x -q
