#!/bin/bash
# compute-sanitizer racecheck + synccheck on every K2 / K3 case of tools/sanitize_cases.py,
# memcheck over all of them (logs: gpurun_out/sanitize_*.log; summaries under profiles/)
# NOTE: compute-sanitizer is now closed on the GPU pool (runs under it left GPUs needing a reset);
# the committed logs under profiles/r02/sanitize_* predate that.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for c in ${CASES:-0 1 2 3 4 5 6 7 8}; do
  for tool in racecheck synccheck; do
    timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py $c > gpurun_out/sanitize_${tool}_case$c.log 2>&1; echo "$tool $c rc=$?" >> gpurun_out/rc.txt
  done
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitize_memcheck_all.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/rc.txt
