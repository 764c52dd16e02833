#!/bin/bash
# parity (new epilogue, bf16), A/B vs the committed build, bench, per-case sanitizers
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/rc.txt
NOTEST=1 MS="1 4 8 16" timeout 1500 bash tools/gpu_ab.sh
echo "ab rc=$?" >> gpurun_out/rc.txt
timeout 600 python bench.py --no-cpu > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/rc.txt
for c in 1 2 3 4 5; do for t in racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_cases.py $c > gpurun_out/san_${t}_$c.log 2>&1
  echo "$t case $c rc=$?" >> gpurun_out/rc.txt
done; done
