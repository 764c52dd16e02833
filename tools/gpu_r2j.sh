#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_config_shapes.py -x -q -m gpu > gpurun_out/pytest_r2j.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
for c in 5 6 7; do
  for tool in racecheck synccheck; do
    timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py $c > gpurun_out/sanitize_${tool}_k3case$c.log 2>&1; echo "$tool $c rc=$?" >> gpurun_out/rc.txt
  done
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitize_memcheck_all.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/rc.txt
