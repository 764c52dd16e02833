#!/bin/bash
# parity of the K2 spread / kpw-tail changes, then A/B against the committed build
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_config_shapes.py tests/test_gpu_kernels.py -x -q -m gpu > gpurun_out/pytest_r2g.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
NOTEST=1 MS="1 8 16" bash tools/gpu_ab.sh
echo "ab done" >> gpurun_out/rc.txt
