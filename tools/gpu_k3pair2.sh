#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_config_shapes.py -x -q -m gpu -k "tcgen05 or k3" > gpurun_out/pytest_pair2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
for s in fp5.33-e2m3 fp4.25-e2m2; do for m in 128 256; do
  r=$(timeout 120 python tools/prof_linear.py --scheme $s --n 28672 --k 4096 --m $m --graph 2>&1 | tail -1 | sed 's/.*: \([0-9.]*\) us\/call.*/\1/')
  echo "$s gate_up M=$m $r" >> gpurun_out/pair_check.txt
done; done
