#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_config_shapes.py -x -q -m gpu -k "tcgen05 or k3" > gpurun_out/pytest_pair.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
rm -f gpurun_out/pair_ab.txt
for s in fp5.33-e2m3 fp4.25-e2m2; do for m in 48 64 128 256; do for nk in "28672 4096" "57344 8192" "14336 4096"; do
  set -- $nk
  a=$(AMSQ_LIB=build/variants/libamsq_nopair.so timeout 120 python tools/prof_linear.py --scheme $s --n $1 --k $2 --m $m --graph --k3min 1 2>&1 | tail -1 | sed 's/.*: \([0-9.]*\) us\/call.*/\1/')
  b=$(timeout 120 python tools/prof_linear.py --scheme $s --n $1 --k $2 --m $m --graph --k3min 1 2>&1 | tail -1 | sed 's/.*: \([0-9.]*\) us\/call.*/\1/')
  echo "$s $1x$2 M=$m single=$a pair=$b" >> gpurun_out/pair_ab.txt
done; done; done
echo "ab done" >> gpurun_out/rc.txt
