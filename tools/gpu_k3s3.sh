#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
rm -f gpurun_out/k3s3.txt
for s in fp5.33-e2m3 fp4.25-e2m2; do for m in 48 64 128 256; do for nk in "28672 4096" "4096 14336" "6144 4096"; do
  set -- $nk
  a=$(timeout 120 python tools/prof_linear.py --scheme $s --n $1 --k $2 --m $m --graph --k3min 1 2>&1 | tail -1 | sed 's/.*: \([0-9.]*\) us\/call.*/\1/')
  b=$(AMSQ_LIB=build/variants/libamsq_big.so timeout 120 python tools/prof_linear.py --scheme $s --n $1 --k $2 --m $m --graph --k3min 1 2>&1 | tail -1 | sed 's/.*: \([0-9.]*\) us\/call.*/\1/')
  echo "$s $1x$2 M=$m base=$a big=$b" >> gpurun_out/k3s3.txt
done; done; done
