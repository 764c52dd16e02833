#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for m in 8 16; do
timeout 300 ncu --set full --clock-control none --import-source on -k regex:amsq_linear_kernel -s 3 -c 1 -o gpurun_out/prof_k2_gu_m$m python tools/prof_linear.py --scheme fp5.33-e2m3 --n 28672 --k 4096 --m $m > gpurun_out/ncu_$m.log 2>&1
done
echo done >> gpurun_out/rc.txt
