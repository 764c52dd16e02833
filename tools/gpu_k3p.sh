#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:amsq_linear_tc -s 2 -c 1 -o gpurun_out/prof_k3t_gu_m128 python tools/prof_linear.py --scheme fp5.33-e2m3 --n 28672 --k 4096 --m 128 > gpurun_out/ncu.log 2>&1
for spec in "28672 4096 128" "4096 4096 128" "28672 4096 256"; do
  set -- $spec
  timeout 120 python tools/trace_tc.py --n $1 --k $2 --m $3 >> gpurun_out/trace_tc.txt 2>&1
done
echo done >> gpurun_out/rc.txt
