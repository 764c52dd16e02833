#!/bin/bash
# sanitizers after the DSMEM/convergence fixes + ncu source-level capture of K2 + launch list
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for t in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$?" >> gpurun_out/rc.txt
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:amsq_linear_kernel -s 3 -c 1 \
  -o gpurun_out/ncu_k2_s7_gu_m1 python tools/prof_linear.py --scheme fp5.33-e2m3 --n 28672 --k 4096 --m 1 > gpurun_out/ncu_a.log 2>&1
echo "ncu_a rc=$?" >> gpurun_out/rc.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_under_ncu.log 2>&1
echo "ncu_launches rc=$?" >> gpurun_out/rc.txt
