#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for c in 5 6 7; do
  timeout 600 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_cases.py $c > gpurun_out/sanitize_racecheck_k3case$c.log 2>&1; echo "racecheck $c rc=$?" >> gpurun_out/rc.txt
done
rm -f gpurun_out/k3f.txt
for s in fp5.33-e2m3 fp4.25-e2m2; do for m in 64 128; do for nk in "28672 4096" "4096 4096"; do
  set -- $nk
  b=$(timeout 120 python tools/prof_linear.py --scheme $s --n $1 --k $2 --m $m --graph --k3min 1 2>&1 | tail -1 | sed 's/.*: \([0-9.]*\) us\/call.*/\1/')
  echo "$s $1x$2 M=$m K3(fenced)=$b" >> gpurun_out/k3f.txt
done; done; done
NOTEST=1 MS="1 4 8" EXTRA_LIBS="build/variants/libamsq_xp1.so" bash tools/gpu_ab.sh
echo "ab done" >> gpurun_out/rc.txt
