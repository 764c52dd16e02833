#!/bin/bash
# full parity suite (8 schemes, bf16, fused TP), A/B with variants, traces, racecheck w/ proxy fence
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 --durations=15 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/rc.txt
NOTEST=1 MS="1 8" EXTRA_LIBS="build/variants/libamsq_nosleep.so build/variants/libamsq_pfence.so" timeout 1500 bash tools/gpu_ab.sh
echo "ab rc=$?" >> gpurun_out/rc.txt
for lib in build/variants/libamsq_base.so paper_2510_16045_b200/libamsq_b200.so; do
  for nk in "4096 4096" "28672 4096"; do set -- $nk
    AMSQ_LIB=$lib timeout 120 python tools/trace_linear.py --n $1 --k $2 --m 1 >> gpurun_out/trace_$(basename $lib .so).txt 2>&1
  done
done
AMSQ_LIB=build/variants/libamsq_pfence.so timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_cases.py 1 > gpurun_out/san_racecheck_1_pfence.log 2>&1
echo "racecheck pfence rc=$?" >> gpurun_out/rc.txt
timeout 600 python bench.py --no-cpu > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/rc.txt
