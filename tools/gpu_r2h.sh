#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_quantize.py -x -q -m gpu > gpurun_out/pytest_quant.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
timeout 300 python tools/bench_quantize.py > gpurun_out/bench_quantize.txt 2>&1; echo "bq rc=$?" >> gpurun_out/rc.txt
for lib in build/variants/libamsq_base.so build/variants/libamsq_coloc.so; do
  AMSQ_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_$(basename $lib .so).json 2>>gpurun_out/bench.err
done
echo "bench done" >> gpurun_out/rc.txt
NOTEST=1 MS="1 4 8" EXTRA_LIBS="build/variants/libamsq_coloc.so" bash tools/gpu_ab.sh
echo "ab done" >> gpurun_out/rc.txt
