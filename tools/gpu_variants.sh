mkdir -p gpurun_out; rm -f gpurun_out/variants.txt
timeout 900 python -m pytest tests -x -q -m gpu -k "linear_matches or deterministic or large_k or subnormal" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for lib in paper_2510_16045_b200/libamsq_b200.so build/variants/libamsq_own8.so; do
  echo "== $lib" >> gpurun_out/variants.txt
  AMSQ_LIB=$lib timeout 300 python -m pytest tests -x -q -m gpu -k "linear_matches_reference_gemv" 2>&1 | tail -1 >> gpurun_out/variants.txt
  for s in fp5.33-e2m3 fp4.25-e2m2; do for m in 1 8; do for nk in "28672 4096" "4096 4096" "6144 4096" "4096 14336"; do
   set -- $nk; AMSQ_LIB=$lib timeout 120 python tools/prof_linear.py --scheme $s --n $1 --k $2 --m $m --graph 2>&1 | cut -c1-90 >> gpurun_out/variants.txt
  done; done; done
done
