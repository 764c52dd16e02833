mkdir -p gpurun_out; rm -f gpurun_out/variants.txt gpurun_out/trace.txt
timeout 900 python -m pytest tests -x -q -m gpu -k "linear_matches or deterministic or large_k" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for lib in paper_2510_16045_b200/libamsq_b200.so build/variants/libamsq_nopf.so build/variants/libamsq_m1.so; do
  echo "== $lib" >> gpurun_out/variants.txt
  for s in fp5.33-e2m3 fp4.25-e2m2; do for m in 1 8; do for nk in "28672 4096" "4096 4096" "6144 4096" "4096 14336"; do
   set -- $nk; AMSQ_LIB=$lib timeout 120 python tools/prof_linear.py --scheme $s --n $1 --k $2 --m $m --graph 2>&1 | cut -c1-90 >> gpurun_out/variants.txt
  done; done; done
done
for args in "--n 4096 --k 4096 --m 1" "--n 28672 --k 4096 --m 1"; do
AMSQ_LIB=build/variants/libamsq_trace.so timeout 120 python tools/trace_linear.py $args >> gpurun_out/trace.txt 2>&1
done
