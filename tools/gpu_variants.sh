mkdir -p gpurun_out; rm -f gpurun_out/variants.txt
timeout 600 python -m pytest tests -x -q -m gpu -k "large_batch or tp_device or cpp_dropin or deterministic" > gpurun_out/pytest_k3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k3.log
for lib in paper_2510_16045_b200/libamsq_b200.so build/variants/libamsq_mode1.so build/variants/libamsq_mode2.so build/variants/libamsq_mode3.so; do
  echo "== $lib" >> gpurun_out/variants.txt
  for s in fp5.33-e2m3 fp4.25-e2m2; do for m in 1; do for nk in "28672 4096" "4096 4096" "6144 4096" "4096 14336"; do
   set -- $nk; AMSQ_LIB=$lib timeout 120 python tools/prof_linear.py --scheme $s --n $1 --k $2 --m $m --graph 2>&1 | cut -c1-90 >> gpurun_out/variants.txt
  done; done; done
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-extra --no-cpu > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
