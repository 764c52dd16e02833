# K2 quick loop: parity subset + graph-timed calls on the 8B shapes (both schemes, M = 1, 8, 16)
mkdir -p gpurun_out; rm -f gpurun_out/k2q.txt
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_k2q.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k2q.log
for lib in ${LIBS:-paper_2510_16045_b200/libamsq_b200.so}; do
  echo "== $lib" >> gpurun_out/k2q.txt
  for s in fp5.33-e2m3 fp4.25-e2m2; do for m in 1 8 16; do for nk in "28672 4096" "4096 4096" "6144 4096" "4096 14336"; do
   set -- $nk; AMSQ_LIB=$lib timeout 120 python tools/prof_linear.py --scheme $s --n $1 --k $2 --m $m --graph 2>&1 2>&1 | tail -1 | cut -c8-64 >> gpurun_out/k2q.txt
  done; done; done
done
