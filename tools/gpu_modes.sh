# K2 decomposition: full kernel vs stream-only (mode1), decode-only (mode2), MMA-only (mode3)
mkdir -p gpurun_out; rm -f gpurun_out/modes.txt
timeout 600 python -m pytest tests -x -q -m gpu -k "linear" > gpurun_out/pytest_modes.log 2>&1
for lib in paper_2510_16045_b200/libamsq_b200.so build/variants/libamsq_mode4.so; do
  echo "== $lib" >> gpurun_out/modes.txt
  for s in fp5.33-e2m3 fp4.25-e2m2; do for m in 1 8 16; do for nk in "28672 4096" "4096 4096" "6144 4096" "4096 14336"; do
   set -- $nk; AMSQ_LIB=$lib timeout 120 python tools/prof_linear.py --scheme $s --n $1 --k $2 --m $m --graph 2>&1 | cut -c1-90 >> gpurun_out/modes.txt
  done; done; done
done
