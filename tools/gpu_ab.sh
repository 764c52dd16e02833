# A/B: time the committed build (build/variants/libamsq_base.so) against the working tree, interleaved
mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
[ -n "$NOTEST" ] || { timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log; }
for rep in 1 2; do
for s in ${SCHEMES:-fp5.33-e2m3 fp4.25-e2m2}; do for m in ${MS:-1 8 16}; do for nk in "28672 4096" "4096 4096" "6144 4096" "4096 14336"; do
  set -- $nk
  for lib in build/variants/libamsq_base.so paper_2510_16045_b200/libamsq_b200.so ${EXTRA_LIBS}; do
    r=$(AMSQ_LIB=$lib timeout 120 python tools/prof_linear.py --scheme $s --n $1 --k $2 --m $m --graph 2>&1 | tail -1 | sed 's/.*: \([0-9.]*\) us\/call.*/\1/')
    echo "$rep $s $1x$2 M=$m $(basename $lib) $r" >> gpurun_out/ab.txt
  done
done; done; done; done
python tools/ab_table.py gpurun_out/ab.txt > gpurun_out/ab_table.txt 2>&1
