# quick GPU loop: correctness of the linear + graph timings at 8B shapes
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "linear or subnormal or determin" > gpurun_out/pytest_q.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q.log
rm -f gpurun_out/graph_times.txt
for s in fp5.33-e2m3 fp4.25-e2m2; do for m in 1 4 8 16; do for nk in "28672 4096" "4096 4096" "6144 4096" "4096 14336"; do
 set -- $nk; python tools/prof_linear.py --scheme $s --n $1 --k $2 --m $m --graph >> gpurun_out/graph_times.txt 2>&1
done; done; done
