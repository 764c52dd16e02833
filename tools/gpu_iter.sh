# quick iteration: parity tests + per-shape graph timings (K2 and K3)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/graph_times.txt
for s in fp5.33-e2m3 fp4.25-e2m2; do for m in 1 8 16 32 128; do for nk in "28672 4096" "4096 4096" "6144 4096" "4096 14336"; do
 set -- $nk; timeout 120 python tools/prof_linear.py --scheme $s --n $1 --k $2 --m $m --graph 2>&1 | cut -c1-90 >> gpurun_out/graph_times.txt
done; done; done
