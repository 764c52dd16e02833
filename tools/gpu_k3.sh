mkdir -p gpurun_out; rm -f gpurun_out/trace_tc.txt gpurun_out/k3_times.txt
timeout 900 python -m pytest tests -x -q -m gpu -k "large_batch or tcgen05 or cpp_dropin" > gpurun_out/pytest_k3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k3.log
for args in "--n 4096 --k 4096 --m 32" "--n 4096 --k 4096 --m 256"; do
timeout 120 python tools/trace_tc.py $args >> gpurun_out/trace_tc.txt 2>&1
done
for s in fp5.33-e2m3 fp4.25-e2m2; do for m in 32 128 256; do for nk in "28672 4096" "4096 4096" "4096 14336"; do
 set -- $nk; timeout 120 python tools/prof_linear.py --scheme $s --n $1 --k $2 --m $m --graph --cublas 2>&1 | cut -c1-90 >> gpurun_out/k3_times.txt
done; done; done
