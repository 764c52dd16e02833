mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "large_batch or tcgen05 or cpp_dropin" > gpurun_out/pytest_k3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k3.log
rm -f gpurun_out/k3_times.txt
for s in fp5.33-e2m3 fp4.25-e2m2; do for m in 32 128 256; do for nk in "28672 4096" "4096 4096"; do
 set -- $nk; timeout 120 python tools/prof_linear.py --scheme $s --n $1 --k $2 --m $m --graph 2>&1 | cut -c1-90 >> gpurun_out/k3_times.txt
done; done; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:amsq_linear_tc -s 2 -c 1 -o gpurun_out/prof_k3_s7_o_m32 python tools/prof_linear.py --scheme fp5.33-e2m3 --n 4096 --k 4096 --m 32 > gpurun_out/ncu_k3.log 2>&1
