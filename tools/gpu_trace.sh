mkdir -p gpurun_out; rm -f gpurun_out/trace.txt
for args in "--n 4096 --k 4096 --m 1" "--n 4096 --k 4096 --m 8" "--n 4096 --k 14336 --m 1" "--n 28672 --k 4096 --m 1"; do
timeout 120 python tools/trace_linear.py $args >> gpurun_out/trace.txt 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:amsq_linear -s 3 -c 1 -o gpurun_out/prof_v1_s7_down_m1 python tools/prof_linear.py --scheme fp5.33-e2m3 --n 4096 --k 14336 --m 1 > gpurun_out/ncu_v1.log 2>&1
