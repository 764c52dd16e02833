mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits > gpurun_out/smi_q.txt 2>&1
for s in fp5.33-e2m3 fp4.25-e2m2; do for m in 1 16; do
 python tools/prof_linear.py --scheme $s --n 28672 --k 4096 --m $m --graph >> gpurun_out/graph_times.txt 2>&1
 python tools/prof_linear.py --scheme $s --n 4096 --k 4096 --m $m --graph >> gpurun_out/graph_times.txt 2>&1
done; done
timeout 300 ncu --set full --import-source on -k regex:amsq_linear -s 4 -c 1 -o gpurun_out/prof_s7_m1 python tools/prof_linear.py --scheme fp5.33-e2m3 --n 28672 --k 4096 --m 1 > gpurun_out/ncu1.log 2>&1
timeout 300 ncu --set full --import-source on -k regex:amsq_linear -s 4 -c 1 -o gpurun_out/prof_s4_m16 python tools/prof_linear.py --scheme fp4.25-e2m2 --n 28672 --k 4096 --m 16 > gpurun_out/ncu2.log 2>&1
