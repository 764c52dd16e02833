mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:amsq_linear -s 3 -c 1 -o gpurun_out/prof_v6_s7_gu_m1 python tools/prof_linear.py --scheme fp5.33-e2m3 --n 28672 --k 4096 --m 1 > gpurun_out/ncu4a.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:amsq_linear -s 3 -c 1 -o gpurun_out/prof_v6_s7_o_m16 python tools/prof_linear.py --scheme fp5.33-e2m3 --n 4096 --k 4096 --m 16 > gpurun_out/ncu4b.log 2>&1
