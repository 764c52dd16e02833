mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "large_batch or cpp_dropin" > gpurun_out/pytest_k3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k3.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:amsq_linear -s 3 -c 1 -o gpurun_out/prof_v2_s7_o_m1 python tools/prof_linear.py --scheme fp5.33-e2m3 --n 4096 --k 4096 --m 1 > gpurun_out/ncu_v2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:amsq_linear -s 3 -c 1 -o gpurun_out/prof_v2_s7_gu_m1 python tools/prof_linear.py --scheme fp5.33-e2m3 --n 28672 --k 4096 --m 1 >> gpurun_out/ncu_v2.log 2>&1
