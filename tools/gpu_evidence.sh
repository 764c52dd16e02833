#!/bin/bash
# round-end evidence on the working tree: parity (all GPU tests), bench (both schemes) + reference
# arm, launch list, ncu --set full of K2 (gate_up M=1, o M=1) and K3 (gate_up M=128), SASS listing
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; lscpu | grep -E 'Model name|^CPU\(s\)' >> gpurun_out/host.txt
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
timeout 900 python bench.py --steps 10 --warmup 3 --extra gpurun_out/bench_extra.json > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/rc.txt
timeout 600 python bench.py --steps 10 --warmup 3 --scheme fp4.25-e2m2 --no-cpu > gpurun_out/bench_s4.json 2>> gpurun_out/bench.err; echo "bench4 rc=$?" >> gpurun_out/rc.txt
timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err; echo "ref rc=$?" >> gpurun_out/rc.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_ncu.log 2>&1; echo "launch rc=$?" >> gpurun_out/rc.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:amsq_linear_kernel -s 3 -c 1 -o gpurun_out/prof_k2_s7_gu_m1 python tools/prof_linear.py --scheme fp5.33-e2m3 --n 28672 --k 4096 --m 1 > gpurun_out/ncu.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:amsq_linear_kernel -s 3 -c 1 -o gpurun_out/prof_k2_s7_o_m1 python tools/prof_linear.py --scheme fp5.33-e2m3 --n 4096 --k 4096 --m 1 >> gpurun_out/ncu.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:amsq_linear_tc -s 2 -c 1 -o gpurun_out/prof_k3_s7_gu_m128 python tools/prof_linear.py --scheme fp5.33-e2m3 --n 28672 --k 4096 --m 128 >> gpurun_out/ncu.log 2>&1
echo "ncu done" >> gpurun_out/rc.txt
