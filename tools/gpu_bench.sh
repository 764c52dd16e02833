mkdir -p gpurun_out
nproc > gpurun_out/host.txt; lscpu | grep -E 'Model name|^CPU\(s\)' >> gpurun_out/host.txt
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --steps 10 --warmup 3 --scheme fp4.25-e2m2 --no-cpu --no-extra > gpurun_out/bench_s4.json 2>> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > gpurun_out/bench_ncu.log 2>&1
