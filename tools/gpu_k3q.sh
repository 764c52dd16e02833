# K3 quick loop: trace two shapes, graph-timed calls, the K3 parity tests
mkdir -p gpurun_out; rm -f gpurun_out/k3q.txt
timeout 120 python tools/trace_tc.py --n 4096 --k 4096 --m 32 >> gpurun_out/k3q.txt 2>&1
timeout 120 python tools/trace_tc.py --n 28672 --k 4096 --m 128 >> gpurun_out/k3q.txt 2>&1
for m in 32 64 128 256; do
  timeout 120 python tools/prof_linear.py --n 28672 --k 4096 --m $m --graph 2>&1 | cut -c1-100 >> gpurun_out/k3q.txt
  timeout 120 python tools/prof_linear.py --n 4096 --k 4096 --m $m --graph 2>&1 | cut -c1-100 >> gpurun_out/k3q.txt
done
timeout 600 python -m pytest tests -q -m gpu -k "tc or large or batch" >> gpurun_out/k3q.txt 2>&1
