mkdir -p gpurun_out; rm -f gpurun_out/trace.txt
for args in "--n 4096 --k 4096 --m 1" "--n 28672 --k 4096 --m 1" "--n 28672 --k 4096 --m 1 --dry" "--n 4096 --k 14336 --m 1" "--n 28672 --k 4096 --m 16"; do
python tools/trace_linear.py $args >> gpurun_out/trace.txt 2>&1
done
