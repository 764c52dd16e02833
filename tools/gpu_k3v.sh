mkdir -p gpurun_out; rm -f gpurun_out/trace_tc.txt
for lib in paper_2510_16045_b200/libamsq_b200.so build/variants/libamsq_nofence.so; do
echo "== $lib" >> gpurun_out/trace_tc.txt
AMSQ_LIB=$lib timeout 120 python tools/trace_tc.py --n 4096 --k 4096 --m 32 >> gpurun_out/trace_tc.txt 2>&1
AMSQ_LIB=$lib timeout 120 python tools/prof_linear.py --n 4096 --k 4096 --m 32 --graph 2>&1 | cut -c1-80 >> gpurun_out/trace_tc.txt
done
