# streaming ceilings + kernel timelines / profiling modes of the fused linear
mkdir -p gpurun_out
timeout 300 build/stream_probe > gpurun_out/stream_probe.txt 2>&1
rm -f gpurun_out/trace.txt gpurun_out/modes.txt
for args in "--n 4096 --k 4096 --m 1" "--n 28672 --k 4096 --m 1" "--n 28672 --k 4096 --m 1 --dry" "--n 4096 --k 4096 --m 1 --dry" "--n 4096 --k 14336 --m 1" "--n 28672 --k 4096 --m 16"; do
timeout 120 python tools/trace_linear.py $args >> gpurun_out/trace.txt 2>&1
done
for m in 1 16; do for d in 0 1 2 3 4; do for nk in "28672 4096" "4096 4096"; do set -- $nk
timeout 120 python tools/prof_linear.py --scheme fp5.33-e2m3 --n $1 --k $2 --m $m --graph --dry $d >> gpurun_out/modes.txt 2>&1
done; done; done
