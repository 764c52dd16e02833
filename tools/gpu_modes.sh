mkdir -p gpurun_out; rm -f gpurun_out/modes.txt
for s in fp5.33-e2m3 fp4.25-e2m2; do for m in 1 16; do for d in 0 1 2 3; do
python tools/prof_linear.py --scheme $s --n 28672 --k 4096 --m $m --graph --dry $d >> gpurun_out/modes.txt 2>&1
done; done; done
