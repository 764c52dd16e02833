mkdir -p gpurun_out; rm -f gpurun_out/modes2.txt
for m in 1 16; do for d in 1 4; do
python tools/prof_linear.py --scheme fp5.33-e2m3 --n 28672 --k 4096 --m $m --graph --dry $d >> gpurun_out/modes2.txt 2>&1
python tools/prof_linear.py --scheme fp5.33-e2m3 --n 4096 --k 4096 --m $m --graph --dry $d >> gpurun_out/modes2.txt 2>&1
done; done
