mkdir -p gpurun_out; rm -f gpurun_out/dry.txt
for m in 1 16; do for nk in "28672 4096" "4096 4096"; do set -- $nk
python tools/prof_linear.py --scheme fp5.33-e2m3 --n $1 --k $2 --m $m --graph --dry >> gpurun_out/dry.txt 2>&1
python tools/prof_linear.py --scheme fp5.33-e2m3 --n $1 --k $2 --m $m --graph >> gpurun_out/dry.txt 2>&1
done; done
python - >> gpurun_out/dry.txt 2>&1 <<'PY'
import torch
x=torch.zeros(1,device='cuda'); g=torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(100): x.add_(1)
g.replay(); torch.cuda.synchronize()
a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20): g.replay()
b.record(); torch.cuda.synchronize(); print("tiny kernel in graph: %.2f us/launch"%(a.elapsed_time(b)*1e3/2000))
PY
timeout 300 ncu --set full --clock-control none -k regex:amsq_linear -s 3 -c 1 -o gpurun_out/prof_v3_s7_m1 python tools/prof_linear.py --scheme fp5.33-e2m3 --n 28672 --k 4096 --m 1 > gpurun_out/ncu3.log 2>&1
for nk in "6144 4096" "4096 14336"; do set -- $nk
python tools/prof_linear.py --scheme fp5.33-e2m3 --n $1 --k $2 --m 1 --graph --dry >> gpurun_out/dry.txt 2>&1
done
