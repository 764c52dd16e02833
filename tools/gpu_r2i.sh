#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python tools/chain_ab.py fp5.33-e2m3 > gpurun_out/chain_ab.txt 2>&1; echo "chain rc=$?" >> gpurun_out/rc.txt
for spec in "28672 4096 1" "4096 4096 1" "6144 4096 1" "4096 14336 1" "28672 4096 16" "4096 4096 16"; do
  set -- $spec
  timeout 120 python tools/trace_linear.py --n $1 --k $2 --m $3 >> gpurun_out/trace.txt 2>&1
done
echo "trace done" >> gpurun_out/rc.txt
