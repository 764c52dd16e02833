#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python tools/chain_ab.py fp5.33-e2m3 > gpurun_out/chain_ab.txt 2>&1
echo "chain rc=$?" >> gpurun_out/rc.txt
NOTEST=1 MS="1 8" EXTRA_LIBS="build/variants/libamsq_epiold.so build/variants/libamsq_lean.so" timeout 1500 bash tools/gpu_ab.sh
echo "ab rc=$?" >> gpurun_out/rc.txt
