#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
AMSQ_LIB=build/variants/libamsq_tcsmem.so timeout 600 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_cases.py 6 > gpurun_out/sanitize_racecheck_case6_smemA.log 2>&1; echo "smemA rc=$?" >> gpurun_out/rc.txt
timeout 600 compute-sanitizer --tool racecheck --racecheck-report all --error-exitcode 9 python tools/sanitize_cases.py 6 > gpurun_out/sanitize_racecheck_case6_all.log 2>&1; echo "tmemA rc=$?" >> gpurun_out/rc.txt
