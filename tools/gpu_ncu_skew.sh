#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_skew -s 4 -c 1 -o gpurun_out/prof_skew_C5 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu --fused on > gpurun_out/ncu_skew.log 2>&1
NSM_DEBUG_FULL_RINGS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_skew -s 4 -c 1 -o gpurun_out/prof_skew_C5_w65280 python tools/skew_exp_once.py C5 65280 > gpurun_out/ncu_skew2.log 2>&1
