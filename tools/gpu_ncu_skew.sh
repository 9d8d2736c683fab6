#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_skew -s 4 -c 1 -o gpurun_out/prof_skew_C5b python bench.py --config C5 --steps 2 --warmup 3 --no-cpu --fused on > gpurun_out/ncu_skew.log 2>&1
