#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ilut.py -m gpu -x -q -k "fused" 2>&1 | tail -3 > gpurun_out/pytest_skew.log
export NSM_DEBUG_FULL_RINGS=1
for cfg in C5 C2 C4; do
for B in 8; do
NSM_DEBUG_SKEW_B=$B timeout 300 python tools/skew_exp.py $cfg 0 2>&1 | grep cfg | sed "s/^/B=$B /"
done; done > gpurun_out/exp4.log
