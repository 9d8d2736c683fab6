#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export NSM_DEBUG_FULL_RINGS=1
for v in "" seq3 seq2; do
for cfg in C5 C2; do
NSM_LIB_VARIANT=$v timeout 300 python tools/skew_exp.py $cfg 0 2>&1 | grep cfg | sed "s/^/v=$v /"
done; done > gpurun_out/exp5.log
