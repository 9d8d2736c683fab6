#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export NSM_DEBUG_FULL_RINGS=1
for cfg in C5 C2; do
for pm in 4 2 1; do
for nst in 2 4; do
NSM_DEBUG_SKEW_PERSM=$pm NSM_DEBUG_SKEW_NST=$nst timeout 300 python tools/skew_exp.py $cfg 0,150,300,600,1000,2000,100000 2>&1 | grep cfg
done; done; done > gpurun_out/exp2.log
