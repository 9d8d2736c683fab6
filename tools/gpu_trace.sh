#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
NSM_DEBUG_SKEW_TRACE=1 timeout 300 python tools/skew_exp_once.py C5 0 > gpurun_out/trace_C5.log 2>&1
NSM_DEBUG_SKEW_TRACE=1 NSM_DEBUG_FULL_RINGS=1 timeout 300 python tools/skew_exp_once.py C5 65280 > gpurun_out/trace_C5_w.log 2>&1
