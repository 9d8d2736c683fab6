#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
run() { python bench.py --steps 10 --warmup 3 --config C5 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['ms_per_step'], d['value'])"; }
run default
NSM_FUSED_NST=1 run nst1
NSM_FUSED_GRID_DIV=2 run grid_half
NSM_FUSED_GRID_DIV=4 run grid_quarter
NSM_FUSED_NST=1 NSM_FUSED_GRID_DIV=2 run nst1_half
