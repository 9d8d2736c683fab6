#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in ""; do
for c in C2 C5 C4; do
NSM_LIB_VARIANT=$v timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('v=$v', '$c', d['ms_per_step'], d['config']['frac_of_hbm_peak'], r['frac'], r.get('sweeps_frac'))"
done; done > gpurun_out/tma4.log 2>&1
