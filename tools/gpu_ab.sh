#!/bin/bash
# A/B of library variants (build.py --variant) on one box: bench C2..C5, two reps, with clocks.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for rep in 1 2; do
for v in "$@"; do
  [ "$v" = default ] && v=""
  for c in C2 C3 C4 C5; do
    printf "v=%-8s %s rep=%s  " "$v" $c $rep >> gpurun_out/ab.log
    NSM_LIB_VARIANT=$v timeout 300 python bench.py --config $c --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print(d['ms_per_step'], r['frac'], r.get('sweeps_frac'), d['clocks']['sm_mhz'])" >> gpurun_out/ab.log
  done
done
done
