#!/bin/bash
# PDL on/off A/B on the 16.7 M-row configs (the library's default is off above 8 M rows).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/pdl.log
for rep in 1 2; do for p in auto on; do for c in C3 C4 C5; do
  printf "pdl=%-4s %s rep=%s  " $p $c $rep >> gpurun_out/pdl.log
  timeout 300 python bench.py --config $c --no-cpu --pdl $p 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print(d['ms_per_step'], r['frac'], r.get('sweeps_frac'))" >> gpurun_out/pdl.log
done; done; done
