#!/bin/bash
# A/B: 4 CTAs/SM register budget for the CH=4 offset-aligned kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for rep in 1 2; do
for v in "" o4all o4sw; do
  for c in C2 C3 C4 C5; do
    echo "== v=$v $c rep=$rep" >> gpurun_out/ofs4.log
    NSM_LIB_VARIANT=$v timeout 300 python bench.py --config $c --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'], d['roofline']['frac'])" >> gpurun_out/ofs4.log
  done
done
done
