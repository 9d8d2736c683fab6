#!/bin/bash
# A/B of a bench option on the given configs: CONFIGS="C3 C5" OPT="--window" VALUES="on off" REPS=2
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
: > gpurun_out/ab.txt
for c in ${CONFIGS:-C2 C3 C5}; do
  for rep in $(seq ${REPS:-2}); do
    for v in ${VALUES:-on off}; do
      r=$(timeout 600 python bench.py --config $c --steps ${STEPS:-30} --no-cpu ${OPT:---window} $v ${EXTRA} 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'], d['roofline']['frac'], d['roofline'].get('sweeps_frac'), d['roofline'].get('alone_frac'))")
      echo "$c ${OPT:---window}=$v rep$rep: ms/frac/sweeps/alone $r" >> gpurun_out/ab.txt
    done
  done
done
