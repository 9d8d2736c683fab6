#!/bin/bash
# Slice-geometry header (producer-staged) A/B: parity subset + bench C2..C5, two reps.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ilut.py -x -q -m gpu 2>&1 | tail -3 > gpurun_out/hdr_pytest.log
for rep in 1 2; do
  for c in C2 C3 C4 C5; do
    echo "== $c rep=$rep" >> gpurun_out/hdr.log
    timeout 300 python bench.py --config $c --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print(d['ms_per_step'], r['frac'], r.get('sweeps_frac'))" >> gpurun_out/hdr.log
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_residual' -s 10 -c 1 -o gpurun_out/prof_residual_C2_hdr python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1
