#!/bin/bash
# fused-pass iteration: parity tests, then bench fused vs per-pass on C2/C5 (and optional more)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ilut.py -m gpu -x -q ${PYTEST_EXTRA} 2>&1 | tail -25 > gpurun_out/pytest_skew.log
for c in ${CONFIGS:-C2 C5}; do
  for f in on off; do
    timeout 300 python bench.py --steps 20 --warmup 5 --config $c --no-cpu --fused $f > gpurun_out/bench_${c}_$f.json 2> gpurun_out/bench_${c}_$f.err
  done
done
