#!/bin/bash
# Symmetric residual A/B: tests, then C3 bench lines with the
# transpose map on and off, twice,
# and ncu of the symmetric residual.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/bench_sym_all.jsonl
timeout 600 python -m pytest tests/test_gpu_symmetric.py -x -q > gpurun_out/sym_tests.log 2>&1
for rep in 1 2; do
  for v in "--sym on" "--sym off"; do
    timeout 600 python bench.py --no-cpu $v > gpurun_out/b.json 2>> gpurun_out/bench_sym.err
    python -c "import json,sys; d=json.load(open('gpurun_out/b.json')); d['ab']='$v'; print(json.dumps(d))" >> gpurun_out/bench_sym_all.jsonl
  done
done
if [ -z "$NONCU" ]; then
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_residual' -s 6 -c 1 -o gpurun_out/prof_residual_sym python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_sym.log 2>&1
fi
