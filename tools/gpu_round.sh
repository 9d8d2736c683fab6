#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + one full capture.
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py --steps 30 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_' -s 20 -c 30 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu > gpurun_out/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_residual' -s 10 -c 1 -o gpurun_out/prof_residual python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_sweep' -s 20 -c 1 -o gpurun_out/prof_sweep python bench.py --steps 2 --warmup 3 --no-cpu >> gpurun_out/ncu_full.log 2>&1
