#!/bin/bash
# Round measurement: tests, smoke, bench lines for every config (default = C3),
# the reference arm, ncu launch lists of the default bench command (C3) and of
# C4, and full captures of the C3 / C4 residual kernels (DRAM traffic).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
if [ -z "$NOTESTS" ]; then
  NSM_SOLVE_N=64 NSM_SOLVE_N4=48 timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
fi
timeout 900 python bench.py > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
for c in C2 C4 C5; do
  timeout 600 python bench.py --config $c --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --coupled on --no-cpu > gpurun_out/bench_C3_coupled.json 2> gpurun_out/bench_C3_coupled.err
timeout 300 python tools/pcie_probe.py > gpurun_out/pcie.txt 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -c 400 --csv --log-file gpurun_out/launches_C3.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:'k_' -c 60 --csv --log-file gpurun_out/launches_C4.csv python bench.py --config C4 --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_residual' -s 6 -c 1 -o gpurun_out/prof_residual_C3 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_sweep' -s 10 -c 1 -o gpurun_out/prof_sweep_C3 python bench.py --steps 2 --warmup 3 --no-cpu >> gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_residual' -s 6 -c 1 -o gpurun_out/prof_residual_C4 python bench.py --config C4 --steps 2 --warmup 3 --no-cpu >> gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_sweeps_coupled' -c 1 -o gpurun_out/prof_coupled_C3 python bench.py --steps 2 --warmup 3 --no-cpu --coupled on >> gpurun_out/ncu_full.log 2>&1
