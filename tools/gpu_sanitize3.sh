#!/bin/bash
# compute-sanitizer on the offset-aligned pipelined kernels (staged offsets + slice header).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL='(lap_aligned_ragged or var27_aligned_40) and pipelined'
timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$SEL" > gpurun_out/san3_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san3_memcheck.log
timeout 1200 $CS --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$SEL and (smooth or residual)" > gpurun_out/san3_sync.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/san3_sync.log
timeout 1500 $CS --tool racecheck --racecheck-report analysis --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "lap_aligned_ragged and pipelined and (residual or pgs_smooth)" > gpurun_out/san3_race.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/san3_race.log
