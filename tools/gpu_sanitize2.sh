#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_solver.py -m gpu -q -x -k "not solve_timing" > gpurun_out/san_solver.log 2>&1; echo "memcheck solver rc=$?" >> gpurun_out/san_solver.log
timeout 1500 $CS --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_solver.py -m gpu -q -x -k "vcycle or workspace" > gpurun_out/san_solver_sync.log 2>&1; echo "synccheck solver rc=$?" >> gpurun_out/san_solver_sync.log
timeout 1500 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "random_irregular and (smooth or residual)" > gpurun_out/san_wide.log 2>&1; echo "memcheck wide rc=$?" >> gpurun_out/san_wide.log
