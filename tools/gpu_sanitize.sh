#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL='lap3d_ragged or random_irregular'
timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "($SEL) and (smooth or tri_solves)" > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_memcheck.log
timeout 900 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_chow_patel.py -m gpu -q -x -k "not full_size" > gpurun_out/san_cp.log 2>&1; echo "memcheck cp rc=$?" >> gpurun_out/san_cp.log
timeout 1200 $CS --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "lap3d_ragged and fused and pgs_smooth" > gpurun_out/san_sync.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/san_sync.log
# solver layer and the offset-aligned pipelined kernels
timeout 1500 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_solver.py -m gpu -q -x -k "not solve_timing" > gpurun_out/san_solver.log 2>&1; echo "memcheck solver rc=$?" >> gpurun_out/san_solver.log
timeout 1500 $CS --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_solver.py -m gpu -q -x -k "vcycle or workspace" > gpurun_out/san_solver_sync.log 2>&1; echo "synccheck solver rc=$?" >> gpurun_out/san_solver_sync.log
timeout 1500 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "random_irregular and (smooth or residual)" > gpurun_out/san_wide.log 2>&1; echo "memcheck wide rc=$?" >> gpurun_out/san_wide.log
SEL='(lap_aligned_ragged or var27_aligned_40) and pipelined'
timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$SEL" > gpurun_out/san3_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san3_memcheck.log
timeout 1200 $CS --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$SEL and (smooth or residual)" > gpurun_out/san3_sync.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/san3_sync.log
timeout 1500 $CS --tool racecheck --racecheck-report analysis --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "lap_aligned_ragged and pipelined and (residual or pgs_smooth)" > gpurun_out/san3_race.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/san3_race.log
