#!/bin/bash
# compute-sanitizer on the kernels added in round 2: windowed pipelined kernels,
# the one-pass windowed pGS, the device builder, the device all-reduce.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "var27_aligned_40 and (pipelined or onepass) and (residual or pgs_smooth or onepass)" > gpurun_out/san_r02_win.log 2>&1; echo "memcheck windows rc=$?" >> gpurun_out/san_r02_win.log
timeout 1200 $CS --tool racecheck --racecheck-report analysis --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "var27_aligned_40 and pipelined and pgs_smooth" > gpurun_out/san_r02_race.log 2>&1; echo "racecheck windows rc=$?" >> gpurun_out/san_r02_race.log
timeout 1200 $CS --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "onepass_windowed and var27_ragged" > gpurun_out/san_r02_sync.log 2>&1; echo "synccheck onepass rc=$?" >> gpurun_out/san_r02_sync.log
timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_builder.py -m gpu -q -x -k "not full_size" > gpurun_out/san_r02_builder.log 2>&1; echo "memcheck builder rc=$?" >> gpurun_out/san_r02_builder.log
timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_dist_solver.py -m gpu -q -x -k "allreduce or vcycle" > gpurun_out/san_r02_comm.log 2>&1; echo "memcheck comm rc=$?" >> gpurun_out/san_r02_comm.log
