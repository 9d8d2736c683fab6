#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL='lap3d_ragged or random_irregular'
timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "($SEL) and (smooth or tri_solves)" > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_memcheck.log
timeout 900 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_chow_patel.py -m gpu -q -x -k "not full_size" > gpurun_out/san_cp.log 2>&1; echo "memcheck cp rc=$?" >> gpurun_out/san_cp.log
timeout 1200 $CS --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "lap3d_ragged and fused and pgs_smooth" > gpurun_out/san_sync.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/san_sync.log
