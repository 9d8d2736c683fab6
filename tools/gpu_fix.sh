#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL='(lap_aligned_ragged or var27_aligned_40) and pipelined'
timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "$SEL" > gpurun_out/san4_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san4_memcheck.log
timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_ilut.py tests/test_gpu_parity.py -m gpu -q -k "aligned or ilut" > gpurun_out/san4b_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san4b_memcheck.log
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 > gpurun_out/fix_pytest.log
rm -f gpurun_out/ab.log
bash tools/gpu_ab.sh default
