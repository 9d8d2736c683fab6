#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_host.py -q 2>&1 | tail -15 > gpurun_out/host_pytest.log
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 600 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_host.py -q > gpurun_out/host_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/host_memcheck.log
timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1
for c in C2 C3 C4 C5; do timeout 300 python bench.py --config $c --no-cpu > gpurun_out/host_bench_$c.json 2> gpurun_out/host_bench_$c.err; done
