#!/bin/bash
# Quick GPU check: selected tests (args: pytest -k expression or file list via TESTS), then the default bench.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest ${TESTS:-tests} -m gpu -x -q ${K:+-k "$K"} 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
if [ -z "$NOBENCH" ]; then
  timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
fi
