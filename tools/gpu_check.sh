#!/bin/bash
# Final check: full GPU suite, smoke(), the default bench line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/check_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/check_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/check_bench.json 2> gpurun_out/check_bench.err
