#!/bin/bash
# quick loop: gpu tests + bench (+ optional ncu launch list)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-C2}; do
  python bench.py --steps 30 --warmup 5 --config $c --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
if [ -n "$NCU" ]; then
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_' -s 20 -c 30 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu > gpurun_out/ncu_bench.log 2>&1
fi
