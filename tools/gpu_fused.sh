#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for c in C1x C3 C5; do :; done
for c in C3 C5; do
  python bench.py --steps 30 --warmup 5 --config $c --no-cpu > gpurun_out/fb_$c.json 2> gpurun_out/fb_$c.err
  python bench.py --steps 30 --warmup 5 --config $c --no-cpu --no-fused > gpurun_out/fbn_$c.json 2>> gpurun_out/fb_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_' -s 10 -c 12 --csv --log-file gpurun_out/launches_fused_C5.csv python bench.py --config C5 --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
