#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --same-device --no-cpu > gpurun_out/bench_2same.json 2> gpurun_out/bench_2same.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_' -s 20 -c 24 --csv --log-file gpurun_out/launches_C3.csv python bench.py --config C3 --steps 4 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_' -s 20 -c 24 --csv --log-file gpurun_out/launches_C5.csv python bench.py --config C5 --steps 4 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_residual_tma -s 3 -c 1 -o gpurun_out/prof_res_tma_C5 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_tma -s 6 -c 2 -o gpurun_out/prof_sweep_tma_C3 python bench.py --config C3 --steps 2 --warmup 3 --no-cpu >> gpurun_out/ncu_full.log 2>&1
