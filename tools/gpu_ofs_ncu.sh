#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in "" ofs; do
NSM_LIB_VARIANT=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_residual -s 3 -c 1 -o gpurun_out/prof_c3res_$v python bench.py --config C3 --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_ofs_$v.log 2>&1
done
