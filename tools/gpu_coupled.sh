# coupled passes: parity, and one ncu --set full capture of the coupled kernel
# and of the per-pass residual (C3) for the shared-memory / stall comparison
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "coupled" 2>&1 | tail -4
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pgs_coupled -c 1 -f -o gpurun_out/cp_full \
  python bench.py --no-cpu --steps 1 --warmup 3 > gpurun_out/cp_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_residual_tma_w -c 1 -f -o gpurun_out/res_full \
  python bench.py --no-cpu --steps 1 --warmup 3 --coupled off > gpurun_out/res_ncu.log 2>&1
ls -la gpurun_out
