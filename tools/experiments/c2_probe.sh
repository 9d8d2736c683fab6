bash tools/experiments/pdl_ab.sh > gpurun_out/pdl.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_residual_tma|k_sweep_tma" -c 5 -f -o gpurun_out/c2_full \
  python bench.py --no-cpu --steps 1 --warmup 3 --config C2 > gpurun_out/c2_ncu.log 2>&1
