timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sweeps_coupled -c 1 -f -o gpurun_out/cps_full \
  python bench.py --no-cpu --steps 1 --warmup 3 --coupled 4000 > gpurun_out/cps_ncu.log 2>&1
