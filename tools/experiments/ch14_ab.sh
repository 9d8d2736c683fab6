# windowed 27-point kernels: the residual at CH = 14 (3 CTAs/SM, default) with the sweeps at CH = 16 (3 CTAs/SM,
# default) or CH = 14 (4 CTAs/SM, libnsm_sw14.so)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "var27 or full_size_parity" 2>&1 | tail -1
for r in 1 2 3; do for v in dflt sw14; do
  if [ $v = dflt ]; then LV=""; else LV="--lib-variant sw14"; fi
  timeout 300 python bench.py --no-cpu --steps 30 --warmup 3 $LV 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', d['ms_per_step'], 'res in-step', r['frac'], 'alone', r.get('alone_frac'), 'sweeps', r.get('sweeps_frac'))"
done; done
