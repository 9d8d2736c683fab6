# coupled sweeps V4 (no publisher warp, chunk-7 sums, 56 registers, four CTAs per SM: two per sweep; libnsm_v4.so)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "coupled" 2>&1 | tail -1
NSM_LIBVARIANT=v4 true
for r in 1 2; do for v in dflt v4; do
  if [ $v = dflt ]; then LV=""; else LV="--lib-variant v4"; fi
  for c in off on; do
  timeout 300 python bench.py --no-cpu --steps 20 --warmup 3 --coupled $c $LV 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v coupled=$c', d['ms_per_step'], 'res', r['frac'], 'sweeps', r.get('sweeps_frac'))"
  done
done; done
