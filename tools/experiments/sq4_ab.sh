# 7-point residual with one triangle at a time (CH = 4) at 4 CTAs per SM (libnsm_sq4.so) vs both in flight at 3
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "lap and residual" 2>&1 | tail -1
for cfg in C5 C2; do for r in 1 2; do for v in dflt sq4; do
  if [ $v = dflt ]; then LV=""; else LV="--lib-variant sq4"; fi
  timeout 300 python bench.py --no-cpu --steps 30 --warmup 3 --config $cfg $LV 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg $v', d['ms_per_step'], 'res in-step', r['frac'], 'alone', r.get('alone_frac'), 'sweeps', r.get('sweeps_frac'))"
done; done; done
