# 7-point residual (CH = 4, offset-aligned / compact) at 4 CTAs per SM (56 registers, libnsm_r4.so) vs 3 (72)
for cfg in C5 C2 C4; do for r in 1 2; do for v in dflt r4; do
  if [ $v = dflt ]; then LV=""; else LV="--lib-variant r4"; fi
  timeout 300 python bench.py --no-cpu --steps 30 --warmup 3 --config $cfg $LV 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg $v', d['ms_per_step'], 'res in-step', r['frac'], 'alone', r.get('alone_frac'), 'sweeps', r.get('sweeps_frac'))"
done; done; done
