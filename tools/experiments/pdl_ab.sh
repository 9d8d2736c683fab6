# PDL on/off per configuration (the setup default: on up to 8 M rows), 2 reps each
for cfg in C2 C3 C4 C5; do for pdl in on off; do for r in 1 2; do
  timeout 300 python bench.py --no-cpu --steps 30 --warmup 3 --config $cfg --pdl $pdl 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg pdl=$pdl', d['ms_per_step'], 'res', r['frac'], 'sweeps', r.get('sweeps_frac'))"
done; done; done
