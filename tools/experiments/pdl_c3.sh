for r in 1 2 3; do for pdl in auto on; do
  timeout 300 python bench.py --no-cpu --steps 30 --warmup 3 --pdl $pdl 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('C3 pdl=$pdl', d['ms_per_step'], 'res', r['frac'], 'sweeps', r.get('sweeps_frac'))"
done; done
