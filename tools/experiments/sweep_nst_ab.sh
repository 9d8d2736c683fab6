# per-pass sweeps: default geometry (most resident consumer warps: 3 CTAs x 1 stage on C3) vs 2 stages x 2 CTAs
for cfg in C3 C5 C4; do for r in 1 2 3; do for v in dflt 2; do
  if [ $v = dflt ]; then unset NSM_SWEEP_NST; else export NSM_SWEEP_NST=$v; fi
  timeout 300 python bench.py --no-cpu --steps 30 --warmup 3 --config $cfg --lib-variant exp 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg nst=$v', d['ms_per_step'], 'res', r['frac'], 'sweeps', r.get('sweeps_frac'))"
done; done; done
