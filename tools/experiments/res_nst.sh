# 7-point residual stage count (NSM_RES_NST, libnsm_exp.so): the default geometry picks 4 stages at 3 CTAs/SM
# (225 KB shared memory, ~30 KB of L1 left for the x gathers); fewer stages leave more L1
for cfg in C2 C5; do for nst in dflt 1 2 3; do
  if [ $nst = dflt ]; then unset NSM_RES_NST; else export NSM_RES_NST=$nst; fi
  timeout 300 python bench.py --no-cpu --steps 30 --warmup 3 --config $cfg --lib-variant exp 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg nst=$nst', d['ms_per_step'], 'res in-step', r['frac'], 'alone', r.get('alone_frac'))"
done; done
