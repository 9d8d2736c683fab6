# per-pass sweeps with a forced stage count (1 stage: 3 CTAs/SM; 3+ stages: 1 CTA/SM) — is one CTA per SM
# with a deep pipeline as fast as three one-stage CTAs?  (libnsm_exp.so: build.py --variant exp -DNSM_EXPERIMENTS)
for nst in 1 2 3 4 5; do
  NSM_SWEEP_NST=$nst timeout 300 python bench.py --no-cpu --steps 20 --warmup 3 --coupled off --lib-variant exp 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('nst=$nst', d['ms_per_step'], 'sweeps_frac', d['roofline'].get('sweeps_frac'))"
done
