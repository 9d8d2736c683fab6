# split residual (L step / U step as separate stages) vs the whole-tile windowed residual, C3 (and C2/C5 unaffected)
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "var27 and (residual or pgs_smooth)" 2>&1 | tail -2
for r in 1 2; do
for v in split nosplit; do
  if [ $v = nosplit ]; then export NSM_NO_SPLIT_RESIDUAL=1; else unset NSM_NO_SPLIT_RESIDUAL; fi
  timeout 300 python bench.py --no-cpu --steps 30 --warmup 3 --lib-variant exp 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', d['ms_per_step'], 'res in-step', r['frac'], r['ms_per_launch'], 'alone', r.get('alone_frac'), 'sweeps', r.get('sweeps_frac'))"
done; done
