# coupled sweeps (NSM_OPT_COUPLED): parity incl. full-size C3, bench A/B on C3
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "coupled or full_size_parity" 2>&1 | tail -4
for c in off on 1200; do
  timeout 300 python bench.py --no-cpu --steps 20 --warmup 3 --coupled $c 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('coupled=$c', d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline'].get('sweeps_frac'), d['detail']['kernels'][:60])"
done
