timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_host.py tests/test_gpu_ilut.py -x -q 2>&1 | tail -1
for r in 1 2; do timeout 300 python bench.py --no-cpu --steps 30 --warmup 3 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('C3', d['ms_per_step'], 'res in-step', r['frac'], 'sweeps', r.get('sweeps_frac'), 'e2e', d['e2e']['value'])"; done
