# windowed 27-point sweeps summed in chunks of 7 at four CTAs per SM (libnsm_sw7.so) vs CH = 16 at three
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "var27 and (tri_solves or pgs_smooth)" 2>&1 | tail -1
for r in 1 2 3; do for v in dflt sw7; do
  if [ $v = dflt ]; then LV=""; else LV="--lib-variant sw7"; fi
  timeout 300 python bench.py --no-cpu --steps 30 --warmup 3 $LV 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', d['ms_per_step'], 'res in-step', r['frac'], 'sweeps', r.get('sweeps_frac'))"
done; done
