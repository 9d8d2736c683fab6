# 7-point matrices with gather windows forced (NSM_WINDOW_ALWAYS, libnsm_exp.so) vs without (the default rule)
timeout 600 python -c "
import os; os.environ['NSM_WINDOW_ALWAYS']='1'
import numpy as np, torch, inputs, oracle, paper_2112_14681_b200 as nsm
nsm.load(variant='exp')
A = inputs.laplace(100, 9, 3); b, x0 = inputs.uniform(0, A.nrows), inputs.uniform(1, A.nrows)
with nsm.Smoother(A, oracle.ilu0(A)[2]) as S:
    print('windows', S.windows())
    x = torch.from_numpy(x0.copy()).cuda(); S.smooth(torch.from_numpy(b).cuda(), x, 'pgs', k_l=2)
    print('pgs bitwise', np.array_equal(x.cpu().numpy(), oracle.pgs_apply(A, b, x0, 2)))
    x = torch.from_numpy(x0.copy()).cuda(); S.smooth(torch.from_numpy(b).cuda(), x, 'ilu', k_l=2, k_u=2)
    print('ilu bitwise', np.array_equal(x.cpu().numpy(), oracle.ilu_apply(A, oracle.ilu0(A), b, x0, 2, 2)))
"
for cfg in C5 C2; do for r in 1 2; do for v in dflt win; do
  if [ $v = dflt ]; then unset NSM_WINDOW_ALWAYS; else export NSM_WINDOW_ALWAYS=1; fi
  timeout 300 python bench.py --no-cpu --steps 30 --warmup 3 --config $cfg --lib-variant exp 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg $v', d['ms_per_step'], 'res in-step', r['frac'], 'alone', r.get('alone_frac'), 'sweeps', r.get('sweeps_frac'))"
done; done; done
