import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from synth.configs import make_config
from oracle import oracle as O
import parity_util as U
cfg = make_config(1)
S = cfg['surface']
tg = (cfg['tx'], cfg['tnormal'], cfg['self_node'], cfg['side'])
t = time.time()
res = U.gpu_build(cfg, S, tg)
print('gpu build', time.time() - t, 'pairs', res['pat'].shape, flush=True)
ptr_o, pat_o = O.near_list(S, cfg['tx'], cfg['self_node'], cfg['eta'])
print('near list equal:', np.array_equal(ptr_o, res['ptr']), np.array_equal(pat_o, res['pat']))
tgt, pat = O.pairs_from_ptr(ptr_o, pat_o)
fit_o, st_o = O.patch_fit(S)
print('fit status', st_o.max(), res['fit_status'].max())
vals_o, sto = O.build_rows(S, cfg['tx'], cfg['tnormal'], cfg['self_node'], cfg['side'], tgt, pat)
print('status gpu', np.bincount(res['status']), 'oracle', np.bincount(sto))
for k in range(4):
    w, ratio = U.compare_rows(res['vals'][k], vals_o[k], tgt, S.n)
    bad = np.argsort(ratio)[-3:]
    print('kernel', k, 'worst ratio', w, 'worst pairs', bad, ratio[bad])
