import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import test_gpu_parity as T
from oracle import oracle as O
import parity_util as U
from synth.configs import make_config
def run(cfg, S, tgs, tg, pa, pos, res):
    vo, sto, kap = O.build_rows(S, *tgs, tg, pa, kappa=True)
    n = S.n
    for k in range(4):
        g = np.stack([res["vals"][k][pp * n:(pp + 1) * n] for pp in pos])
        err = np.abs(g - vo[k])
        rowmax = np.abs(vo[k]).max(1, keepdims=True)
        ratio_k = err / kap[k]
        print('kernel', k, 'max err/kappa %.3g' % ratio_k.max(), ' median %.3g' % np.median(ratio_k),
              ' max kappa/rowmax %.3g' % (kap[k] / rowmax).max(), ' max err/rowmax %.3g' % (err / rowmax).max())
cfg, S, tgs, rng = T._sampled_config(2, 4000, 4000, 10)
res = U.gpu_build(cfg, S, tgs)
ptr, pat = res["ptr"], res["pat"]
patches = rng.choice(np.unique(pat), size=10, replace=False)
tg, pa = O.near_pairs_for_patches(S, tgs[0], tgs[2], cfg["eta"], patches)
pos = T._gpu_rows_of(ptr, pat, tg, pa)
print('cfg2'); run(cfg, S, tgs, tg, pa, pos, res)
for p in [8, 10]:
    cfg = make_config(1, p=p, n_off=300); S = cfg['surface']
    tgs = (cfg['tx'], cfg['tnormal'], cfg['self_node'], cfg['side'])
    res = U.gpu_build(cfg, S, tgs)
    tg, pa = O.pairs_from_ptr(res['ptr'], res['pat'])
    print('cfg1 p', p); run(cfg, S, tgs, tg, pa, np.arange(tg.size), res)
