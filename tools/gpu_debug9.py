import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import test_gpu_parity as T
from oracle import oracle as O
import parity_util as U
from synth.configs import make_config
cfg = make_config(5, n_off=3000)
S = cfg["surface"]
tgs = (cfg["tx"], cfg["tnormal"], cfg["self_node"], cfg["side"])
res = U.gpu_build(cfg, S, tgs)
Tn = cfg["tx"].shape[0]
tg = np.arange(Tn, dtype=np.int64); pa = np.zeros(Tn, np.int32)
vo, sto, kap = O.build_rows(S, *tgs, tg, pa, kappa=True)
n = S.n
delta = T._edge_distance(S, cfg["tx"], 0)
hn = np.abs(np.linalg.norm(cfg["tx"], axis=1) - 1) / 0.2
for k in [1, 3]:
    g = res["vals"][k][:Tn * n].reshape(Tn, n)
    rowmax = np.abs(vo[k]).max(1)
    tol = np.maximum(np.maximum(1e-11 * rowmax[:, None], 1e-13), 1e-11 * kap[k])
    ratio = (np.abs(g - vo[k]) / tol).max(1)
    bad = np.argsort(ratio)[-8:]
    for b in bad:
        d = O.pair_debug(S, 0, cfg["tx"][b], cfg["tnormal"][b], side=int(cfg["side"][b]))
        print('k', k, 'ratio %.2f' % ratio[b], 'normal dist/h %.2e' % hn[b], 'edge dist/h %.2e' % delta[b],
              'swap', d['swap'], 't0', ['%.3f%+.2ei' % (z.real, z.imag) for z in d['t0']])
