import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from oracle import oracle as O
import parity_util as U
from synth.configs import make_config
cfg = make_config(5, n_off=3000)
S = cfg["surface"]
tgs = (cfg["tx"], cfg["tnormal"], cfg["self_node"], cfg["side"])
res = U.gpu_build(cfg, S, tgs)
perm, Z = res['ctx'].debug_zeta(10**7)
inv = np.empty(perm.max() + 1, np.int64); inv[perm] = np.arange(perm.size)
Tn = cfg["tx"].shape[0]; n = S.n; p = S.p; npb = p*(p+1)//2
tg = np.arange(Tn, dtype=np.int64); pa = np.zeros(Tn, np.int32)
vo, sto, kap = O.build_rows(S, *tgs, tg, pa, kappa=True)
k = 1
g = res["vals"][k][:Tn * n].reshape(Tn, n)
rowmax = np.abs(vo[k]).max(1)
tol = np.maximum(np.maximum(1e-11 * rowmax[:, None], 1e-13), 1e-11 * kap[k])
ratio = (np.abs(g - vo[k]) / tol).max(1)
bad = np.argsort(ratio)[-6:]
for b in list(bad) + list(np.random.default_rng(0).choice(Tn, 4)):
    d = O.pair_debug(S, 0, cfg["tx"][b], cfg["tnormal"][b], side=int(cfg["side"][b]))
    W = d['W']; zo = np.concatenate([d['Theta'], W[:, 0], -W[:, 1], -W[:, 2], -W[:, 3]])
    zg = Z[inv[b]][:5 * npb]
    e = np.abs(zg - zo)
    print('ratio %.2f' % ratio[b], 'zeta err/max %.2e' % (e.max() / np.abs(zo).max()),
          'argmax comp', np.argmax(e), 'Om0 %.4e' % d['Omega0'], 'swap', d['swap'],
          'Om0 gpu-vs-orc?')
