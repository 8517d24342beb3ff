import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import test_gpu_parity as T
from oracle import oracle as O
import parity_util as U
cfg, S, tgs, rng = T._sampled_config(2, 4000, 4000, 10)
res = U.gpu_build(cfg, S, tgs)
ptr, pat = res["ptr"], res["pat"]
perm, Z = res['ctx'].debug_zeta(10**8)
inv = np.empty(perm.max() + 1, np.int64); inv[perm] = np.arange(perm.size)
tgt = np.repeat(np.arange(ptr.size - 1), np.diff(ptr))
n, p = S.n, S.p
npb = p * (p + 1) // 2
rows = []
ks = rng.choice(perm.size, 400, replace=False)
for k in perm[ks]:
    t, P = tgt[k], pat[k]
    sl = int(tgs[2][t] % n) if tgs[2][t] >= 0 and tgs[2][t] // n == P else -1
    d = O.pair_debug(S, P, tgs[0][t], tgs[1][t], self_local=sl, side=int(tgs[3][t]))
    W, dW, Th = d['W'], d['dW'], d['Theta']
    zo = np.concatenate([Th, W[:, 0], -W[:, 1], -W[:, 2], -W[:, 3], dW[:, 0], -dW[:, 1], -dW[:, 2], -dW[:, 3]])
    g = Z[inv[k]][:9 * npb]
    e = np.abs(g - zo)
    rows.append((e[:npb].max() / np.abs(Th).max(), e[npb:5*npb].max() / np.abs(zo[npb:5*npb]).max(),
                 e[5*npb:].max() / np.abs(zo[5*npb:]).max(), sl, str(d['swap']), str(d['conv']),
                 min(abs(x.imag) for x in d['t0']), d['Omega0']))
rows.sort(key=lambda r: -max(r[0], r[1], r[2]))
for r in rows[:12]:
    print('eTh %.2e eW %.2e edW %.2e self %d swap %s conv %s min|Im t0| %.2e Om0 %.3f' % r)
print('median', np.median([max(r[0], r[1], r[2]) for r in rows]))
