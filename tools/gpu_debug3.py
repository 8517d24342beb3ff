import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from synth.configs import make_config
from oracle import oracle as O
import parity_util as U
p = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cfg = make_config(1, p=p, n_off=40)
S = cfg['surface']
n, npb = S.n, p * (p + 1) // 2
tg_ = (cfg['tx'], cfg['tnormal'], cfg['self_node'], cfg['side'])
res = U.gpu_build(cfg, S, tg_)
perm, Z = res['ctx'].debug_zeta(100000)
ptr, pat = res['ptr'], res['pat']
tgt = np.repeat(np.arange(ptr.size - 1), np.diff(ptr))
worst = []
for i in range(0, len(perm), max(1, len(perm) // 40)):
    k = perm[i]; t = tgt[k]; P = pat[k]
    sl = int(cfg['self_node'][t] % n) if cfg['self_node'][t] >= 0 and cfg['self_node'][t] // n == P else -1
    d = O.pair_debug(S, P, cfg['tx'][t], cfg['tnormal'][t], self_local=sl, side=int(cfg['side'][t]))
    W, dW, Th = d['W'], d['dW'], d['Theta']
    zW = np.concatenate([W[:, 0], -W[:, 1], -W[:, 2], -W[:, 3]])
    zdW = np.concatenate([dW[:, 0], -dW[:, 1], -dW[:, 2], -dW[:, 3]])
    g = Z[i]
    eT = np.abs(g[:npb] - Th).max() / max(1e-300, np.abs(Th).max())
    eW = np.abs(g[npb:5 * npb] - zW).max() / np.abs(zW).max()
    edW = np.abs(g[5 * npb:9 * npb] - zdW).max() / np.abs(zdW).max()
    worst.append((eW, edW, eT, k, t, P, d['swap'], d['conv']))
worst.sort(key=lambda r: -r[0])
for w in worst[:8]:
    print('eW %.2e edW %.2e eTh %.2e pair %d t %d P %d swap %s conv %s' % w)
# per (l,m) error profile for the worst
k = worst[0][3]; i = int(np.where(perm == k)[0][0]); t = tgt[k]; P = pat[k]
d = O.pair_debug(S, P, cfg['tx'][t], cfg['tnormal'][t], side=int(cfg['side'][t]))
print('Omega0', d['Omega0'], 't0', d['t0'])
W = d['W']
gW = Z[i][npb:5 * npb].reshape(4, npb)
for l in range(1, p + 1):
    idx = [l * (l - 1) // 2 + m - 1 for m in range(1, l + 1)]
    print(l, np.abs(gW[0, idx] - W[idx, 0]).max(), np.abs(W[idx, 0]).max())
