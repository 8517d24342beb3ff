import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import test_gpu_parity as T
from oracle import oracle as O
import parity_util as U
from synth.geometry import Surface
cfg, S, tgs, rng = T._sampled_config(2, 4000, 4000, 10)
raw = True
res = U.gpu_build(cfg, S, tgs, raw=raw)
ptr, pat = res["ptr"], res["pat"]
perm, Z = res['ctx'].debug_zeta(10**7)
inv = np.empty(perm.max() + 1, np.int64); inv[perm] = np.arange(perm.size)
tgt = np.repeat(np.arange(ptr.size - 1), np.diff(ptr))
n, p = S.n, S.p
npb = p * (p + 1) // 2
# self pairs
selfk = np.where((tgs[2][tgt] >= 0) & (tgs[2][tgt] // n == pat))[0]
sample = selfk[:: max(1, selfk.size // 30)]
rows = []
for k in sample:
    t, P = tgt[k], pat[k]
    sl = int(tgs[2][t] % n)
    d = O.pair_debug(S, P, tgs[0][t], tgs[1][t], self_local=sl, side=int(tgs[3][t]), raw=raw)
    W, dW, Th = d['W'], d['dW'], d['Theta']
    zW = np.concatenate([W[:, 0], -W[:, 1], -W[:, 2], -W[:, 3]])
    g = Z[inv[k]]
    eZ = np.abs(g[npb:5 * npb] - zW).max() / np.abs(zW).max()
    # oracle fit for this patch
    Ss = Surface(p=p, q=S.q, nodes=S.nodes[[P]], normals=S.normals[[P]], weights=S.weights[[P]], verts=S.verts[[P]],
                 edge_x=S.edge_x[[P]], edge_dx=S.edge_dx[[P]], uv=S.uv)
    fo, _ = O.patch_fit(Ss)
    PD = fo[0][:4 * npb]
    rD_or = d['rows'][1]
    rD_gpu = res['vals'][1][k * n:(k + 1) * n]
    rD_np_gZ = g[npb:5 * npb] @ PD
    rD_np_oZ = zW @ PD
    sc = np.abs(rD_or).max()
    rows.append((np.abs(rD_gpu - rD_or).max() / sc, eZ, np.abs(rD_np_gZ - rD_gpu).max() / sc,
                 np.abs(rD_np_oZ - rD_or).max() / sc, np.abs(PD).max(), sc, sl, d['Omega0']))
rows.sort(key=lambda r: -r[0])
for r in rows[:10]:
    print('rowerr %.2e Zerr %.2e |gZ.P - gpu| %.2e |oZ.P - orc| %.2e  |PD|max %.2e rowmax %.2e self %d Om0 %.4f' % r)
