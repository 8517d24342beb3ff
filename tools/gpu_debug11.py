import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import test_gpu_parity as T
from oracle import oracle as O
import parity_util as U
cfg, S, tgs, rng = T._sampled_config(2, 3000, 3000, 0)
res = U.gpu_build(cfg, S, tgs)
perm, Z = res["ctx"].debug_zeta(10 ** 8)
inv = np.empty(perm.max() + 1, np.int64); inv[perm] = np.arange(perm.size)
ptr, pat = res["ptr"], res["pat"]
tgt = np.repeat(np.arange(ptr.size - 1), np.diff(ptr))
n, p = S.n, S.p; npb = p * (p + 1) // 2
rows = []
for k in rng.choice(perm, 150, replace=False):
    t, P = tgt[k], pat[k]
    sl = int(tgs[2][t] % n) if tgs[2][t] >= 0 and tgs[2][t] // n == P else -1
    d = O.pair_debug(S, P, tgs[0][t], tgs[1][t], self_local=sl, side=int(tgs[3][t]))
    W, dW, Th = d["W"], d["dW"], d["Theta"]
    for nm, a, b, ref in [("Th", 0, npb, Th), ("W", npb, 5 * npb, np.concatenate([W[:, 0], -W[:, 1], -W[:, 2], -W[:, 3]])),
                          ("dW", 5 * npb, 9 * npb, np.concatenate([dW[:, 0], -dW[:, 1], -dW[:, 2], -dW[:, 3]]))]:
        e = np.abs(Z[inv[k]][a:b] - ref)
        j = int(np.argmax(e)); bb, c = divmod(j, npb) if nm != "Th" else (0, j)
        rows.append((e.max() / np.abs(ref).max(), nm, bb, c, sl, str(d['swap']), min(abs(z.imag) for z in d['t0']),
                     np.linalg.norm(tgs[0][t] - S.nodes[P].mean(0)) / 0.05, d['dOmega0'], np.abs(d['dOmega']).max()))
rows.sort(key=lambda r: -r[0])
for r in rows[:10]:
    print('%.2e %s comp %d lm %d self %d swap %s min|Imt0| %.2e dist~%.2f dOm0 %.3e |dOm| %.3e' % r)
