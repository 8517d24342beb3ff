import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import test_gpu_parity as T
from oracle import oracle as O
import parity_util as U
cfg, S, tgs, rng = T._sampled_config(2, 4000, 4000, 10)
res = U.gpu_build(cfg, S, tgs)
ptr, pat = res["ptr"], res["pat"]
patches = rng.choice(np.unique(pat), size=10, replace=False)
tg, pa = O.near_pairs_for_patches(S, tgs[0], tgs[2], cfg["eta"], patches)
pos = T._gpu_rows_of(ptr, pat, tg, pa)
vo, sto = O.build_rows(S, *tgs, tg, pa)
band = T._band_for_pairs(S, tgs[0], tg, pa)
n = S.n
for k in range(4):
    g = np.stack([res["vals"][k][pp * n:(pp + 1) * n] for pp in pos])
    err = np.abs(g - vo[k]).max(1) / np.maximum(np.abs(vo[k]).max(1), 1e-300)
    bad = np.argsort(err)[-5:]
    print('kernel', k, 'worst rel err (pair-row)', err[bad], 'band', band[bad], 'self', tgs[2][tg[bad]])
print('worst (row-relative, banded):', T._compare(res["vals"], vo, pos, tg, n, band))
