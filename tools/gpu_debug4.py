import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from synth.configs import make_config
from oracle import oracle as O
from paper_2411_08342_b200 import RRQ, DeviceSurface
for p in [4, 6, 8, 10]:
    cfg = make_config(1, p=p, n_off=10)
    S = cfg['surface']
    ctx = RRQ(p, eta=1.0)
    ds = DeviceSurface.from_numpy(S)
    fit, st = ctx.patch_fit(ds)
    torch.cuda.synchronize()
    stride = ctx.fit_bytes(1) // 8
    g = fit.view(S.n_patches, stride).cpu().numpy()
    n, npb, E, Q = p * p, p * (p + 1) // 2, 6 * p, 2 * p
    off = 32 + 6 * E + 9 * Q
    fo, sto = O.patch_fit(S)
    for P in [0, 7]:
        gb = g[P, off:off + 13 * npb * n].reshape(13 * npb, n)
        names = [('PD', 0, 4 * npb), ('PSp', 4 * npb, 8 * npb), ('PSd', 8 * npb, 9 * npb), ('PSg', 9 * npb, 13 * npb)]
        print(p, P, 'status', int(st[P]), sto[P], ' '.join('%s %.2e' % (nm, np.abs(gb[a:b] - fo[P][a:b]).max() / np.abs(fo[P][a:b]).max()) for nm, a, b in names))
