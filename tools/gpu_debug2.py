import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from synth.configs import make_config
from oracle import oracle as O
import parity_util as U
for p in [4, 6, 8, 10]:
    cfg = make_config(1, p=p, n_off=300)
    S = cfg['surface']
    tg_ = (cfg['tx'], cfg['tnormal'], cfg['self_node'], cfg['side'])
    res = U.gpu_build(cfg, S, tg_)
    ptr_o, pat_o = O.near_list(S, cfg['tx'], cfg['self_node'], cfg['eta'])
    tgt, pat = O.pairs_from_ptr(ptr_o, pat_o)
    vals_o, sto = O.build_rows(S, *tg_, tgt, pat)
    out = [p, np.array_equal(ptr_o, res['ptr'])]
    for k in range(4):
        w, ratio = U.compare_rows(res['vals'][k], vals_o[k], tgt, S.n)
        out.append(round(w, 3))
        if w > 1:
            bad = np.argsort(ratio)[-3:]
            g = res['vals'][k][: tgt.size * S.n].reshape(-1, S.n)
            print('  k', k, 'bad pairs', bad, 'self', cfg['self_node'][tgt[bad]], 'patch', pat[bad], 'ratio', ratio[bad])
            print('  gpu', g[bad[-1], :6], '\n  orc', vals_o[k][bad[-1], :6])
    print(out, flush=True)
