"""Localise a high-order (p >= 12) GPU/oracle disagreement: fit operators, then the contraction vectors zeta
(Theta | W | dW blocks), then the rows, on the small sphere of tests/test_gpu_highorder.py."""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from synth.configs import make_config
from synth.geometry import Surface
from oracle import oracle as O
import parity_util as U

for p in [int(a) for a in sys.argv[1:]] or [10, 12]:
    cfg = make_config(2, n_off=300, freq=2, p=p)
    S = cfg["surface"]
    keep = np.concatenate([np.arange(0, S.n_patches * S.n, 11), np.arange(S.n_patches * S.n, cfg["tx"].shape[0])])
    tgs = (cfg["tx"][keep], cfg["tnormal"][keep], cfg["self_node"][keep], cfg["side"][keep])
    res = U.gpu_build(cfg, S, tgs)
    print(f"p = {p}: fit status max {int(res['fit_status'].max())}, pair status max {int(res['status'].max())}, pairs {res['pat'].size}")
    n, npb = S.n, p * (p + 1) // 2
    stride = res["ctx"].fit_bytes(1) // 8
    g = res["fit"].view(S.n_patches, stride).cpu().numpy()
    E, Q = 6 * p, 2 * p
    off = 32 + 6 * E + 9 * Q
    nf = n + ((4 - n % 16) + 16) % 16
    two = np.array([0, 1])
    Ssub = Surface(p=p, q=S.q, nodes=S.nodes[two], normals=S.normals[two], weights=S.weights[two],
                   verts=S.verts[two], edge_x=S.edge_x[two], edge_dx=S.edge_dx[two], uv=S.uv)
    fo, _ = O.patch_fit(Ssub, prec="d")
    for i, P in enumerate(two):
        gb = g[P, off:off + 13 * npb * nf].reshape(13 * npb, nf)[:, :n]
        for nm, a, b in (("P_D", 0, 4 * npb), ("P_Sp", 4 * npb, 8 * npb), ("P_Sd", 8 * npb, 9 * npb), ("P_Sg", 9 * npb, 13 * npb)):
            print(f"  patch {P} {nm}: |g-o|/max|o| = {np.abs(gb[a:b] - fo[i][a:b]).max() / np.abs(fo[i][a:b]).max():.2e}")
    perm, Z = res["ctx"].debug_zeta(10 ** 8)
    ptr, pat = res["ptr"], res["pat"]
    tgt = np.repeat(np.arange(ptr.size - 1), np.diff(ptr))
    sample = np.sort(perm)[:: max(1, perm.size // int(__import__("os").environ.get("DBG_N", "200")))]
    inv = np.empty(perm.max() + 1, np.int64); inv[perm] = np.arange(perm.size)
    r = O.build_rows(S, *tgs, tgt[sample], pat[sample], prec="d", zeta=True)
    zo = U.zeta_to_gpu_layout(r[2], npb)
    zg = np.stack([Z[inv[k]][: 9 * npb] for k in sample])
    for nm, a, b in (("Theta", 0, npb), ("W", npb, 5 * npb), ("dW", 5 * npb, 9 * npb)):
        sc = np.abs(zo[:, a:b]).max(1)
        er = np.abs(zg[:, a:b] - zo[:, a:b]).max(1) / sc
        print(f"  zeta {nm}: rel err median {np.median(er):.2e} max {er.max():.2e} (pair {sample[er.argmax()]})")
        # per degree l
        if nm != "Theta":
            blk = (zg[:, a:b] - zo[:, a:b]).reshape(len(sample), 4, npb); ref = zo[:, a:b].reshape(len(sample), 4, npb)
        else:
            blk = (zg[:, a:b] - zo[:, a:b]).reshape(len(sample), 1, npb); ref = zo[:, a:b].reshape(len(sample), 1, npb)
        per_l = []
        for l in range(1, p + 1):
            c0, c1 = l * (l - 1) // 2, l * (l + 1) // 2
            per_l.append(np.abs(blk[:, :, c0:c1]).max() / max(np.abs(ref[:, :, c0:c1]).max(), 1e-300))
        print("    per l:", " ".join(f"{x:.1e}" for x in per_l))
    go = [res["vals"][k].reshape(-1, n)[sample] for k in range(4)]
    for k, nm in enumerate(("S", "D", "Sp", "Dp")):
        o = r[0][k]
        er = np.abs(go[k] - o).max(1) / np.abs(o).max(1)
        print(f"  rows {nm}: rel err median {np.median(er):.2e} max {er.max():.2e}")
    # which pairs are off (Theta block), by position in the patch-major order
    a, b = 0, npb
    sc = np.abs(zo[:, a:b]).max(1); er = np.abs(zg[:, a:b] - zo[:, a:b]).max(1) / sc
    bad = np.where(er > 1e-6)[0]
    pos = inv[sample]
    print(f"  bad pairs {bad.size} of {sample.size}; positions mod 32: {np.bincount(pos[bad] % 32, minlength=32).tolist()}")
    print(f"  positions mod 24: {np.bincount(pos[bad] % 24, minlength=24).tolist()}")
    print("  first bad: pos", pos[bad][:12].tolist(), "k", sample[bad][:12].tolist(), "status", res["status"][sample[bad]][:12].tolist(),
          "self", (tgs[2][tgt[sample[bad]]] >= 0)[:12].tolist())
    print("  status of all sampled:", np.bincount(res["status"][sample]).tolist(), " of bad:", np.bincount(res["status"][sample[bad]]).tolist())
