"""high order p = 12, 14 (Table 3 needs p >= 12 for
E_inf <= 1e-9) through the C ABI on the GPU, against the binary128 truth with the fp64
rounding envelope (tests/parity_util.py): a coarse unit sphere (80 patches, the near rule of config 2),
on-surface node targets and off-surface targets at 10^U(-12,0) h on both sides; near lists bit-exact; the
fit operators of two patches within the envelope; rows of a seeded sample of pairs (spread over patches so
the binary128 fits run in parallel) through the parity bar."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O
from synth.configs import make_config
from synth.geometry import Surface
import parity_util as U

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("p", [12, 14])
def test_high_order_sphere(p):
    cfg = make_config(2, n_off=300, freq=2, p=p)
    S = cfg["surface"]
    keep = np.concatenate([np.arange(0, S.n_patches * S.n, 11), np.arange(S.n_patches * S.n, cfg["tx"].shape[0])])
    tgs = (cfg["tx"][keep], cfg["tnormal"][keep], cfg["self_node"][keep], cfg["side"][keep])
    res = U.gpu_build(cfg, S, tgs)
    assert int(res["fit_status"].max()) == 0
    ptr_o, pat_o = O.near_list(S, tgs[0], tgs[2], cfg["eta"])
    assert np.array_equal(res["ptr"], ptr_o) and np.array_equal(res["pat"], pat_o)
    tg, pa = O.pairs_from_ptr(ptr_o, pat_o)
    rng = np.random.default_rng(p)
    patches = rng.choice(S.n_patches, 12, replace=False)
    sel = np.concatenate([rng.permutation(np.where(pa == q)[0])[:30] for q in patches])
    sel = np.sort(sel)
    ref = U.reference(S, tgs, tg[sel], pa[sel])
    inv = np.unique(tg[sel], return_inverse=True)[1]
    st = U.gate_all([res["vals"][k].reshape(-1, S.n)[sel] for k in range(4)], ref, inv, tag=f"p={p}")
    print(f"p = {p}: {sel.size} pairs of {len(patches)} patches; stats {st}")
    # fit operators of two patches against the truth (Layout<P>::FIT block, rows padded to NF)
    n, npb = S.n, p * (p + 1) // 2
    stride = res["ctx"].fit_bytes(1) // 8
    g = res["fit"].view(S.n_patches, stride).cpu().numpy()
    E, Q = 6 * p, 2 * p
    off = 32 + 6 * E + 9 * Q
    nf = n + ((4 - n % 16) + 16) % 16
    two = np.array([int(patches[0]), int(patches[1])])
    Ssub = Surface(p=p, q=S.q, nodes=S.nodes[two], normals=S.normals[two], weights=S.weights[two],
                   verts=S.verts[two], edge_x=S.edge_x[two], edge_dx=S.edge_dx[two], uv=S.uv)
    ft, _ = O.patch_fit(Ssub, prec="q")
    fo, _ = O.patch_fit(Ssub, prec="d")
    for i, P in enumerate(two):
        gb = g[P, off:off + 13 * npb * nf].reshape(13 * npb, nf)[:, :n]
        err, eo, scale = np.abs(gb - ft[i]).max(), np.abs(fo[i] - ft[i]).max(), np.abs(ft[i]).max()
        print(f"p = {p} patch {P}: fit error GPU {err / scale:.2e}, fp64 oracle {eo / scale:.2e} (x max|P|)")
        assert err <= 8 * eo + 1e-15 * scale
