"""the paper's evaluation-phase workload (E4) on the oracle: four
interlocking tori (a = 3, b = 0.5, shifted 4.95 along x) and a uniform grid over
[-5,20] x [-6,6]^2.  Pins: the enclosed volume (closed form 4 * 2 pi^2 a b^2), the paper's
exterior-point count N_T at 101^3, and Green's representation S[du/dn] - D[u] = 0 at close
exterior targets for u harmonic inside the tori (P:L1841-1845 off the surface), with the operators
split as smooth rule + near correction."""
import numpy as np

from oracle import oracle as O
from synth.configs import make_config
from synth.geometry import make_interlocked_tori, inside_interlocked_tori


def test_tori_geometry_and_grid():
    S = make_interlocked_tori(6, 36, 4, 8)
    x = S.nodes.reshape(-1, 3); n = S.normals.reshape(-1, 3); w = S.weights.reshape(-1)
    assert abs((x * n).sum(1) @ w / 3 - 4 * 2 * np.pi ** 2 * 3.0 * 0.25) < 1e-9
    assert not inside_interlocked_tori(x + 1e-6 * n).any() and inside_interlocked_tori(x - 1e-6 * n).all()
    G = 101
    gx = np.linspace(-5.0, 20.0, G); gy = np.linspace(-6.0, 6.0, G)
    X = np.stack(np.meshgrid(gx, gy, gy, indexing="ij"), -1).reshape(-1, 3)
    n_ext = int((~inside_interlocked_tori(X)).sum())
    assert abs(n_ext - 1013571) <= 10, n_ext      # P:L1984 (grid points on the surfaces may go either way)


def green_residuals(S, tx, eta=1.5, seed=11):
    """|S[du/dn] - D[u]| / max|u| at exterior targets tx, u = sum a_j / |x - x_j| with x_j outside."""
    rng = np.random.default_rng(seed)
    src = rng.normal(size=(4, 3)); src = 30.0 * src / np.linalg.norm(src, axis=1, keepdims=True) + [7.4, 0, 0]
    a = rng.normal(size=4)
    xs = S.nodes.reshape(-1, 3); ns = S.normals.reshape(-1, 3); ws = S.weights.reshape(-1)
    U = sum(a[j] / np.linalg.norm(xs - src[j], axis=1) for j in range(4))
    dU = sum(-a[j] * np.sum((xs - src[j]) * ns, 1) / np.linalg.norm(xs - src[j], axis=1) ** 3 for j in range(4))
    T = tx.shape[0]
    sn = np.full(T, -1, np.int64); sd = np.ones(T, np.int8)
    ptr, pat = O.near_list(S, tx, sn, eta)
    tg, pa = O.pairs_from_ptr(ptr, pat)
    vals, _ = O.build_rows(S, tx, np.zeros_like(tx), sn, sd, tg, pa)
    n = S.n
    res = np.zeros(T)
    for i in range(T):
        d = tx[i] - xs
        r = np.linalg.norm(d, axis=1)
        s_sm = (ws / r) @ dU / (4 * np.pi)
        d_sm = (ws * np.sum(d * ns, 1) / r ** 3) @ U / (4 * np.pi)
        sel = np.where(tg == i)[0]
        c_s = sum(vals[0][k] @ dU[pa[k] * n:(pa[k] + 1) * n] for k in sel)
        c_d = sum(vals[1][k] @ U[pa[k] * n:(pa[k] + 1) * n] for k in sel)
        res[i] = abs(s_sm + c_s - d_sm - c_d) / np.abs(U).max()
    return res, np.diff(ptr)


def test_green_representation_close_targets():
    cfg = make_config(7, p=6, n_off=41)      # 41^3 grid keeps the oracle run short
    S = cfg["surface"]
    rng = np.random.default_rng(2)
    # close exterior targets: grid points with near pairs, plus points 1e-3 .. 1e-9 outside along normals
    xs = S.nodes.reshape(-1, 3); ns = S.normals.reshape(-1, 3)
    k = rng.choice(xs.shape[0], 8, replace=False)
    close = xs[k] + (10.0 ** -rng.uniform(3, 9, 8))[:, None] * ns[k]
    tx = np.concatenate([cfg["tx"][rng.choice(cfg["tx"].shape[0], 40, replace=False)], close])
    res, npairs = green_residuals(S, tx)
    print("Green representation residuals (exterior):", res.max(), np.median(res), "targets with pairs",
          int((npairs > 0).sum()))
    assert (npairs[-8:] > 0).all()
    assert res.max() < 1e-5
