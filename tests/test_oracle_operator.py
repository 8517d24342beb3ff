"""Full-operator pins of the oracle on closed surfaces (north star; SURVEY §8(c) full-operator table):
Gauss law D[1], unit-sphere eigenrelations of S, D, S', D' for Y_l^m, Green's third
identity, the correction/smooth splitting, and the near list vs a k-d tree."""
import numpy as np
import pytest
from scipy.spatial import cKDTree

from oracle import oracle as O
from synth.geometry import make_sphere_surface, make_torus_surface


def _all_pairs(T, P):
    return np.repeat(np.arange(T), P).astype(np.int64), np.tile(np.arange(P), T).astype(np.int32)


@pytest.fixture(scope="module")
def sphere8():
    S = make_sphere_surface(4, 8, 16)
    x0 = S.nodes[3, 5]
    tx = np.array([x0, 0.6 * x0, 1.4 * x0, x0 * (1 - 1e-9), x0 * (1 + 1e-9)])
    nu = np.tile(x0, (5, 1))
    sn = np.array([3 * S.n + 5, -1, -1, -1, -1], np.int64)
    sd = np.array([0, -1, 1, -1, 1], np.int8)
    tg, pa = _all_pairs(5, S.n_patches)
    vals, st = O.build_rows(S, tx, nu, sn, sd, tg, pa, raw=True)
    return S, x0, vals.reshape(4, 5, S.n_patches * S.n), st


def test_gauss_law(sphere8):
    S, x0, vals, st = sphere8
    D1 = vals[1].sum(1)
    assert np.abs(D1 - np.array([-0.5, -1.0, 0.0, -1.0, 0.0])).max() < 5e-12


def test_unit_sphere_eigenrelations(sphere8):
    """Density Y = z (l = 1) and Y = Re R_3^2-type cubic: closed forms of the SURVEY table."""
    S, x0, vals, st = sphere8
    xs = S.nodes.reshape(-1, 3)
    r = np.array([1.0, 0.6, 1.4, 1.0, 1.0])
    for l, Y, Yt in [(1, xs[:, 2], x0[2]), (2, xs[:, 0] * xs[:, 1], x0[0] * x0[1]),
                     (3, xs[:, 2] * (5 * xs[:, 2] ** 2 - 3), x0[2] * (5 * x0[2] ** 2 - 3))]:
        c = 2 * l + 1
        exp = {
            0: [1 / c, r[1] ** l / c, r[2] ** (-l - 1) / c, 1 / c, 1 / c],
            1: [-1 / (2 * c), -(l + 1) * r[1] ** l / c, l * r[2] ** (-l - 1) / c, -(l + 1) / c, l / c],
            2: [-1 / (2 * c), l * r[1] ** (l - 1) / c, -(l + 1) * r[2] ** (-l - 2) / c, l / c, -(l + 1) / c],
            3: [-l * (l + 1) / c] * 5,
        }
        exp[3][1] = -l * (l + 1) * r[1] ** (l - 1) / c
        exp[3][2] = -l * (l + 1) * r[2] ** (-l - 2) / c
        for k in range(4):
            got = vals[k] @ Y / Yt
            # D' at 1e-9 from the surface sees the per-patch fit residual through a hypersingular kernel
            tol = np.array([2e-5, 5e-6, 5e-6, 2e-4, 2e-4]) if k == 3 else (5e-6 if k == 2 else 5e-7)
            assert (np.abs(got - np.array(exp[k])) < tol).all(), (l, k, got, exp[k])


def test_greens_identity_torus():
    """u harmonic inside (sources outside): 1/2 u = S[du/dnu] - D_PV[u] on S, u inside,
    0 outside; 1/2 du/dnu = S'_PV[du/dnu] - D'[u] on S."""
    S = make_torus_surface(2.0, 0.5, 16, 24, 6, 12)
    rng = np.random.default_rng(3)
    src = rng.normal(size=(4, 3)); src = 3.2 * src / np.linalg.norm(src, axis=1, keepdims=True)
    a = rng.normal(size=4)
    xs = S.nodes.reshape(-1, 3); ns = S.normals.reshape(-1, 3)
    def u_of(x):
        return sum(a[j] / np.linalg.norm(x - src[j], axis=-1) for j in range(4))
    def dudn(x, n):
        return sum(-a[j] * np.sum((x - src[j]) * n, -1) / np.linalg.norm(x - src[j], axis=-1) ** 3 for j in range(4))
    U = u_of(xs); dU = dudn(xs, ns)
    g = [17, 401, 2000]
    tx = np.concatenate([xs[g], np.array([[2.0, 0.0, 0.1], [0.0, 0.0, 0.0]])])
    nu = np.concatenate([ns[g], np.array([[1.0, 0, 0], [0, 0, 1.0]])])
    sn = np.array(g + [-1, -1], np.int64); sd = np.array([0, 0, 0, -1, 1], np.int8)
    tg, pa = _all_pairs(len(tx), S.n_patches)
    vals, st = O.build_rows(S, tx, nu, sn, sd, tg, pa, raw=True)
    vals = vals.reshape(4, len(tx), -1)
    rep = vals[0] @ dU - vals[1] @ U
    ref = np.concatenate([0.5 * U[g], [u_of(tx[3]), 0.0]])
    assert np.abs(rep - ref).max() < 1e-5 * np.abs(U).max()       # p = 6 (cf. Table 3: 2e-5)
    rep_n = vals[2] @ dU - vals[3] @ U
    ref_n = np.concatenate([0.5 * dU[g], [dudn(tx[3], nu[3]), 0.0]])
    assert np.abs(rep_n - ref_n).max() < 3e-4 * np.abs(dU).max()     # converges under refinement


def test_correction_plus_smooth_equals_operator():
    """D_total = D_smooth(all nodes, self node skipped) + correction rows on near pairs (P:L1581-1598,
    reading A14): reproduces the eigenrelations for all four kernels with density Y = z."""
    S = make_sphere_surface(4, 8, 16)
    x0 = S.nodes[7, 9]
    tx = np.array([x0, 0.93 * x0, 1.05 * x0])
    nu = np.tile(x0, (3, 1)); sn = np.array([7 * S.n + 9, -1, -1], np.int64); sd = np.array([0, -1, 1], np.int8)
    ptr, pat = O.near_list(S, tx, sn, 1.5)
    tg, pa = O.pairs_from_ptr(ptr, pat)
    vals, st = O.build_rows(S, tx, nu, sn, sd, tg, pa, raw=False)
    xs = S.nodes.reshape(-1, 3); ns = S.normals.reshape(-1, 3); w = S.weights.reshape(-1)
    Y = xs[:, 2]
    for t in range(3):
        d = tx[t] - xs
        r = np.linalg.norm(d, axis=1)
        msk = np.arange(len(xs)) != sn[t]
        dn = np.sum(d * ns, 1); dnp = d @ nu[t]
        K = [1 / r, dn / r ** 3, -dnp / r ** 3, (ns @ nu[t]) / r ** 3 - 3 * dn * dnp / r ** 5]
        sel = tg == t
        cols = (pa[sel][:, None] * S.n + np.arange(S.n)[None]).ravel()
        tot = []
        for k in range(4):
            sm = np.sum((K[k] * w * Y)[msk]) / (4 * np.pi)
            tot.append(sm + vals[k][sel].ravel() @ Y[cols])
        rr = np.linalg.norm(tx[t])
        if t == 0:
            ref = [1 / 3, -1 / 6, -1 / 6, -2 / 3]
        elif t == 1:
            ref = [rr / 3, -2 * rr / 3, 1 / 3, -2 / 3]
        else:
            ref = [rr ** -2 / 3, rr ** -2 / 3, -2 * rr ** -3 / 3, -2 * rr ** -3 / 3]
        assert np.abs(np.array(tot) / x0[2] - np.array(ref)).max() < 1e-4


def test_near_list_vs_kdtree():
    S = make_torus_surface(2.0, 0.5, 12, 20, 4, 8)
    rng = np.random.default_rng(1)
    tx = np.concatenate([S.nodes.reshape(-1, 3)[::7], rng.uniform(-2.6, 2.6, (500, 3)) * [1, 1, 0.3]])
    sn = np.full(len(tx), -1, np.int64); sn[: len(S.nodes.reshape(-1, 3)[::7])] = np.arange(0, S.n_patches * S.n, 7)
    ptr, pat = O.near_list(S, tx, sn, 1.5)
    # independent: k-d tree ball query around every patch ball (reading A6 definitions)
    w = S.weights
    c = np.einsum("pi,pia->pa", w, S.nodes) / w.sum(1)[:, None]
    pts = np.concatenate([S.nodes, S.verts, S.edge_x.reshape(S.n_patches, -1, 3)], 1)
    R = np.linalg.norm(pts - c[:, None], axis=2).max(1)
    h = np.max(np.stack([np.linalg.norm(S.verts[:, i] - S.verts[:, (i + 1) % 3], axis=1) for i in range(3)], 1), 1)
    tree = cKDTree(tx)
    sets = [set() for _ in range(len(tx))]
    for P in range(S.n_patches):
        for t in tree.query_ball_point(c[P], R[P] + 1.5 * h[P]):
            sets[t].add(P)
    for t in range(len(tx)):
        if sn[t] >= 0:
            sets[t].add(int(sn[t] // S.n))
        got = pat[ptr[t]:ptr[t + 1]]
        assert list(got) == sorted(sets[t])


@pytest.mark.parametrize("p", [12, 14])
def test_high_order_sphere_operators(p):
    """SURVEY §8(f) NEXT(3) at the oracle: p = 12, 14 on a 180-patch sphere.  Gauss law and the Y_3 eigenrelations of
    S and D on the surface, inside and outside improve on p = 8 (~1e-7 on the surface: Table 3 reaches
    ~1e-9 .. 1e-11 at p = 12, 14)."""
    S = make_sphere_surface(3, p, 2 * p)
    x0 = S.nodes[3, 5]
    tx = np.array([x0, 0.6 * x0, 1.4 * x0])
    nu = np.tile(x0, (3, 1))
    sn = np.array([3 * S.n + 5, -1, -1], np.int64)
    sd = np.array([0, -1, 1], np.int8)
    tg, pa = _all_pairs(3, S.n_patches)
    vals, st = O.build_rows(S, tx, nu, sn, sd, tg, pa, raw=True)
    assert (st & 6).max() == 0
    V = vals.reshape(4, 3, -1)
    # Gauss law holds to the fp64 rounding of the fit (grows with p: ~1e-11 at p = 8, ~1e-10 at p = 12, 14)
    assert np.abs(V[1].sum(1) - np.array([-0.5, -1.0, 0.0])).max() < 1e-9
    xs = S.nodes.reshape(-1, 3)
    l, c = 3, 7
    Y = xs[:, 2] * (5 * xs[:, 2] ** 2 - 3)
    Yt = x0[2] * (5 * x0[2] ** 2 - 3)
    r = np.array([1.0, 0.6, 1.4])
    expS = np.array([1 / c, r[1] ** l / c, r[2] ** (-l - 1) / c])
    expD = np.array([-1 / (2 * c), -(l + 1) * r[1] ** l / c, l * r[2] ** (-l - 1) / c])
    eS, eD = np.abs(V[0] @ Y / Yt - expS), np.abs(V[1] @ Y / Yt - expD)
    print(p, eS, eD)
    # p = 12: S ~1e-10, D ~1e-11 (p = 8: ~1e-7 / 1e-6 on the surface).  p = 14: fp64 rounding dominates (the
    # same rows in long double: S 1.4e-10 / 1.8e-11 / 1.0e-9, D 1.1e-11 / 9e-13 / 7.7e-11 -- DESIGN.md §11)
    bS, bD = (1e-9, 2e-10) if p == 12 else (3e-7, 2e-9)
    assert eS.max() < bS and eD.max() < bD
