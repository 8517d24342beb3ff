"""Per-pair pins of the oracle (SURVEY §8(c) "What pins each part"): brute-force 2-form surface
integrals (Thm 3.4 / Thm 3.5), Van Oosterom-Strackee solid angles
(P:L1090-1096), finite differences for D', an independent least-squares fit
(P:L715-746), the mu = 1 row-sum identity and frame invariance."""
import copy

import numpy as np
import pytest

from oracle import oracle as O
import indep
from synth.geometry import make_sphere_surface, make_torus_surface, make_flat_surface


def _brute_W_Theta(S, P, dbg, rp_loc, with_grad=False):
    """W^{(l,m)} = -sqrt2 Im int_P (0,gradG)(0,nu)(0,grad S^{(l,m)}) da   (eq cdlp1form + wlmdef)
    Theta^{(l,m)} = sqrt2 Im int_P (G grad S - gradG S).nu da              (eq cslp1form, G2)
    in the patch's scaled local frame, by adaptive quadrature over the exact patch map."""
    p = S.p
    o, Rm, h = dbg["origin"], dbg["Rm"], dbg["h"]
    Sf = indep.S_funcs(p)
    npb = p * (p + 1) // 2

    def f(s, t):
        X, Xs, Xt = S.eval_patch(P, s, t)
        Xl = (X - o) @ Rm.T / h; Xsl = Xs @ Rm.T / h; Xtl = Xt @ Rm.T / h
        N = np.cross(Xsl, Xtl)
        d = rp_loc[None] - Xl
        r = np.linalg.norm(d, axis=1)
        gG = d / (4 * np.pi * r[:, None] ** 3); G = 1 / (4 * np.pi * r)
        Sv, Gv, _ = Sf(Xl[:, 0], Xl[:, 1], Xl[:, 2])
        ab0 = -np.sum(gG * N, 1); abv = np.cross(gG, N)
        out = []
        for l in range(1, p + 1):
            for m in range(1, l + 1):
                k = indep.hidx(l, m)
                g = Gv[k].T
                s0 = -np.sum(abv * g, 1)
                sv = ab0[:, None] * g + np.cross(abv, g)
                th = np.sum((G[:, None] * g - gG * Sv[k][:, None]) * N, 1)
                out.append(np.concatenate([s0[:, None], sv, th[:, None]], 1))
        return np.concatenate(out, 1)
    tot = indep.adaptive_triangle(f, tol=1e-13).reshape(npb, 5)
    return -np.sqrt(2) * tot[:, :4].imag, np.sqrt(2) * tot[:, 4].imag


def _targets(S, P):
    c = S.nodes[P].mean(0)
    nrm = S.normals[P].mean(0); nrm /= np.linalg.norm(nrm)
    v = S.verts[P]
    h = max(np.linalg.norm(v[i] - v[(i + 1) % 3]) for i in range(3))
    mid = 0.5 * (S.edge_x[P, 0, S.q // 2] + S.edge_x[P, 0, S.q // 2 - 1])
    return [(c + 0.3 * h * nrm, 1, 1e-11), (c - 0.1 * h * nrm, -1, 1e-11),
            (mid - 0.05 * h * nrm, -1, 2e-9), (v[2] + 0.08 * h * nrm, 1, 1e-9), (c + 2 * h * nrm, 1, 1e-12),
            (S.nodes[P, 7] + 0.02 * h * nrm, 1, 1e-10)]


@pytest.mark.parametrize("geom,prec", [("sphere", "d"), ("torus", "d"), ("sphere", "q")])
def test_W_Theta_vs_bruteforce_2form(geom, prec):
    """prec "q": the binary128 truth build of the same source meets the same pins."""
    if geom == "sphere":
        S = make_sphere_surface(2, 6, 16); P = 5
    else:
        S = make_torus_surface(2.0, 0.5, 6, 10, 6, 16); P = 7
    for x, side, tol in _targets(S, P):
        dbg = O.pair_debug(S, P, x, None, side=side, prec=prec)
        rp = (x - dbg["origin"]) @ dbg["Rm"].T / dbg["h"]
        W, Th = _brute_W_Theta(S, P, dbg, rp)
        sc = max(np.abs(W).max(), np.abs(Th).max())
        assert np.abs(W - dbg["W"]).max() <= tol * sc, (x, np.abs(W - dbg["W"]).max())
        assert np.abs(Th - dbg["Theta"]).max() <= tol * sc


def test_solid_angle_flat_triangle_vs_van_oosterom_strackee():
    """Omega_0 := -int grad(1/|r'-r|).nu da (reading G1) equals the VOS signed solid angle."""
    tri = np.array([[0.0, 0.0, 0.0], [1.0, 0.1, 0.0], [0.2, 0.9, 0.0]])
    S = make_flat_surface([tri], 4, 16)
    rng = np.random.default_rng(0)
    for _ in range(25):
        x = np.array([rng.uniform(-0.5, 1.5), rng.uniform(-0.5, 1.5), rng.choice([-1, 1]) * 10 ** rng.uniform(-6, 0)])
        side = 1 if x[2] > 0 else -1
        dbg = O.pair_debug(S, 0, x, None, side=side)
        ref = indep.vos_solid_angle(tri[0], tri[1], tri[2], x)
        assert abs(dbg["Omega0"] - ref) < 1e-10, (x, dbg["Omega0"], ref)
    # self target on a flat patch: principal value 0 (reading A7)
    dbg = O.pair_debug(S, 0, S.nodes[0, 5], None, self_local=5, side=0)
    assert abs(dbg["Omega0"]) < 1e-10


def test_dW_and_Dprime_vs_finite_differences():
    S = make_sphere_surface(2, 6, 16); P = 5
    c = S.nodes[P].mean(0)
    for x, side in [(c + 0.2 * 0.5 * c, 1), (0.9 * c, -1), (S.nodes[P, 3] * 1.05, 1)]:
        nu = x / np.linalg.norm(x)
        dbg = O.pair_debug(S, P, x, nu, side=side)
        eps = 1e-5
        dp = O.pair_debug(S, P, x + eps * nu, nu, side=side)
        dm = O.pair_debug(S, P, x - eps * nu, nu, side=side)
        fdW = (dp["W"] - dm["W"]) / (2 * eps) * dbg["h"]       # local scaled units
        assert np.abs(fdW - dbg["dW"]).max() < 1e-7 * max(1, np.abs(dbg["dW"]).max())
        fdD = (dp["rows"][1] - dm["rows"][1]) / (2 * eps)       # D' row = d/dnu' of the D row
        assert np.abs(fdD - dbg["rows"][3]).max() < 1e-7 * np.abs(dbg["rows"][3]).max()
        fdO = (dp["Omega0"] - dm["Omega0"]) / (2 * eps) * dbg["h"]
        assert abs(fdO - dbg["dOmega0"]) < 1e-7 * max(1, abs(dbg["dOmega0"]))


def test_fit_vs_independent_least_squares():
    """P_D = A^+[:, :n], P_Sp, P_Sd = B^+, P_Sg = P_D Hm P_Sd (reading A1) vs numpy's SVD
    pseudo-inverse of A assembled from the sympy harmonics."""
    p = 5
    S = make_sphere_surface(2, p, 10)
    fit, st = O.patch_fit(S)
    assert (st == 0).all()
    n, npb = p * p, p * (p + 1) // 2
    f = indep.S_funcs(p)
    for P in (0, 11, 63):
        dbg = O.pair_debug(S, P, S.nodes[P].mean(0) * 1.5, None)
        Xl = (S.nodes[P] - dbg["origin"]) @ dbg["Rm"].T / dbg["h"]
        nl = S.normals[P] @ dbg["Rm"].T
        Sv, Gv, _ = f(Xl[:, 0], Xl[:, 1], Xl[:, 2])
        idx = [indep.hidx(l, m) for l in range(1, p + 1) for m in range(1, l + 1)]
        F = np.sqrt(2) * Gv[idx].imag            # [np, 3, n]
        Hm = np.sqrt(2) * Sv[idx].imag.T         # [n, np]
        F1, F2, F3 = F[:, 0].T, F[:, 1].T, F[:, 2].T
        Z = np.zeros_like(F1)
        A = np.block([[Z, -F1, -F2, -F3], [F1, Z, -F3, F2], [F2, F3, Z, -F1], [F3, -F2, F1, Z]])
        Ap = np.linalg.pinv(A)
        B = F1 * nl[:, :1] + F2 * nl[:, 1:2] + F3 * nl[:, 2:3]      # grad H . nu
        Bp = np.linalg.pinv(B)
        PD = Ap[:, :n]
        PSp = sum(nl[:, a][None, :] * Ap[:, (a + 1) * n:(a + 2) * n] for a in range(3))
        PSg = PD @ Hm @ Bp
        ref = np.concatenate([PD, PSp, Bp, PSg], 0)
        got = fit[P]
        assert np.abs(got - ref).max() < 1e-10 * np.abs(ref).max()


def test_mu_one_row_sum_identity():
    """mu = 1 fits exactly with c^{(1,1)} = (0,0,0,-1) (H^{(1,1)} = z), so every RAW D row sums to
    -Omega_0/4pi."""
    S = make_torus_surface(2.0, 0.5, 6, 10, 5, 10)
    rng = np.random.default_rng(9)
    for P in (0, 17, 60):
        for _ in range(3):
            x = S.nodes[P, rng.integers(S.n)] + rng.normal(0, 0.2, 3)
            dbg = O.pair_debug(S, P, x, None, side=2)
            assert abs(dbg["rows"][1].sum() + dbg["Omega0"] / (4 * np.pi)) < 1e-13 * max(1, np.abs(dbg["rows"][1]).sum())
    # self target: the principal-value shift is included (A7)
    dbg = O.pair_debug(S, 3, S.nodes[3, 4], None, self_local=4, side=0)
    assert abs(dbg["rows"][1].sum() + dbg["Omega0"] / (4 * np.pi)) < 1e-13


def test_frame_invariance():
    """A rigid motion of all inputs leaves every weight unchanged."""
    S = make_sphere_surface(2, 5, 10)
    th = 0.7
    Q = np.array([[np.cos(th), -np.sin(th), 0], [np.sin(th), np.cos(th), 0], [0, 0, 1.0]]) @ \
        np.array([[1, 0, 0], [0, np.cos(0.3), -np.sin(0.3)], [0, np.sin(0.3), np.cos(0.3)]])
    b = np.array([0.3, -1.2, 2.0])
    S2 = copy.copy(S)
    S2.nodes = S.nodes @ Q.T + b; S2.normals = S.normals @ Q.T; S2.verts = S.verts @ Q.T + b
    S2.edge_x = S.edge_x @ Q.T + b; S2.edge_dx = S.edge_dx @ Q.T
    x = np.array([S.nodes[4, 3] * 1.01, S.nodes[4, 7] * 0.98, S.nodes[9, 0]])
    nu = x / np.linalg.norm(x, axis=1, keepdims=True)
    sn = np.array([-1, -1, 9 * S.n + 0], np.int64); sd = np.array([1, -1, 0], np.int8)
    tg = np.array([0, 0, 1, 1, 2, 2], np.int64); pa = np.array([4, 5, 4, 6, 9, 10], np.int32)
    v1, _ = O.build_rows(S, x, nu, sn, sd, tg, pa)
    v2, _ = O.build_rows(S2, x @ Q.T + b, nu @ Q.T, sn, sd, tg, pa)
    for k in range(4):
        assert np.abs(v1[k] - v2[k]).max() <= 1e-11 * np.abs(v1[k]).max()
