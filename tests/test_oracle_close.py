"""Close-evaluation pins of the oracle: the north star's "twelve-digit close evaluation" (
uniformity test S:L704), against independent mpmath truths (tests/close_truth.py) for density 1, where the
harmonic fit is exact (c^(1,1) = (0,0,0,-1)) and only the line-integral quadrature (Newton
t0, SSQ, the sinh-split Omega_0 rule, readings A5, A9-A12) is exercised.

Two statements, measured separately (full tables: tools/close_sweep.py -> profiles/r02_close_sweep.txt):
* the METHOD (the oracle in binary128: no rounding) is accurate to ~12 digits uniformly in the normal distance
  delta = 1e-1 .. 1e-14 h, over interior, near-edge (lateral l >= 1e-6 h) and near-vertex (1e-4 h)
  projections, on both sides;
* an fp64 EVALUATION additionally carries the rounding floor ~ eps h / l of targets at lateral distance l from
  an edge (the solid angle moves by ~2 eps / l when the edge moves normally by eps, and the local-frame
  coordinates are rounded at eps h), and is otherwise uniform in delta: the error at 1e-12 h and
  1e-14 h is within 10x of the error at 0.1 h plus that floor."""
import numpy as np
import pytest

from oracle import oracle as O
from synth.geometry import make_flat_surface, make_cap_surface
import close_truth as CT

EPS = 2.0 ** -53
FLAT_TRI = np.array([[0.0, 0.0, 0.0], [1.0, 0.125, 0.0], [0.25, 0.875, 0.0]])


def flat_families(h, laterals=(1e-4, 1e-6, 1e-8), vertex=(1e-2, 1e-4)):
    """name -> (projection xy, lateral distance to the nearest edge or vertex / h)."""
    fam = {"interior": (np.array([0.4, 0.33]), 0.2)}
    a, b = FLAT_TRI[0, :2], FLAT_TRI[1, :2]
    u = (b - a) / np.linalg.norm(b - a)
    nin = np.array([-u[1], u[0]])
    foot = a + 0.37 * (b - a)
    for l in laterals:
        fam[f"edge+{l:g}"] = (foot + l * h * nin, l)
        fam[f"edge-{l:g}"] = (foot - l * h * nin, l)
    v1 = FLAT_TRI[1, :2]
    bis = (FLAT_TRI[0, :2] - v1) / np.linalg.norm(FLAT_TRI[0, :2] - v1) + \
        (FLAT_TRI[2, :2] - v1) / np.linalg.norm(FLAT_TRI[2, :2] - v1)
    bis /= np.linalg.norm(bis)
    for l in vertex:
        fam[f"vertex+{l:g}"] = (v1 + l * h * bis, l)
        fam[f"vertex-{l:g}"] = (v1 - l * h * bis, l)
    return fam


def cap_families(S, h, laterals=(1e-4, 1e-6, 1e-8), vertex=(1e-2, 1e-4, 1e-6)):
    """Projections on the exact patch of a cap: name -> (point on the surface, lateral distance / h)."""
    def sp(s_, t_):
        X, Xs, Xt = S.eval_patch(0, s_, t_)
        N = np.cross(Xs[0], Xt[0])
        return X[0], Xs[0], Xt[0], N / np.linalg.norm(N)
    X0, _, _, _ = sp(1 / 3, 1 / 3)
    fam = {"interior": (X0, 0.2)}
    Xe, Xs, Xt, N = sp(0.37, 0.0)
    nin = np.cross(N, Xs / np.linalg.norm(Xs))
    for l in laterals:
        fam[f"edge+{l:g}"] = (Xe + l * h * nin, l)
        fam[f"edge-{l:g}"] = (Xe - l * h * nin, l)
    Xv, Xs, Xt, N = sp(1.0, 0.0)
    a_ = -Xs / np.linalg.norm(Xs)
    b_ = (Xt - Xs) / np.linalg.norm(Xt - Xs)
    bis = a_ + b_
    bis -= np.dot(bis, N) * N
    bis /= np.linalg.norm(bis)
    for l in vertex:
        fam[f"vertex+{l:g}"] = (Xv + l * h * bis, l)
        fam[f"vertex-{l:g}"] = (Xv - l * h * bis, l)
    return fam


DELTAS = (1e-1, 1e-4, 1e-8, 1e-12, 1e-14)


@pytest.mark.parametrize("p", [8])
def test_flat_patch_close_evaluation_vs_closed_forms(p):
    """Density 1 on a flat triangle: RAW row sums of S, D, S', D' (nu' = z) against the closed forms, both sides."""
    S = make_flat_surface([FLAT_TRI], p, 2 * p)
    h = max(np.linalg.norm(FLAT_TRI[i] - FLAT_TRI[(i + 1) % 3]) for i in range(3))
    fams = flat_families(h, laterals=(1e-6,), vertex=(1e-4,))
    print(f"\nflat p={p}: max error over S (rel), D, S' (abs), D' (rel) at delta/h = {DELTAS}")
    for nm, (xy, ell) in fams.items():
        for sg in (1, -1):
            X = np.array([[xy[0], xy[1], sg * d * h] for d in DELTAS])
            T = len(X)
            args = (S, X, np.tile([0, 0, 1.0], (T, 1)), np.full(T, -1, np.int64), np.full(T, sg, np.int8),
                    np.arange(T, dtype=np.int64), np.zeros(T, np.int32))
            rows = {pr: O.build_rows(*args, raw=True, prec=pr)[0].sum(2) for pr in ("d", "q")}
            err = {pr: np.zeros(T) for pr in rows}
            for i in range(T):
                tr = CT.flat_truths(FLAT_TRI, X[i])
                for pr in rows:
                    err[pr][i] = max(abs(rows[pr][k, i] - tr[key]) / (max(abs(tr[key]), 1.0) if key in ("S", "Dp") else 1.0)
                                     for k, key in enumerate(("S", "D", "Sp", "Dp")))
            print(f"  {nm:12s} {sg:+d}  fp64 " + " ".join(f"{v:.0e}" for v in err["d"]) +
                  "   quad " + " ".join(f"{v:.0e}" for v in err["q"]))
            floor = 1e-12 + 30 * EPS / ell
            assert (err["q"] <= 1e-11).all(), (nm, sg, err["q"])          # the method: 12 digits
            assert (err["d"] <= floor).all(), (nm, sg, err["d"], floor)     # fp64: + rounding floor
            assert err["d"][-2:].max() <= 10 * err["d"][0] + floor          # uniform in delta


def test_curved_patch_solid_angle_close_evaluation():
    """Density 1 on config 5's curved patch (p = 10): Omega_0 (= -4pi D[1]) and the Biot-Savart dOmega_0/dnu'
    (= -4pi D'[1]) against adaptive mpmath line integrals along the same edge interpolant."""
    p = 10
    S = make_cap_surface(0.2, p, 2 * p)
    v = S.verts[0]
    h = max(np.linalg.norm(v[i] - v[(i + 1) % 3]) for i in range(3))
    EC = CT.EdgeCurves(S.edge_x[0], S.edge_dx[0], S.verts[0])
    fams = cap_families(S, h, laterals=(1e-6,), vertex=(1e-4,))
    deltas = (1e-2, 1e-8, 1e-14)
    print(f"\ncap p={p}: Omega_0/4pi abs | dOmega_0 rel at delta/h = {deltas}")
    for nm in ("interior", "edge+1e-06", "vertex+0.0001"):
        x0, ell = fams[nm]
        nrm = x0 / np.linalg.norm(x0)
        X = np.array([x0 + d * h * nrm for d in deltas])
        NU = np.tile(nrm, (len(X), 1))
        res = {pr: O.pairs_debug(S, 0, X, NU, side=np.ones(len(X), np.int32), prec=pr) for pr in ("d", "q")}
        tr = [EC.solid_angle(X[i], NU[i], 1) for i in range(len(X))]
        for pr in ("d", "q"):
            e0 = np.array([abs(res[pr]["Omega0"][i] - tr[i][0]) / (4 * np.pi) for i in range(len(X))])
            e1 = np.array([abs(res[pr]["dOmega0"][i] / h - tr[i][1]) / max(1.0, abs(tr[i][1])) for i in range(len(X))])
            print(f"  {nm:14s} {pr}: " + " ".join(f"{x:.0e}" for x in e0) + " | " + " ".join(f"{x:.0e}" for x in e1))
            if pr == "q":
                assert (e0 <= 1e-12).all() and (e1 <= 1e-11).all(), (nm, e0, e1)
            else:
                floor = 1e-12 + 30 * EPS / ell
                assert (e0 <= floor).all() and (e1 <= 10 * floor).all(), (nm, e0, e1, floor)
