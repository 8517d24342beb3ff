"""the paper's solve-phase workload (E3) on the oracle: the
stellarator of eq (stellarator) and Green's third identity,
1/2 u = S[du/dn] - D[u] on S for u harmonic inside (sources outside), with the operators split as
smooth rule + near correction (the product's use of the correction).  Pins: outward
orientation (enclosed volume > 0), the map against the printed formula, and Green's identity whose
residual falls with p (the discretisation error; Table 3 reports E_inf 2.1e-5 at p = 6, 2.8e-7 at p = 8
on its own mesh)."""
import numpy as np
import pytest

from oracle import oracle as O
from synth.geometry import make_stellarator_surface, STELLARATOR_DELTA


def test_stellarator_map_and_orientation():
    S = make_stellarator_surface(6, 18, 4, 8)
    x = S.nodes.reshape(-1, 3); n = S.normals.reshape(-1, 3); w = S.weights.reshape(-1)
    assert (x * n).sum(1) @ w / 3 > 0                      # outward normals: enclosed volume > 0
    assert np.abs(w @ n).max() < 1e-12 * w.sum()            # closed surface: integral of n dA = 0
    # vertices of patch 0 = r(u, v) of the printed formula at its parameter corners
    v, u = 0.0, 0.0
    r = sum(d * np.array([np.cos(v) * np.cos((1 - i) * u + j * v), np.sin(v) * np.cos((1 - i) * u + j * v),
                          np.sin((1 - i) * u + j * v)]) for (i, j), d in STELLARATOR_DELTA.items())
    assert np.allclose(S.verts[0][0], r, atol=1e-13)


def _green_residuals(p, nu_=12, nv_=36, eta=1.5):
    S = make_stellarator_surface(nu_, nv_, p, 2 * p)
    rng = np.random.default_rng(5)
    src = rng.normal(size=(4, 3)); src = 9.0 * src / np.linalg.norm(src, axis=1, keepdims=True)
    a = rng.normal(size=4)
    xs = S.nodes.reshape(-1, 3); ns = S.normals.reshape(-1, 3); ws = S.weights.reshape(-1)
    U = sum(a[j] / np.linalg.norm(xs - src[j], axis=1) for j in range(4))
    dU = sum(-a[j] * np.sum((xs - src[j]) * ns, 1) / np.linalg.norm(xs - src[j], axis=1) ** 3 for j in range(4))
    g = np.sort(rng.choice(xs.shape[0], 6, replace=False))
    tx, nu, sn, sd = xs[g], ns[g], g.astype(np.int64), np.zeros(len(g), np.int8)
    ptr, pat = O.near_list(S, tx, sn, eta)
    tg, pa = O.pairs_from_ptr(ptr, pat)
    vals, st = O.build_rows(S, tx, nu, sn, sd, tg, pa)        # near rows minus the smooth rule (A14)
    n = S.n
    res = []
    for i, t in enumerate(g):
        d = tx[i] - xs
        r = np.linalg.norm(d, axis=1); r[t] = np.inf           # the smooth rule skips the self node
        s_sm = (ws / r) @ dU / (4 * np.pi)
        d_sm = (ws * np.sum(d * ns, 1) / r ** 3) @ U / (4 * np.pi)
        sel = np.where(tg == i)[0]
        c_s = sum(vals[0][k] @ dU[pa[k] * n:(pa[k] + 1) * n] for k in sel)
        c_d = sum(vals[1][k] @ U[pa[k] * n:(pa[k] + 1) * n] for k in sel)
        res.append(abs(s_sm + c_s - d_sm - c_d - 0.5 * U[t]) / np.abs(U).max())
    return np.array(res)


def test_greens_identity_stellarator():
    r4, r8 = _green_residuals(4), _green_residuals(8)
    print("Green residuals p=4", r4, "p=8", r8)
    assert r8.max() < 2e-5
    assert np.median(r8) < np.median(r4) / 50
