"""Independent reference constructions used to PIN the oracle (test-only; never imported by it).

* Solid harmonics from the explicit Cartesian formula of PAPER.md P:L573-587,
  R_l^m = sqrt((l-m)!/(l+m)!) Pi_l^m(z, r) (x + i y)^m with
  Pi_l^m = sum_k gamma_lk^(m) r^{2k} z^{l-2k-m},
  gamma_lk^(m) = (-1)^k 2^{-l} C(l,k) C(2l-2k,l) (l-2k)!/(l-2k-m)!,
  built as exact sympy polynomials and differentiated symbolically (a different route from the
  oracle's Legendre recurrence + derivative rules).
* An adaptive (4-way refinement) triangle quadrature for 2-form surface integrals over the exact
  patch map (brute force of SURVEY §8(c) "What pins each part").
"""
import functools
import math

import numpy as np
import sympy as sp

_x, _y, _z = sp.symbols("x y z", real=True)


@functools.lru_cache(maxsize=None)
def R_poly(l, m):
    """R_l^m(x,y,z) as a sympy expression (no Condon-Shortley phase), any -l<=m<=l."""
    if m < 0:
        return sp.expand((-1) ** (-m) * sp.conjugate(R_poly(l, -m)))
    r2 = _x ** 2 + _y ** 2 + _z ** 2
    Pi = 0
    for k in range((l - m) // 2 + 1):
        g = sp.Rational((-1) ** k, 2 ** l) * sp.binomial(l, k) * sp.binomial(2 * l - 2 * k, l) * \
            sp.factorial(l - 2 * k) / sp.factorial(l - 2 * k - m)
        Pi += g * r2 ** k * _z ** (l - 2 * k - m)
    N = sp.sqrt(sp.factorial(l - m) / sp.factorial(l + m))
    return sp.expand(N * Pi * (_x + sp.I * _y) ** m)


@functools.lru_cache(maxsize=None)
def S_funcs(p, hess=False):
    """Lambdified S^{(l,m)}(x,y,z) = R_l^m(y,z,x), gradient (and Hessian) for 0<=l<=p, all m.
    Returns f(x,y,z) -> (S [L,N], G [L,3,N], H [L,3,3,N] or None) with L = (p+1)^2, index l*l+l+m."""
    exprs = []
    for l in range(p + 1):
        for m in range(-l, l + 1):
            R = R_poly(l, m)
            S = R.subs({_x: _y, _y: _z, _z: _x}, simultaneous=True)
            exprs.append(S)
    grads = [[sp.diff(S, v) for v in (_x, _y, _z)] for S in exprs]
    f_S = sp.lambdify((_x, _y, _z), exprs, "numpy")
    f_G = sp.lambdify((_x, _y, _z), grads, "numpy")
    f_H = None
    if hess:
        hs = [[[sp.diff(g, v) for v in (_x, _y, _z)] for g in gr] for gr in grads]
        f_H = sp.lambdify((_x, _y, _z), hs, "numpy")

    def bc(v, N):
        a = np.asarray(v, dtype=np.complex128)
        return np.broadcast_to(a, (N,)) if a.ndim == 0 else a

    def f(x, y, z):
        x = np.atleast_1d(np.asarray(x, np.float64))
        y = np.atleast_1d(np.asarray(y, np.float64))
        z = np.atleast_1d(np.asarray(z, np.float64))
        N = x.size
        S = np.array([bc(v, N) for v in f_S(x, y, z)])
        G = np.array([[bc(v, N) for v in g] for g in f_G(x, y, z)])
        H = None
        if f_H is not None:
            H = np.array([[[bc(v, N) for v in r] for r in hh] for hh in f_H(x, y, z)])
        return S, G, H
    return f


def hidx(l, m):
    return l * l + l + m


# --------------------------------------------------------------------------- adaptive quadrature

def _tri_rule(k):
    """Collapsed k x k Gauss-Legendre rule on the reference triangle: (u, v) -> (s, t), weights."""
    x, w = np.polynomial.legendre.leggauss(k)
    x = (x + 1) / 2; w = w / 2
    U, V = np.meshgrid(x, x, indexing="ij")
    WU, WV = np.meshgrid(w, w, indexing="ij")
    s = U.ravel(); t = (V * (1 - U)).ravel(); ww = (WU * WV * (1 - U)).ravel()
    return s, t, ww


def adaptive_triangle(f, tol=1e-13, k_lo=10, k_hi=14, max_tris=400000):
    """Integrate vector-valued f(s, t) -> [N, C] over the reference triangle (0,0),(1,0),(0,1).
    4-way subdivision of triangles whose two rules differ by more than tol*area fraction."""
    rl = _tri_rule(k_lo); rh = _tri_rule(k_hi)
    tris = np.array([[[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]]])
    total = None
    scale0 = None
    while len(tris):
        A, B, C = tris[:, 0], tris[:, 1], tris[:, 2]
        area2 = np.abs((B[:, 0] - A[:, 0]) * (C[:, 1] - A[:, 1]) - (C[:, 0] - A[:, 0]) * (B[:, 1] - A[:, 1]))

        def apply(rule):
            s, t, w = rule
            S = A[:, None, 0] + s[None] * (B - A)[:, None, 0] + t[None] * (C - A)[:, None, 0]
            T = A[:, None, 1] + s[None] * (B - A)[:, None, 1] + t[None] * (C - A)[:, None, 1]
            vals = f(S.ravel(), T.ravel())
            vals = vals.reshape(len(tris), len(s), -1)
            return np.einsum("nkc,k->nc", vals, w) * area2[:, None]
        lo = apply(rl); hi = apply(rh)
        err = np.max(np.abs(hi - lo), axis=1)
        ok = err <= tol * np.maximum(area2 / 1.0, 1e-300) * 0.5 + 1e-300
        if scale0 is None:
            scale0 = np.abs(hi).max()
        ok |= err <= 1e-16 * scale0                             # rounding floor
        ok |= area2 < 1e-14
        acc = hi[ok].sum(0)
        total = acc if total is None else total + acc
        bad = tris[~ok]
        if len(bad) == 0:
            break
        if len(bad) * 4 > max_tris:
            raise RuntimeError("adaptive_triangle: too many triangles")
        A, B, C = bad[:, 0], bad[:, 1], bad[:, 2]
        ab, bc_, ca = (A + B) / 2, (B + C) / 2, (C + A) / 2
        tris = np.concatenate([np.stack([A, ab, ca], 1), np.stack([ab, B, bc_], 1),
                               np.stack([ca, bc_, C], 1), np.stack([ab, bc_, ca], 1)])
    return total


def vos_solid_angle(v0, v1, v2, r):
    """Van Oosterom-Strackee signed solid angle of the flat triangle (v0,v1,v2) seen from r:
    int (x - r).nu / |x - r|^3 da with nu along (v1-v0)x(v2-v0)."""
    R1, R2, R3 = v0 - r, v1 - r, v2 - r
    n1, n2, n3 = np.linalg.norm(R1), np.linalg.norm(R2), np.linalg.norm(R3)
    num = np.dot(R1, np.cross(R2, R3))
    den = n1 * n2 * n3 + np.dot(R1, R2) * n3 + np.dot(R1, R3) * n2 + np.dot(R2, R3) * n1
    return 2 * math.atan2(num, den)
