"""Pins of the oracle's harmonic building blocks (§2.3; §3.2)."""
import json
import math
import os

import numpy as np
import pytest
import scipy.special as sps

from oracle import oracle as O
import indep

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")))


def test_legendre_vs_scipy_textbook():
    # scipy's lpmv carries the Condon-Shortley phase; the paper drops it (reading G5)
    for x in (-0.93, -0.3, 0.0, 0.41, 0.999):
        P = O.legendre(10, x)
        for l in range(11):
            for m in range(l + 1):
                ref = (-1) ** m * sps.lpmv(m, l, x)
                assert abs(P[l, m] - ref) <= 1e-12 * max(1.0, abs(ref)), (l, m, x)
    assert abs(O.legendre(2, 0.5)[2, 0] - GOLD["P20_at_half"]["value"]) < 1e-15
    assert abs(O.legendre(1, 0.0)[1, 1] - GOLD["P11_at_0_noCS"]["value"]) < 1e-15


def test_solid_harmonics_vs_explicit_cartesian_formula():
    """R_l^m against the independent sympy polynomial of P:L573-587 (values, gradient, Hessian)."""
    p = 6
    f = indep.S_funcs(p, hess=True)
    rng = np.random.default_rng(1)
    for _ in range(6):
        x, y, z = rng.uniform(-1.2, 1.2, 3)
        S, G, H = O.harmonics_S(p, x, y, z)
        Si, Gi, Hi = f(x, y, z)
        assert np.abs(S - Si[:, 0]).max() < 1e-13
        assert np.abs(G - Gi[:, :, 0]).max() < 1e-12
        assert np.abs(H - Hi[:, :, :, 0]).max() < 1e-11
    # the origin and the polar axis (no trig shortcuts break there)
    for pt in [(0.0, 0.0, 0.0), (0.0, 0.0, 0.7), (0.3, 0.0, 0.0)]:
        S, G, H = O.harmonics_S(p, *pt)
        Si, Gi, Hi = f(*pt)
        assert np.abs(S - Si[:, 0]).max() < 1e-13 and np.abs(G - Gi[:, :, 0]).max() < 1e-12


def test_homogeneity_symmetry_and_low_order():
    p = 8
    R1 = O.solid_R(p, 0.3, -0.2, 0.7)
    R2 = O.solid_R(p, 0.6, -0.4, 1.4)
    for l in range(p + 1):
        for m in range(-l, l + 1):
            k = l * l + l + m
            assert abs(R2[k] - 2 ** l * R1[k]) <= 1e-13 * max(1, abs(R2[k]))
            km = l * l + l - m
            assert abs(R1[km] - (-1) ** m * np.conj(R1[k])) < 1e-15
    assert abs(R1[0] - 1) < 1e-16 and abs(R1[2] - 0.7) < 1e-16   # R_0^0 = 1, R_1^0 = z


def test_addition_theorem():
    """R_l^m(a+b) = sum_j sum_k R_j^k(a) R_{l-j}^{m-k}(b) T_{jk,lm} (eq l2ltranslation)."""
    p = 7
    rng = np.random.default_rng(2)
    a = rng.uniform(-0.6, 0.6, 3); b = rng.uniform(-0.6, 0.6, 3)
    Ra, Rb, Rab = O.solid_R(p, *a), O.solid_R(p, *b), O.solid_R(p, *(a + b))
    def g(R, l, m):
        return R[l * l + l + m] if abs(m) <= l else 0.0
    def T(j, k, l, m):
        def C(n, r):
            return math.comb(n, r) if 0 <= r <= n and n >= 0 else 0
        return math.sqrt(C(l + m, j + k) * C(l - m, j - k))
    assert abs(T(1, 1, 2, 2) - GOLD["T_11_22"]["value"]) < 1e-15
    for l in range(p + 1):
        for m in range(-l, l + 1):
            s = sum(g(Ra, j, k) * g(Rb, l - j, m - k) * T(j, k, l, m)
                    for j in range(l + 1) for k in range(-j, j + 1))
            assert abs(s - g(Rab, l, m)) < 1e-13, (l, m)


def test_H11_is_z_and_flat_gradients():
    """H^{(l,m)} = sqrt2 Im S^{(l,m)}: H^{(1,1)} = z; dH/dx = dH/dy = 0 on z = 0."""
    p = 8
    rng = np.random.default_rng(3)
    for _ in range(5):
        x, y, z = rng.uniform(-1, 1, 3)
        S, G, _ = O.harmonics_S(p, x, y, z, hess=False)
        assert abs(np.sqrt(2) * S[1 * 1 + 1 + 1].imag - z) < 1e-15
        S, G, _ = O.harmonics_S(p, x, y, 0.0, hess=False)
        for l in range(1, p + 1):
            for m in range(1, l + 1):
                gH = np.sqrt(2) * G[l * l + l + m].imag
                assert abs(gH[0]) < 1e-13 and abs(gH[1]) < 1e-13


@pytest.mark.parametrize("p", [4, 8, 10])
def test_theorem_3_1_flat_basis_complete(p):
    """span{dH/dz |_{z=0}} = polynomials of degree <= p-1 (Theorem 3.1)."""
    rng = np.random.default_rng(p)
    pts = rng.uniform(-0.5, 0.5, (3 * p * p, 2))
    F = []
    for x, y in pts:
        S, G, _ = O.harmonics_S(p, x, y, 0.0, hess=False)
        F.append([np.sqrt(2) * G[l * l + l + m][2].imag for l in range(1, p + 1) for m in range(1, l + 1)])
    F = np.array(F)
    mono = np.array([[x ** i * y ** j for i in range(p) for j in range(p - i)] for x, y in pts])
    npb = p * (p + 1) // 2
    assert np.linalg.matrix_rank(F, tol=1e-9 * np.abs(F).max()) == npb
    assert np.linalg.matrix_rank(np.hstack([F / np.abs(F).max(), mono / np.abs(mono).max()]), tol=1e-9) == npb


def test_quaternion_product():
    """qprule: ij = k, ji = -k, |fg| = |f||g|, associativity."""
    assert np.allclose(O.qmul([0, 1, 0, 0], [0, 0, 1, 0]), [0, 0, 0, 1])
    assert np.allclose(O.qmul([0, 0, 1, 0], [0, 1, 0, 0]), [0, 0, 0, -1])
    rng = np.random.default_rng(5)
    def ham(a, b):   # 16-term Hamilton expansion
        a0, a1, a2, a3 = a; b0, b1, b2, b3 = b
        return np.array([a0*b0 - a1*b1 - a2*b2 - a3*b3, a0*b1 + a1*b0 + a2*b3 - a3*b2,
                         a0*b2 - a1*b3 + a2*b0 + a3*b1, a0*b3 + a1*b2 - a2*b1 + a3*b0])
    for _ in range(20):
        f, g, h = rng.standard_normal((3, 4))
        fg = O.qmul(f, g)
        assert np.allclose(fg, ham(f, g), atol=1e-15)
        assert abs(np.linalg.norm(fg) - np.linalg.norm(f) * np.linalg.norm(g)) < 1e-13
        assert np.allclose(O.qmul(fg, h), O.qmul(f, O.qmul(g, h)), atol=1e-13)


def test_pinv_qr_vs_svd():
    rng = np.random.default_rng(7)
    A = rng.standard_normal((40, 17))
    Ap, st = O.pinv_qr(A)
    assert st == 0
    assert np.abs(Ap - np.linalg.pinv(A)).max() < 1e-12
