"""Pins of the oracle's singularity-swap building blocks (§2.4, §3.5
P:L1212-1258; readings A4, A5, A11, A12)."""
import json
import os

import mpmath as mp
import numpy as np
import pytest

from oracle import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")))


@pytest.mark.parametrize("q", [8, 12, 16, 20])
def test_gauss_legendre_and_vandermonde_inverse(q):
    t, w, U = O.tables(q)
    x, wx = np.polynomial.legendre.leggauss(q)
    assert np.abs(t - x).max() < 1e-15 and np.abs(w - wx).max() < 1e-14
    mp.mp.dps = 60
    for tk, wk in zip(t, w):   # nodes are roots of P_q and weights 2/((1-t^2) P_q'(t)^2), to 60 digits
        tt = mp.findroot(lambda s: mp.legendre(q, s), mp.mpf(float(tk)))
        assert float(tt) == tk
        dp = mp.diff(lambda s: mp.legendre(q, s), tt)
        assert float(2 / ((1 - tt ** 2) * dp ** 2)) == wk
    # U = V^{-1} correctly rounded: compare against an mpmath inverse (60 digits) of the same nodes
    Vm = mp.matrix([[mp.mpf(float(tk)) ** j for j in range(q)] for tk in t])
    Um = Vm ** -1
    for i in range(q):
        for k in range(q):
            assert U[i, k] == float(Um[i, k]), (i, k)


def _mp_model(a, b, k, m):
    mp.mp.dps = 40
    f = lambda t: t ** k / (((t - a) ** 2 + b ** 2) ** (mp.mpf(m) / 2))
    pts = [-1, 1]
    if -1 < a < 1:
        pts = [-1, a, 1]
    return float(mp.quad(f, pts))


@pytest.mark.parametrize("t0", [0.3 + 0.2j, -0.7 + 0.01j, 0.0 + 1.0j, 1.15 + 0.05j, -1.3 + 0.4j,
                                0.9 + 1e-4j])
def test_model_integrals_vs_mpmath(t0):
    q = 16
    I, J = O.model_integrals(t0.real, abs(t0.imag), q)
    for k in range(q):
        ri = _mp_model(t0.real, abs(t0.imag), k, 1)
        rj = _mp_model(t0.real, abs(t0.imag), k, 3)
        # scale: integral of |t|^k against the kernel (the recurrence's natural error scale, A5)
        si = _mp_model(0.0, abs(t0.imag) + abs(t0.real), 0, 1)
        sj = _mp_model(t0.real, abs(t0.imag), 0, 3)
        assert abs(I[k] - ri) <= 1e-11 * max(si, 1.0), (k, I[k], ri)
        assert abs(J[k] - rj) <= 1e-10 * max(sj, 1.0), (k, J[k], rj)


@pytest.mark.parametrize("t0", [0.15 + 1.17j, -1.6 + 1.3j, 1.8 + 0.8j, 1.3 + 0.01j, 0.0 + 2.0j])
def test_model_integrals_direct_rule_vs_mpmath(t0):
    """Reading A11': outside rho = 1.6 the model integrals come from a 48-point Gauss-Legendre rule."""
    q = 20
    assert O.bernstein_rho(t0) >= 1.6
    I, J = O.model_integrals_direct(t0.real, abs(t0.imag), q)
    for k in range(q):
        ri = _mp_model(t0.real, abs(t0.imag), k, 1)
        rj = _mp_model(t0.real, abs(t0.imag), k, 3)
        si = _mp_model(0.0, abs(t0.imag) + abs(t0.real), 0, 1)
        sj = _mp_model(t0.real, abs(t0.imag), 0, 3)
        assert abs(I[k] - ri) <= 1e-14 * max(si, 1.0), (k, I[k], ri)
        assert abs(J[k] - rj) <= 1e-14 * max(sj, 1.0), (k, J[k], rj)


def test_model_integral_closed_forms():
    I, J = O.model_integrals(0.0, 1.0, 8)
    assert abs(I[0] - GOLD["ssq_I0_t0_i"]["value"]) < 1e-15
    assert abs(I[1] - GOLD["ssq_I1_t0_i"]["value"]) < 1e-15
    assert abs(J[0] - np.sqrt(2.0)) < 1e-15      # int dt/(t^2+1)^{3/2} = [t/sqrt(t^2+1)] = sqrt 2
    # conjugate symmetry: only |Im t0| enters
    a1 = O.model_integrals(0.4, 0.3, 8); a2 = O.model_integrals(0.4, -0.3, 8)
    assert np.abs(a1[0] - O.model_integrals(0.4, 0.3, 8)[0]).max() == 0


def test_t0_straight_edge_closed_form():
    """r(t) = (t, 0, 0) (Legendre coefficient a_1 = e_x), target (0.3, d, 0) -> t0 = 0.3 + i d."""
    q = 12
    C = np.zeros((q, 3)); C[1, 0] = 1.0
    for d in (1e-12, 1e-6, 0.01, 0.3, 1.5):
        t0, conv = O.find_t0(C, np.array([0.3, d, 0.0]))
        assert conv and abs(t0 - (0.3 + 1j * d)) < 1e-14 * (1 + abs(t0))


def test_t0_curved_edge_is_a_root():
    """On a curved interpolated edge the returned t0 is a root of sum_c (x_c(t) - r'_c)^2."""
    q = 16
    t, w, U = O.tables(q)
    th = 0.4 * t
    y = np.stack([np.sin(th), 1 - np.cos(th), 0.1 * th ** 2], 1)
    C = np.polynomial.legendre.legfit(t, y, q - 1)      # Legendre coefficients (reading A4')
    rng = np.random.default_rng(4)
    for _ in range(20):
        tr = rng.uniform(-1.1, 1.1)
        rp = np.array([np.sin(0.4 * tr), 1 - np.cos(0.4 * tr), 0.1 * (0.4 * tr) ** 2]) + rng.normal(0, 0.05, 3)
        t0, conv = O.find_t0(C, rp)
        assert conv and t0.imag >= 0
        x = np.polynomial.legendre.legval(t0, C)
        assert abs(np.sum((x - rp) ** 2)) < 1e-13


def test_bernstein_regime():
    assert O.bernstein_rho(10j) > 3.0 and O.bernstein_rho(0.5 + 0.01j) < 3.0
    assert abs(O.bernstein_rho(2j) - (2 + np.sqrt(5))) < 1e-14
    assert abs(O.bernstein_rho(0.3 + 0j) - 1.0) < 1e-14


def test_ssq_integral_of_smooth_data_vs_mpmath():
    """Edge integral int F(t)/|t - t0|^m dt by the swap weights [M^T U]_k equals the
    30-digit mpmath integral (m = 1, 3); smooth F as in SURVEY App. B.8b."""
    q = 16
    t, w, U = O.tables(q)
    mp.mp.dps = 30
    for t0 in (0.2 + 1e-3j, -0.8 + 0.05j, 0.95 + 1e-6j, 0.1 + 0.6j):
        I, J = O.model_integrals(t0.real, abs(t0.imag), q)
        F = np.cos(2 * t) + t ** 3 + 0.3 * np.exp(t)
        val1 = (I @ U) @ F
        val3 = (J @ U) @ F
        f = lambda s, m: (mp.cos(2 * s) + s ** 3 + 0.3 * mp.exp(s)) / ((s - t0.real) ** 2 + t0.imag ** 2) ** (mp.mpf(m) / 2)
        pts = [-1, t0.real, 1] if -1 < t0.real < 1 else [-1, 1]
        r1 = float(mp.quad(lambda s: f(s, 1), pts))
        r3 = float(mp.quad(lambda s: f(s, 3), pts))
        assert abs(val1 - r1) < 2e-11 * abs(r1)
        assert abs(val3 - r3) < 2e-11 * abs(r3)
