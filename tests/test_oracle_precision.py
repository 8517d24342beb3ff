"""Pins of the extended-precision truth reference (oracle/liboracle_q.so, binary128) and of the parity bar
built on it (tests/parity_util.py).

The truth is the same source as the fp64 oracle compiled with `real` = __float128, so it is pinned like
the oracle itself (brute-force 2-form integrals, Gauss law) and by the precision ladder: fp64, x87 long
double and binary128 evaluations of the same rows must converge (each step shrinking the error by about
the ratio of the unit roundoffs), and agree with one another to rounding where the rows are well
conditioned (config 1, p = 4)."""
import numpy as np
import pytest

from oracle import oracle as O
from synth.configs import make_config
from synth.geometry import make_sphere_surface
import parity_util as U


def _has_fma():
    try:
        with open("/proc/cpuinfo") as f:
            return " fma" in f.read()
    except OSError:
        return False


def _sample(cfgid, npatch, maxpairs, seed=0, **kw):
    cfg = make_config(cfgid, **kw)
    S = cfg["surface"]
    rng = np.random.default_rng(seed)
    patches = rng.choice(S.n_patches, size=min(npatch, S.n_patches), replace=False)
    tgs = (cfg["tx"], cfg["tnormal"], cfg["self_node"], cfg["side"])
    tg, pa = O.near_pairs_for_patches(S, tgs[0], tgs[2], cfg["eta"], patches, all_pairs=cfg["all_pairs"])
    if tg.size > maxpairs:
        sel = np.sort(rng.choice(tg.size, maxpairs, replace=False))
        tg, pa = tg[sel], pa[sel]
    return S, tgs, tg, pa


def _row_err(v, t, inv):
    R = inv.max() + 1
    e = np.zeros(R); M = np.zeros(R)
    np.maximum.at(e, inv, np.abs(v - t).max(1))
    np.maximum.at(M, inv, np.abs(t).max(1))
    return e, M


def test_well_conditioned_rows_agree_across_precisions():
    """Config 1 (p = 4): the rows of fp64, long double and binary128 agree to the rounding level of each
    (median row ~1e-16; the worst rows are targets 1e-8 h above a node, where the smooth subtraction of
    P:L1581-1598 is itself the ill-conditioned step).  (The
    Newton status bits may differ: an fp64 iteration that stalls at its rounding floor above the tolerance
    for a far root is flagged and takes the plain rule, which the converged root selects anyway.)"""
    S, tgs, tg, pa = _sample(1, 4, 2000, n_off=200)
    vq, _ = O.build_rows(S, *tgs, tg, pa, prec="q")
    vd, _ = O.build_rows(S, *tgs, tg, pa, prec="d")
    vl, _ = O.build_rows(S, *tgs, tg, pa, prec="ld")
    inv = np.unique(tg, return_inverse=True)[1]
    for k in range(4):
        ed, M = _row_err(vd[k], vq[k], inv)
        el, _ = _row_err(vl[k], vq[k], inv)
        rd, rl = ed / M, el / M
        print(k, np.median(rd), rd.max(), np.median(rl), rl.max())
        assert np.median(rd) < 1e-11 and rd.max() < 1e-10, (k, np.median(rd), rd.max())
        assert np.median(rl) < 1e-2 * np.median(rd) and rl.max() < 1e-2 * rd.max(), (k, np.median(rl), rl.max())


def test_precision_ladder_converges():
    """Config 2 (p = 8), where the correction rows are ill-conditioned (median row loses ~9 digits in fp64):
    long double (64-bit significand) must be ~2^11 more accurate than fp64 against the binary128 truth."""
    S, tgs, tg, pa = _sample(2, 2, 300)
    vq, _ = O.build_rows(S, *tgs, tg, pa, prec="q")
    vd, _ = O.build_rows(S, *tgs, tg, pa, prec="d")
    vl, _ = O.build_rows(S, *tgs, tg, pa, prec="ld")
    inv = np.unique(tg, return_inverse=True)[1]
    for k in range(4):
        ed, M = _row_err(vd[k], vq[k], inv)
        el, _ = _row_err(vl[k], vq[k], inv)
        rd, rl = np.median(ed / M), np.median(el / M)
        print(k, rd, rl)
        assert rl < rd / 200, (k, rd, rl)
        assert np.max(el / M) < np.max(ed / M) / 50


def test_truth_gauss_law_and_fit():
    """Gauss law D[1] = -1/2 (PV), -1 inside, 0 outside on a 320-patch sphere at p = 6 in
    binary128: the same discretisation bound as the fp64 oracle's pin (tests/test_oracle_operator.py)."""
    S = make_sphere_surface(4, 6, 12)
    x0 = S.nodes[3, 5]
    tx = np.array([x0, 0.6 * x0, 1.4 * x0])
    nu = np.tile(x0, (3, 1))
    sn = np.array([3 * S.n + 5, -1, -1], np.int64)
    sd = np.array([0, -1, 1], np.int8)
    tg = np.repeat(np.arange(3), S.n_patches).astype(np.int64)
    pa = np.tile(np.arange(S.n_patches), 3).astype(np.int32)
    vals, st = O.build_rows(S, tx, nu, sn, sd, tg, pa, raw=True, prec="q")
    assert (st & 6).max() == 0      # finite, full-rank fits (bit 0: far-root Newton stops, plain rule anyway)
    D1 = vals[1].reshape(3, -1).sum(1)
    assert np.abs(D1 - np.array([-0.5, -1.0, 0.0])).max() < 1e-9, D1


def test_truth_fit_is_the_unique_least_squares_operator():
    """The binary128 fit operators agree with the fp64 ones to the fp64 rounding of a unique operator."""
    cfg = make_config(1, n_off=10)
    S = cfg["surface"]
    fq, _ = O.patch_fit(S, prec="q")
    fd, _ = O.patch_fit(S, prec="d")
    for i in range(S.n_patches):
        assert np.abs(fd[i] - fq[i]).max() <= 1e-13 * np.abs(fq[i]).max()


@pytest.mark.skipif(not _has_fma(), reason="host CPU has no FMA")
def test_parity_bar_admits_a_second_fp64_build_and_rejects_defects():
    """The bar of tests/parity_util.py on config 3 (p = 6): the oracle built with FMA contraction (a correct
    fp64 evaluation with a different rounding) passes; a row with an error 10x its bound, and every row
    carrying 3x the fp64 oracle's own error (a systematic defect at the rounding level), fail."""
    S, tgs, tg, pa = _sample(3, 3, 500)
    ref = U.reference(S, tgs, tg, pa)
    vf, _ = O.build_rows(S, *tgs, tg, pa, prec="fma")
    inv = np.unique(tg, return_inverse=True)[1]
    for k in range(4):
        ok, st = U.gate_rows(vf[k], ref, k, inv)
        assert ok, (k, st)
        assert st["worst_row_ratio"] < 0.5
        # isolated defect in one row
        bad = vf[k].copy()
        j = int(np.argmax(np.abs(ref["t"][k]).max(1)))
        bound = U.ROW_FACTOR * ref["env"][k][inv == inv[j]].max() + U.FLOOR_REL * np.abs(ref["t"][k][inv == inv[j]]).max()
        bad[j, 0] = ref["t"][k][j, 0] + 10 * bound
        assert not U.gate_rows(bad, ref, k, inv)[0]
        # systematic defect: 3x the fp64 error everywhere
        sysd = ref["t"][k] + 3 * (ref["o"][k] - ref["t"][k])
        assert not U.gate_rows(sysd, ref, k, inv)[0]
