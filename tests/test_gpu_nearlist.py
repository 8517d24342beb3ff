"""Full-size near-list equality ("agree exactly" with a brute-force scan, reading
A6): every (target, patch) pair of BASELINE.json config 4 (50,000 patches, 4.2M targets, 143M pairs) from the
GPU against an independent construction: patch balls in numpy with the same sequence of separately rounded
IEEE operations (the near decision is taken in one fixed arithmetic on both sides), candidate
targets from a scipy k-d tree per patch (query radius inflated by 1e-12 relative: a superset), then the exact
test |t - c_P| <= R_P + eta h_P."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
from scipy.spatial import cKDTree

from synth.configs import make_config

pytestmark = pytest.mark.gpu


def _balls_numpy(S):
    """Sequential sums over the nodes, each product/sum a separate (correctly rounded) numpy ufunc."""
    P, n = S.weights.shape
    c = np.zeros((P, 3)); ws = np.zeros(P)
    for i in range(n):
        w = S.weights[:, i]
        ws = ws + w
        c = c + w[:, None] * S.nodes[:, i, :]
    c = c / ws[:, None]

    def nrm(d):
        return np.sqrt((d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2])
    pts = np.concatenate([S.nodes, S.verts, S.edge_x.reshape(P, -1, 3)], 1)
    R = nrm(pts - c[:, None, :]).max(1)
    v = S.verts
    h = np.maximum(np.maximum(nrm(v[:, 1] - v[:, 0]), nrm(v[:, 2] - v[:, 1])), nrm(v[:, 0] - v[:, 2]))
    return c, R, h


def test_cfg4_near_list_equals_kdtree_exactly():
    from paper_2411_08342_b200 import RRQ, DeviceSurface, DeviceTargets
    cfg = make_config(4)
    S = cfg["surface"]
    tx, sn, eta = cfg["tx"], cfg["self_node"], cfg["eta"]
    ctx = RRQ(S.p, eta=eta)
    ptr, pat = ctx.near_list(DeviceSurface.from_numpy(S), DeviceTargets.from_numpy(tx, cfg["tnormal"], sn, cfg["side"]))
    ptr, pat = ptr.cpu().numpy(), pat.cpu().numpy()
    T = tx.shape[0]
    # GPU pairs grouped by patch: (patch, target) sorted
    tg = np.repeat(np.arange(T, dtype=np.int64), np.diff(ptr))
    order = np.lexsort((tg, pat))
    gp, gt = pat[order], tg[order]
    bounds = np.searchsorted(gp, np.arange(S.n_patches + 1))
    c, R, h = _balls_numpy(S)
    rad = R + eta * h
    tree = cKDTree(tx)
    selfP = np.where(sn >= 0, sn // S.n, -1)
    npairs = 0
    for P0 in range(0, S.n_patches, 2000):
        Ps = np.arange(P0, min(P0 + 2000, S.n_patches))
        cand = tree.query_ball_point(c[Ps], rad[Ps] * (1 + 1e-12), return_sorted=True)
        for j, P in enumerate(Ps):
            t = np.asarray(cand[j], np.int64)
            d = tx[t] - c[P]
            dist = np.sqrt((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2])
            keep = (dist <= rad[P]) | (selfP[t] == P)   # a node of P is always within R_P (A6 self rule)
            ref = t[keep]
            got = gt[bounds[P]:bounds[P + 1]]
            assert np.array_equal(got, np.sort(ref)), (P, got.size, ref.size, np.setxor1d(got, ref)[:10])
            npairs += ref.size
    assert npairs == pat.size == ptr[-1]
    print(f"cfg4 near list: {npairs} pairs of {T} targets x {S.n_patches} patches equal the k-d tree construction")
