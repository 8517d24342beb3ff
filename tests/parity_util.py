"""Shared helpers of the GPU parity tests: run the CUDA path through the C ABI and the oracle on the
same seeded inputs, and gate the GPU rows against an extended-precision truth.

The parity bar.  t = the oracle evaluated in IEEE binary128 (oracle/liboracle_q.so: same algorithm, same
fp64 inputs, ~34 digits), o = the fp64 oracle (round to nearest), o_m = the fp64 oracle run under each
IEEE rounding mode m in {nearest, up, down, toward zero}; s = max_m |o_m - t| (the rounding envelope of
an fp64 evaluation of this formulation).  For every CSR row r (a target's sampled pairs), with
M_r = max_i |t_i|, e_X(r) = max_i |X_i - t_i|:
  (a) per row:       e_g(r) <= ROW_FACTOR * s(r) + 1e-11 * M_r
  (b) distribution:  the median and 90th percentile of e_g / M over the rows are within Q_FACTOR of the
                     same quantiles of the fp64 oracle's e_o / M (+1e-13), and max e_g / M within
                     MAX_FACTOR of max e_o / M (+1e-11).
(a) catches an isolated defect in any row, (b) a systematic one at twice the rounding level.  Why not
"e_g <= 4 e_o per row": two correct fp64 builds of the oracle (no FMA vs FMA contraction) already violate
that on 2-8 % of the rows of configs 2-5 (max ratio 11; profiles/r02_parity_spread.txt), because e_o of a
single evaluation can be small by chance; the rounding-mode envelope does not have that failure mode
(FMA build vs envelope: worst per-row ratio 4.0 of ROW_FACTOR's 8 over cfg1-5)."""
import numpy as np
import torch

from oracle import oracle as O

MODES = ("nearest", "up", "down", "zero")
ROW_FACTOR = 8.0
Q_FACTOR = 2.0
MAX_FACTOR = 4.0
FLOOR_REL = 1e-11


def gpu_build(cfg, surf_np, targets, mask=15, raw=False, row_range=None):
    from paper_2411_08342_b200 import RRQ, DeviceSurface, DeviceTargets
    S = surf_np
    ctx = RRQ(S.p, eta=cfg["eta"] if np.isfinite(cfg["eta"]) else 0.0, all_pairs=cfg["all_pairs"])
    ds = DeviceSurface.from_numpy(S)
    dt = DeviceTargets.from_numpy(*targets)
    ptr, pat = ctx.near_list(ds, dt)
    fit, fst = ctx.patch_fit(ds)
    rb, re_ = row_range if row_range else (0, dt.n_targets)
    out = ctx.build_correction(ds, dt, ptr, pat, fit, mask=mask, raw=raw, row_begin=rb, row_end=re_)
    torch.cuda.synchronize()
    res = dict(ptr=ptr.cpu().numpy(), pat=pat.cpu().numpy(), fit=fit, fit_status=fst.cpu().numpy(),
               row_ptr=out["row_ptr"].cpu().numpy(), col=out["col_idx"].cpu().numpy(),
               vals=[v.cpu().numpy() if v is not None else None for v in out["vals"]],
               status=out["status"].cpu().numpy(), ctx=ctx)
    return res


def reference(S, tgs, tg, pa, mask=15, raw=False, zeta=False):
    """Truth (quad), the fp64 oracle (nearest) and the rounding envelope s = max_m |o_m - t| on the pairs
    (tg, pa).  tgs = (tx, tnormal, self_node, side)."""
    out = {}
    r = O.build_rows(S, *tgs, tg, pa, mask=mask, raw=raw, prec="q", zeta=zeta)
    out["t"], out["st_t"] = r[0], r[1]
    if zeta:
        out["zt"] = r[2]
    env = None
    zenv = None
    for m in MODES:
        r = O.build_rows(S, *tgs, tg, pa, mask=mask, raw=raw, prec="d", rounding=m, zeta=zeta)
        e = np.abs(r[0] - out["t"])
        env = e if env is None else np.maximum(env, e)
        if zeta:
            ez = np.abs(r[2] - out["zt"])
            zenv = ez if zenv is None else np.maximum(zenv, ez)
        if m == "nearest":
            out["o"], out["st_o"] = r[0], r[1]
            if zeta:
                out["zo"] = r[2]
    out["env"] = env
    if zeta:
        out["zenv"] = zenv
    return out


def _per_row(x, inv, R):
    y = np.zeros(R)
    np.maximum.at(y, inv, x)
    return y


def gate_rows(g, ref, k, inv, stats=None, tag=""):
    """Parity bar (a) + (b) of the module docstring for kernel k (0 S, 1 D, 2 S', 3 D').  g: [npairs, n] GPU
    values of the same pairs as ref; inv: row index of each pair (0..R-1).  Returns (ok, stats)."""
    t, o, env = ref["t"][k], ref["o"][k], ref["env"][k]
    npairs = t.shape[0]
    g = np.asarray(g).reshape(npairs, -1)
    st = {} if stats is None else stats
    if npairs == 0:
        return True, st
    R = int(inv.max()) + 1
    M = _per_row(np.abs(t).max(1), inv, R)
    eg = _per_row(np.abs(g - t).max(1), inv, R)
    eo = _per_row(np.abs(o - t).max(1), inv, R)
    s = _per_row(env.max(1), inv, R)
    bound = ROW_FACTOR * s + FLOOR_REL * M
    ratio = np.where(bound > 0, eg / np.where(bound > 0, bound, 1.0), np.where(eg > 0, np.inf, 0.0))
    ok_a = bool(np.all(ratio <= 1.0))
    nz = M > 0
    ok_b = True
    if nz.any():
        rg, ro = eg[nz] / M[nz], eo[nz] / M[nz]
        q = {}
        for qq in (50, 90):
            a, b = np.percentile(rg, qq), np.percentile(ro, qq)
            q[qq] = (float(a), float(b))
            ok_b &= bool(a <= Q_FACTOR * b + 1e-13)
        ok_b &= bool(rg.max() <= MAX_FACTOR * ro.max() + FLOOR_REL)
        st.update(rows=int(R), rows_nonzero=int(nz.sum()),
                  gpu_med=q[50][0], oracle_med=q[50][1], gpu_p90=q[90][0], oracle_p90=q[90][1],
                  gpu_max=float(rg.max()), oracle_max=float(ro.max()),
                  gpu_frac_1e11=float(np.mean(rg <= FLOOR_REL)), oracle_frac_1e11=float(np.mean(ro <= FLOOR_REL)))
    st.update(worst_row_ratio=float(ratio.max()), row_gate=ok_a, distribution_gate=ok_b)
    if tag:
        print(tag, "S D Sp Dp".split()[k], {a: (round(b, 4) if isinstance(b, float) and b > 1e-3 else b)
                                            for a, b in st.items()})
    return ok_a and ok_b, st


def gate_all(gvals, ref, inv, tag="", kernels=range(4)):
    """gvals[k]: [npairs, n] GPU values per kernel; asserts the bar for every kernel."""
    allst = {}
    bad = []
    for k in kernels:
        ok, st = gate_rows(gvals[k], ref, k, inv, tag=tag)
        allst["S D Sp Dp".split()[k]] = st
        if not ok:
            bad.append(("S D Sp Dp".split()[k], st))
    assert not bad, f"{tag}: parity bar failed: {bad}"
    return allst


def gate_zeta(zg, ref, tag=""):
    """Component-wise gate of the Steps 4-7 outputs (Theta, W, dW) of each pair against the truth:
    |z_g - z_t| <= ROW_FACTOR * s_z + 1e-14 * max|z_t of the pair's block| (s_z: rounding envelope)."""
    zt, zenv = ref["zt"], ref["zenv"]
    npairs, w = zt.shape
    npb = w // 9
    worst = 0.0
    for a, b in ((0, npb), (npb, 5 * npb), (5 * npb, 9 * npb)):
        scale = np.abs(zt[:, a:b]).max(1, keepdims=True)
        bound = ROW_FACTOR * zenv[:, a:b] + 1e-14 * scale
        err = np.abs(zg[:, a:b] - zt[:, a:b])
        r = np.where(bound > 0, err / np.where(bound > 0, bound, 1.0), np.where(err > 0, np.inf, 0.0))
        worst = max(worst, float(r.max()))
    if tag:
        print(tag, "zeta worst ratio", worst)
    return worst


def zeta_to_gpu_layout(z, npb):
    """Oracle zeta rows [Theta | W (np, 4) | dW (np, 4)] -> the C-ABI debug layout [Theta | zeta(W) | zeta(dW)]
    with zeta(X) = (X0, -X1, -X2, -X3) stacked over (l, m) in c-layout blocks (App. A.7)."""
    Th = z[:, :npb]
    W = z[:, npb:5 * npb].reshape(-1, npb, 4)
    dW = z[:, 5 * npb:9 * npb].reshape(-1, npb, 4)
    sg = np.array([1.0, -1.0, -1.0, -1.0])
    return np.concatenate([Th, (W * sg).transpose(0, 2, 1).reshape(-1, 4 * npb),
                           (dW * sg).transpose(0, 2, 1).reshape(-1, 4 * npb)], 1)


def zeta_env_to_gpu_layout(e, npb):
    """The same re-layout for a non-negative envelope (signs dropped)."""
    return np.abs(zeta_to_gpu_layout(e, npb))
