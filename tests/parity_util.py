"""Shared helpers of the GPU parity tests: run the CUDA path through the C ABI and the oracle on the
same seeded inputs, compare CSR rows element by element (DESIGN.md §5 parity bar)."""
import numpy as np
import torch

from oracle import oracle as O


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


def compare_rows(g_vals, o_vals, pair_target, n, rel=1e-11, abs_=1e-13, band=None):
    """Per CSR row (target): |g - o| <= max(rel * max|o_row|, abs_).
    g_vals/o_vals: [n_pairs*n] for one kernel, ordered like the pairs; pair_target [n_pairs].
    band: optional per-pair relaxation factor (conditioning band).  Returns (worst ratio, n rows)."""
    npairs = pair_target.shape[0]
    g = g_vals[: npairs * n].reshape(npairs, n)
    o = o_vals.reshape(npairs, n)
    T = int(pair_target.max()) + 1 if npairs else 0
    rowmax = np.zeros(T)
    np.maximum.at(rowmax, pair_target, np.abs(o).max(1))
    tol = np.maximum(rel * rowmax[pair_target], abs_)
    if band is not None:
        tol = tol * band
    ratio = (np.abs(g - o).max(1) / tol)
    return float(ratio.max()) if npairs else 0.0, ratio
