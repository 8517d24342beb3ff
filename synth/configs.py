"""The five BASELINE.json workloads as seeded synthetic inputs (recipes: DESIGN.md §3).

One numpy Generator(PCG64) per config, seed = 2411083420 + cfg id, draws in the listed order.
`scale` arguments shrink the target counts for parity tests; the surfaces are always the named ones
unless `freq`/`p` overrides are given (used only by tests that need small cases).
"""
import math
import numpy as np
import torch

from .geometry import (make_sphere_surface, make_torus_surface, make_cap_surface, make_stellarator_surface,
                       make_interlocked_tori, inside_interlocked_tori,
                       bumpy_radius_fn, _eval_map, _radial_map)

CONFIG_SEEDS = {c: 2411083420 + c for c in range(1, 8)}


def patch_h(S):
    """h_P := max vertex chord; used only to place synthetic targets."""
    v = S.verts
    d = [np.linalg.norm(v[:, i] - v[:, (i + 1) % 3], axis=1) for i in range(3)]
    return np.max(np.stack(d, 1), 1)


def node_targets(S):
    P, n = S.n_patches, S.n
    x = S.nodes.reshape(-1, 3).copy()
    nu = S.normals.reshape(-1, 3).copy()
    self_node = np.arange(P * n, dtype=np.int64)
    side = np.zeros(P * n, dtype=np.int8)
    return x, nu, self_node, side


def offsurface_normal_targets(S, rng, count, exponents, sides=None):
    """Random node, displaced by side*10^e*h_P along its normal (the node's normal is the target's)."""
    P, n = S.n_patches, S.n
    h = patch_h(S)
    node = rng.integers(0, P * n, size=count)
    e = exponents(rng, count)
    if sides is None:
        sides = np.where(rng.random(count) < 0.5, -1, 1)
    pid = node // n
    x0 = S.nodes.reshape(-1, 3)[node]
    nu = S.normals.reshape(-1, 3)[node]
    x = x0 + (sides * 10.0 ** e * h[pid])[:, None] * nu
    return x, nu.copy(), np.full(count, -1, np.int64), sides.astype(np.int8)


def _assemble(S, parts, params):
    x = np.concatenate([p[0] for p in parts])
    nu = np.concatenate([p[1] for p in parts])
    sn = np.concatenate([p[2] for p in parts])
    sd = np.concatenate([p[3] for p in parts])
    return dict(surface=S, tx=np.ascontiguousarray(x), tnormal=np.ascontiguousarray(nu),
                self_node=sn, side=sd, **params)


def make_config(cfg, n_off=None, include_nodes=True, freq=None, p=None, seed_offset=0):
    """Return dict(surface, tx, tnormal, self_node, side, p, q, eta, all_pairs, name[, mask]); `mask` (kernel
    mask, default all four) is S|D for config 7, whose grid targets carry no normal."""
    rng = np.random.Generator(np.random.PCG64(CONFIG_SEEDS[cfg] + seed_offset))
    if cfg == 1:
        pp = p or 4
        S = make_sphere_surface(freq or 1, pp, 2 * pp)
        parts = [node_targets(S)] if include_nodes else []
        cnt = 1000 if n_off is None else n_off
        parts.append(offsurface_normal_targets(
            S, rng, cnt, lambda r, c: -r.integers(1, 9, size=c).astype(np.float64)))
        return _assemble(S, parts, dict(p=pp, q=2 * pp, eta=1.0, all_pairs=False, name=f"cfg1-sphere{S.n_patches}-p{pp}"))
    if cfg == 2:
        pp = p or 8
        S = make_sphere_surface(freq or 8, pp, 2 * pp)
        parts = [node_targets(S)] if include_nodes else []
        cnt = 100_000 if n_off is None else n_off
        P, n = S.n_patches, S.n
        h = patch_h(S)
        node = rng.integers(0, P * n, size=cnt)
        pid = node // n
        x0 = S.nodes.reshape(-1, 3)[node]
        # tangential offset uniform in a disk of radius 0.25 h_P, re-projected radially
        nu0 = x0 / np.linalg.norm(x0, axis=1, keepdims=True)
        a = rng.standard_normal((cnt, 3))
        t1 = a - np.sum(a * nu0, 1, keepdims=True) * nu0
        t1 /= np.linalg.norm(t1, axis=1, keepdims=True)
        rad = 0.25 * h[pid] * np.sqrt(rng.random(cnt))
        y = x0 + rad[:, None] * t1
        xs = y / np.linalg.norm(y, axis=1, keepdims=True)
        e = rng.uniform(-12.0, 0.0, size=cnt)
        sides = np.where(rng.random(cnt) < 0.5, -1, 1)
        x = xs * (1.0 + sides * 10.0 ** e * h[pid])[:, None]
        parts.append((x, xs.copy(), np.full(cnt, -1, np.int64), sides.astype(np.int8)))
        return _assemble(S, parts, dict(p=pp, q=2 * pp, eta=1.5, all_pairs=False, name=f"cfg2-sphere{S.n_patches}-p{pp}"))
    if cfg == 3:
        pp = p or 6
        nth, nph = (64, 80) if freq is None else freq
        S = make_torus_surface(2.0, 0.5, nth, nph, pp, 2 * pp)
        parts = [node_targets(S)] if include_nodes else []
        cnt = 500_000 if n_off is None else n_off
        h = patch_h(S)
        th = rng.uniform(0, 2 * np.pi, cnt)
        ph = rng.uniform(0, 2 * np.pi, cnt)
        e = rng.uniform(-10.0, math.log10(0.5), cnt)
        sides = np.where(rng.random(cnt) < 0.5, -1, 1)
        # patch containing (phi, theta): quad (i,j), lower/upper triangle by the diagonal
        i = np.minimum((ph / (2 * np.pi) * nph).astype(int), nph - 1)
        j = np.minimum((th / (2 * np.pi) * nth).astype(int), nth - 1)
        fu = ph / (2 * np.pi) * nph - i
        fv = th / (2 * np.pi) * nth - j
        pid = 2 * (i * nth + j) + (fv > fu)
        rho = 2.0 + 0.5 * np.cos(th)
        x0 = np.stack([rho * np.cos(ph), rho * np.sin(ph), 0.5 * np.sin(th)], 1)
        nu = np.stack([np.cos(th) * np.cos(ph), np.cos(th) * np.sin(ph), np.sin(th)], 1)
        x = x0 + (sides * 10.0 ** e * h[pid])[:, None] * nu
        parts.append((x, nu, np.full(cnt, -1, np.int64), sides.astype(np.int8)))
        return _assemble(S, parts, dict(p=pp, q=2 * pp, eta=1.5, all_pairs=False, name=f"cfg3-torus{S.n_patches}-p{pp}"))
    if cfg == 4:
        pp = p or 8
        while True:
            coef = {}
            for l in range(1, 7):
                for m in range(-l, l + 1):
                    coef[(l, m)] = rng.standard_normal() / l
            rf = bumpy_radius_fn(coef)
            test = torch.as_tensor(rng.standard_normal((20000, 3)))
            test = test / torch.linalg.norm(test, dim=1, keepdim=True)
            if float(rf(test).min()) >= 0.5:
                break
        S = make_sphere_surface(freq or 50, pp, 2 * pp, radius_fn=rf)
        parts = [node_targets(S)] if include_nodes else []
        cnt = 1_000_000 if n_off is None else n_off
        sides = np.where(np.arange(cnt) < cnt // 2, -1, 1)
        sides = rng.permutation(sides)
        parts.append(offsurface_normal_targets(S, rng, cnt, lambda r, c: r.uniform(-12.0, 0.0, c), sides))
        return _assemble(S, parts, dict(p=pp, q=2 * pp, eta=1.5, all_pairs=False, name=f"cfg4-bumpy{S.n_patches}-p{pp}"))
    if cfg == 5:
        pp = p or 10
        chord = 0.2
        S = make_cap_surface(chord, pp, 2 * pp)
        cnt = 10_000_000 if n_off is None else n_off
        v = S.pdata.reshape(3, 3)
        lo, hi = v[:, :2].min(0), v[:, :2].max(0)
        ctr, half = (lo + hi) / 2, (hi - lo) / 2
        ab = ctr + 3.0 * half * rng.uniform(-1.0, 1.0, (cnt, 2))
        qd = np.concatenate([ab, np.ones((cnt, 1))], 1)
        qd /= np.linalg.norm(qd, axis=1, keepdims=True)
        sides = np.where(rng.random(cnt) < 0.5, -1, 1)
        d = 10.0 ** rng.uniform(-14.0, math.log10(2 * chord), cnt)
        x = qd * (1.0 + sides * d)[:, None]
        parts = [(x, qd.copy(), np.full(cnt, -1, np.int64), sides.astype(np.int8))]
        return _assemble(S, parts, dict(p=pp, q=2 * pp, eta=float("inf"), all_pairs=True, name="cfg5-cap-p10"))
    if cfg == 6:
        # SURVEY §8(f) NEXT(1), the paper's solve-phase throughput workload (E3): the
        # stellarator of eq (stellarator), n_u x n_v rectangles halved, on-surface node targets only
        # (Table 3's X_RRQ = N / T_RRQ counts all discretisation points); n_off adds off-surface targets
        pp = p or 8
        nu_, nv_ = (16, 48) if freq is None else freq
        S = make_stellarator_surface(nu_, nv_, pp, 2 * pp)
        parts = [node_targets(S)] if include_nodes else []
        if n_off:
            parts.append(offsurface_normal_targets(S, rng, n_off, lambda r, c: r.uniform(-12.0, 0.0, c)))
        return _assemble(S, parts, dict(p=pp, q=2 * pp, eta=1.5, all_pairs=False,
                                        name=f"cfg6-stellarator{S.n_patches}-p{pp}"))
    if cfg == 7:
        # SURVEY §8(f) NEXT(2), the paper's evaluation-phase workload (E4): four interlocking
        # tori (a = 3, b = 0.5, 4.95 apart), each n_theta x n_phi rectangles halved, and the exterior points
        # of a uniform G^3 grid over the box [-5,20] x [-6,6]^2 with G = 1 + 100 n_theta / 6 (the paper's
        # pairing 6x36 <-> 101^3 ... 24x144 <-> 401^3).  No target normals (u itself: S and D; S', D' rows are
        # then zero).  Close targets are those the near rule (A6) pairs with some patch.
        pp = p or 8
        nth, nph = (6, 36) if freq is None else freq
        S = make_interlocked_tori(nth, nph, pp, 2 * pp)
        G = int(round(1 + 100 * nth / 6)) if n_off is None else int(n_off)
        gx = np.linspace(-5.0, 20.0, G); gy = np.linspace(-6.0, 6.0, G)
        X = np.stack(np.meshgrid(gx, gy, gy, indexing="ij"), -1).reshape(-1, 3)
        X = X[~inside_interlocked_tori(X)]
        cnt = X.shape[0]
        parts = [(X, np.zeros_like(X), np.full(cnt, -1, np.int64), np.ones(cnt, np.int8))]
        return _assemble(S, parts, dict(p=pp, q=2 * pp, eta=1.5, all_pairs=False, mask=3,
                                        name=f"cfg7-tori{S.n_patches}-grid{G}-p{pp}"))
    raise ValueError(cfg)
