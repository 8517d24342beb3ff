"""Close-evaluation sweep of the oracle (north star's "twelve-digit close evaluation", P:L21, P:L209;
DESIGN.md §2.2): normal distances delta = 1e-1 .. 1e-14 h on both sides, over projections in the interior,
near an edge (lateral 1e-4 .. 1e-8 h, inside and outside) and near a vertex (1e-2 .. 1e-6 h), against the
independent mpmath truths of tests/close_truth.py, for the fp64 oracle and its binary128 build (the
method's own error, free of rounding).

    python tools/close_sweep.py > profiles/r02_close_sweep.txt
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from synth.geometry import make_flat_surface, make_cap_surface  # noqa: E402
import close_truth as CT  # noqa: E402
from test_oracle_close import FLAT_TRI, flat_families, cap_families  # noqa: E402

DELTAS = [10.0 ** -k for k in (1, 2, 4, 6, 8, 10, 12, 14)]


def flat(p):
    S = make_flat_surface([FLAT_TRI], p, 2 * p)
    h = max(np.linalg.norm(FLAT_TRI[i] - FLAT_TRI[(i + 1) % 3]) for i in range(3))
    print(f"== flat triangle, p = {p}, density 1: row sums vs closed forms "
          f"(S rel, D abs, S' abs, D' rel; max over the four)  columns: delta/h = " + " ".join(f"{d:.0e}" for d in DELTAS))
    for nm, (xy, ell) in flat_families(h).items():
        for sg in (1, -1):
            X = np.array([[xy[0], xy[1], sg * d * h] for d in DELTAS])
            T = len(X)
            args = (S, X, np.tile([0, 0, 1.0], (T, 1)), np.full(T, -1, np.int64), np.full(T, sg, np.int8),
                    np.arange(T, dtype=np.int64), np.zeros(T, np.int32))
            rows = {pr: O.build_rows(*args, raw=True, prec=pr)[0].sum(2) for pr in ("d", "q")}
            err = {pr: [] for pr in rows}
            for i in range(T):
                tr = CT.flat_truths(FLAT_TRI, X[i])
                for pr in rows:
                    e = [abs(rows[pr][k, i] - tr[key]) / (max(abs(tr[key]), 1.0) if key in ("S", "Dp") else 1.0)
                         for k, key in enumerate(("S", "D", "Sp", "Dp"))]
                    err[pr].append(max(e))
            for pr, lab in (("d", "fp64"), ("q", "quad")):
                print(f"  {nm:14s} side {sg:+d} {lab}: " + " ".join(f"{v:.0e}" for v in err[pr]))
        sys.stdout.flush()


def cap(p):
    S = make_cap_surface(0.2, p, 2 * p)
    v = S.verts[0]
    h = max(np.linalg.norm(v[i] - v[(i + 1) % 3]) for i in range(3))
    EC = CT.EdgeCurves(S.edge_x[0], S.edge_dx[0], S.verts[0])
    print(f"== unit-sphere cap (config 5 patch), p = {p}, density 1: Omega_0/4pi abs | dOmega_0/dnu' rel  columns: "
          "delta/h = " + " ".join(f"{d:.0e}" for d in DELTAS))
    for nm, (x0, ell) in cap_families(S, h).items():
        nrm = x0 / np.linalg.norm(x0)
        for sg in (1, -1):
            t0 = time.time()
            X = np.array([x0 + sg * d * h * nrm for d in DELTAS])
            NU = np.tile(nrm, (len(X), 1))
            res = {pr: O.pairs_debug(S, 0, X, NU, side=np.full(len(X), sg, np.int32), prec=pr) for pr in ("d", "q")}
            tr = [EC.solid_angle(X[i], NU[i], sg) for i in range(len(X))]
            for pr, lab in (("d", "fp64"), ("q", "quad")):
                e0 = [abs(res[pr]["Omega0"][i] - tr[i][0]) / (4 * np.pi) for i in range(len(X))]
                e1 = [abs(res[pr]["dOmega0"][i] / h - tr[i][1]) / max(1.0, abs(tr[i][1])) for i in range(len(X))]
                print(f"  {nm:14s} side {sg:+d} {lab}: " + " ".join(f"{v:.0e}" for v in e0) + "  | "
                      + " ".join(f"{v:.0e}" for v in e1) + (f"  ({time.time() - t0:.0f} s)" if pr == "q" else ""))
            sys.stdout.flush()


if __name__ == "__main__":
    flat(8)
    flat(10)
    cap(10)
