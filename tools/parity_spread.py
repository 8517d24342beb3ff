"""Measure what an fp64 evaluation of the RRQ correction rows can attain, against the binary128 truth
(DESIGN.md §5).  Calls only oracle/ (test infrastructure): for a seeded sample of near pairs per config it
evaluates the rows in binary128 (truth t), in fp64 under the four IEEE rounding modes, with FMA
contraction (a second correct fp64 rounding, standing in for "another implementation") and in long
double; prints per kernel the row-error quantiles relative to the row max, and how the FMA build fares
under (i) the per-row gate e <= 4 e_o + 1e-11 M and (ii) the parity bar of tests/parity_util.py.

    python tools/parity_spread.py [cfg ...] > profiles/r02_parity_spread.txt
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from synth.configs import make_config  # noqa: E402
import parity_util as U  # noqa: E402

SAMPLE = {1: (20, 10 ** 6), 2: (4, 1200), 3: (6, 1500), 4: (6, 2000), 5: (1, 1200), 6: (6, 1200), 7: (8, 1200)}


def main(cfgs):
    for cfgid in cfgs:
        npatch, maxpairs = SAMPLE[cfgid]
        kw = {1: {}, 5: dict(n_off=3000), 7: dict(p=8)}.get(cfgid, {})
        cfg = make_config(cfgid, **kw)
        S = cfg["surface"]
        rng = np.random.default_rng(cfgid)
        patches = rng.choice(S.n_patches, size=min(npatch, S.n_patches), replace=False)
        tgs = (cfg["tx"], cfg["tnormal"], cfg["self_node"], cfg["side"])
        tg, pa = O.near_pairs_for_patches(S, tgs[0], tgs[2], cfg["eta"], patches, all_pairs=cfg["all_pairs"])
        if tg.size > maxpairs:
            sel = np.sort(rng.choice(tg.size, maxpairs, replace=False))
            tg, pa = tg[sel], pa[sel]
        t0 = time.time()
        ref = U.reference(S, tgs, tg, pa)
        tq = time.time() - t0
        fma, _ = O.build_rows(S, *tgs, tg, pa, prec="fma")
        ld, _ = O.build_rows(S, *tgs, tg, pa, prec="ld")
        inv = np.unique(tg, return_inverse=True)[1]
        R = inv.max() + 1
        print(f"== config {cfgid}: p = {S.p}, {tg.size} pairs of {len(patches)} patches, {R} rows "
              f"(truth + 4 rounding modes: {tq:.1f} s on {os.cpu_count()} cores)")
        for k, name in enumerate("S D Sp Dp".split()):
            t = ref["t"][k]
            M = U._per_row(np.abs(t).max(1), inv, R)
            nz = M > 0
            if not nz.any():
                print(f"  {name:2s}: all rows identically zero")
                continue

            def rel(v):
                return U._per_row(np.abs(v - t).max(1), inv, R)[nz] / M[nz]
            eo, ef, el = rel(ref["o"][k]), rel(fma[k]), rel(ld[k])
            s = U._per_row(ref["env"][k].max(1), inv, R)[nz] / M[nz]
            g1 = ef / (4 * eo + 1e-11)
            g2 = ef / (U.ROW_FACTOR * s + 1e-11)
            q = lambda v: "/".join(f"{x:.1e}" for x in np.percentile(v, [50, 90, 100]))  # noqa: E731
            ok, st = U.gate_rows(fma[k], ref, k, inv)
            print(f"  {name:2s}: rows/M med/p90/max  fp64 {q(eo)}  fma {q(ef)}  envelope {q(s)}  long-double {q(el)}"
                  f"  | frac <= 1e-11: fp64 {np.mean(eo <= 1e-11):.3f}")
            print(f"      fma under e <= 4 e_o + 1e-11 M: {np.mean(g1 > 1) * 100:.1f} % rows fail (max ratio {g1.max():.2f});"
                  f"  under the bar: worst row ratio {g2.max() * U.ROW_FACTOR:.2f} / {U.ROW_FACTOR:.0f}, gate {'pass' if ok else 'FAIL'}")
        sys.stdout.flush()


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5, 6, 7])
