"""One pass of every C-ABI entry point on config 1 (20-patch sphere, p = 4) for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): near list (both phases), patch fit, the correction build
with overlap on (two sub-chunks via a small scratch budget) and RAW, apply, smooth apply.  Prints a
checksum so a clean run is visibly a complete one.  Usage: compute-sanitizer --tool X python tools/sanitize_cfg1.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("RRQ_SCRATCH_BYTES", "3e6")   # force several sub-chunks (producer/consumer overlap)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from synth.configs import make_config  # noqa: E402
from paper_2411_08342_b200 import RRQ, DeviceSurface, DeviceTargets  # noqa: E402


def main():
    p = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    cfg = make_config(1, n_off=200) if p == 4 else make_config(2, n_off=200, freq=2)
    S = cfg["surface"]
    ctx = RRQ(S.p, eta=cfg["eta"])
    ds = DeviceSurface.from_numpy(S)
    dt = DeviceTargets.from_numpy(cfg["tx"], cfg["tnormal"], cfg["self_node"], cfg["side"])
    ptr, pat = ctx.near_list(ds, dt)
    fit, fst = ctx.patch_fit(ds)
    out = ctx.build_correction(ds, dt, ptr, pat, fit)
    raw = ctx.build_correction(ds, dt, ptr, pat, fit, raw=True, row_begin=5, row_end=dt.n_targets - 3)
    dens = torch.ones(S.n_patches * S.n, dtype=torch.float64, device="cuda")
    y = torch.zeros(dt.n_targets, dtype=torch.float64, device="cuda")
    ctx.apply_correction(out["row_ptr"], out["col_idx"], out["vals"][1], dens, y)
    ys = torch.zeros(dt.n_targets, dtype=torch.float64, device="cuda")
    ctx.apply_smooth(ds, dt.x, dt.self_node, dens, ys)
    torch.cuda.synchronize()
    cs = sum(float(v.abs().sum()) for v in out["vals"]) + sum(float(v.abs().sum()) for v in raw["vals"])
    print(f"sanitize p={S.p}: {pat.numel()} pairs, fit status max {int(fst.max())}, checksum {cs:.6e}, "
          f"y sum {float(y.sum()):.6e}, smooth sum {float(ys.sum()):.6e}, launches {ctx.launch_count()}")


if __name__ == "__main__":
    main()
