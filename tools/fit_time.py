"""Device time of rrq_patch_fit on config 4's full surface (50k patches, p = 8)."""
import sys, torch
sys.path.insert(0, '/root/repo')
from synth.configs import make_config
from paper_2411_08342_b200 import RRQ, DeviceSurface
cfg = make_config(4, n_off=1000)
S = cfg["surface"]
ctx = RRQ(S.p, eta=cfg["eta"])
ds = DeviceSurface.from_numpy(S)
ctx.patch_fit(ds)
torch.cuda.synchronize()
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ctx.patch_fit(ds); e1.record(); torch.cuda.synchronize()
    print('patches', S.n_patches, 'patch_fit ms', round(e0.elapsed_time(e1), 2))
