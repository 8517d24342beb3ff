"""Phase split of k_patch_fit_q (SM cycles between its CTA barriers, summed over CTAs) on config 4's surface."""
import sys, ctypes, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from synth.configs import make_config
import parity_util as U
import paper_2411_08342_b200 as pkg
cfg = make_config(4, n_off=20000, freq=10)
res = U.gpu_build(cfg, cfg['surface'], (cfg['tx'], cfg['tnormal'], cfg['self_node'], cfg['side']))
lib = pkg.load_library()
lib.rrq_debug_fit_cycles.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
out = np.zeros(8, np.uint64)
lib.rrq_debug_fit_cycles(res['ctx'].h, out.ctypes.data, 1)
tot = out.sum()
names = ['node tables', 'quaternion QR', 'Q^H e_c', 'quat backsub', 'real QR', 'Q_B^T e_c', 'real backsub', 'HP + P_Sg']
for i, n in enumerate(names):
    print('%-14s %5.1f%%  %8.1f kcycles/patch-CTA' % (n, 100 * out[i] / tot, out[i] / 1e3 / cfg['surface'].n_patches))
print('patches', cfg['surface'].n_patches)
