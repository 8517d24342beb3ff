import sys, ctypes, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from synth.configs import make_config
import parity_util as U
import paper_2411_08342_b200 as pkg
cfg = make_config(4, n_off=20000, freq=10)
res = U.gpu_build(cfg, cfg['surface'], (cfg['tx'], cfg['tnormal'], cfg['self_node'], cfg['side']))
lib = pkg.load_library()
lib.rrq_debug_phase_cycles.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
out = np.zeros(8, np.uint64)
lib.rrq_debug_phase_cycles(res['ctx'].h, out.ctypes.data, 1)
tot = out[:3].sum()
for i, n in enumerate(['load+list', 'model+sinh', 'weights']):   # k_edge_lines' steps
    print('%-14s %5.1f%%' % (n, 100 * out[i] / tot))
