"""ctypes binding of librrq.so with the same entry-point names as include/rrq.h.

Argument marshalling only: every step of the path runs in the library's CUDA kernels.  Device memory
and streams come from torch (plumbing).  Tensors must be CUDA, C-contiguous, of the dtype the header
states; the binding checks that and raises RRQError otherwise.
"""
import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("RRQ_LIBRARY") or os.path.join(_HERE, "librrq.so")   # override: kernel-variant experiments
KERNELS = ("S", "D", "Sp", "Dp")
RRQ_S, RRQ_D, RRQ_SP, RRQ_DP, RRQ_ALL, RRQ_RAW = 1, 2, 4, 8, 15, 16


class RRQError(RuntimeError):
    pass


class _Params(ctypes.Structure):
    _fields_ = [("p", ctypes.c_int32), ("n_nodes", ctypes.c_int32), ("p_edge", ctypes.c_int32),
                ("n_omega", ctypes.c_int32), ("eta", ctypes.c_double), ("rho_swap", ctypes.c_double),
                ("all_pairs", ctypes.c_int32)]


class _Surface(ctypes.Structure):
    _fields_ = [("n_patches", ctypes.c_int64)] + [(k, ctypes.c_void_p) for k in
                                                   ("nodes", "normals", "weights", "verts", "edge_x", "edge_dx")]


class _Targets(ctypes.Structure):
    _fields_ = [("n_targets", ctypes.c_int64), ("x", ctypes.c_void_p), ("normal", ctypes.c_void_p),
                ("self_node", ctypes.c_void_p), ("side", ctypes.c_void_p)]


_lib = None


def load_library():
    """Load librrq.so (fails loudly if it is missing: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise RRQError(f"librrq.so not built at {_LIB_PATH}; run __graft_entry__.build()")
    lib = ctypes.CDLL(_LIB_PATH)
    vp, i64, i32, u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32
    lib.rrq_create.argtypes = [ctypes.POINTER(_Params), ctypes.POINTER(vp)]
    lib.rrq_create.restype = ctypes.c_int
    lib.rrq_destroy.argtypes = [vp]
    lib.rrq_last_error.argtypes = [vp]
    lib.rrq_last_error.restype = ctypes.c_char_p
    lib.rrq_near_list.argtypes = [vp, ctypes.POINTER(_Surface), ctypes.POINTER(_Targets), vp, vp,
                                  ctypes.POINTER(i64), vp]
    lib.rrq_near_list.restype = ctypes.c_int
    lib.rrq_fit_bytes.argtypes = [vp, i64]
    lib.rrq_fit_bytes.restype = ctypes.c_size_t
    lib.rrq_patch_fit.argtypes = [vp, ctypes.POINTER(_Surface), vp, vp, vp]
    lib.rrq_patch_fit.restype = ctypes.c_int
    lib.rrq_build_correction.argtypes = [vp, ctypes.POINTER(_Surface), ctypes.POINTER(_Targets), vp, vp, i64, i64,
                                         i64, vp, u32, vp, vp, ctypes.POINTER(vp * 4), vp, vp]
    lib.rrq_build_correction.restype = ctypes.c_int
    lib.rrq_apply_correction.argtypes = [vp, i64, vp, vp, vp, vp, vp, vp]
    lib.rrq_apply_correction.restype = ctypes.c_int
    lib.rrq_apply_smooth.argtypes = [vp, i64, vp, vp, ctypes.POINTER(_Surface), ctypes.c_double, ctypes.c_double,
                                     vp, vp, vp]
    lib.rrq_apply_smooth.restype = ctypes.c_int
    lib.rrq_get_tables.argtypes = [vp, vp, vp, vp]
    lib.rrq_get_tables.restype = ctypes.c_int
    lib.rrq_launch_count.argtypes = [vp]
    lib.rrq_launch_count.restype = ctypes.c_int64
    lib.rrq_set_timing.argtypes = [vp, ctypes.c_int]
    lib.rrq_set_timing.restype = ctypes.c_int
    lib.rrq_set_overlap.argtypes = [vp, ctypes.c_int]
    lib.rrq_set_overlap.restype = ctypes.c_int
    lib.rrq_reset_timing.argtypes = [vp]
    lib.rrq_reset_timing.restype = ctypes.c_int
    lib.rrq_get_timing.argtypes = [vp, vp, vp, vp]
    lib.rrq_get_timing.restype = ctypes.c_int
    lib.rrq_debug_zeta.argtypes = [vp, i64, vp, vp, ctypes.POINTER(i64)]
    lib.rrq_debug_zeta.restype = ctypes.c_int
    _lib = lib
    return lib


def _ptr(t, dtype=None, name="tensor"):
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise RRQError(f"{name} must be a CUDA tensor")
    if dtype is not None and t.dtype != dtype:
        raise RRQError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise RRQError(f"{name} must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class DeviceSurface:
    """Surface arrays resident on the device."""

    def __init__(self, nodes, normals, weights, verts, edge_x, edge_dx):
        self.nodes, self.normals, self.weights = nodes, normals, weights
        self.verts, self.edge_x, self.edge_dx = verts, edge_x, edge_dx
        f64 = torch.float64
        self.c = _Surface(nodes.shape[0], _ptr(nodes, f64, "nodes"), _ptr(normals, f64, "normals"),
                          _ptr(weights, f64, "weights"), _ptr(verts, f64, "verts"), _ptr(edge_x, f64, "edge_x"),
                          _ptr(edge_dx, f64, "edge_dx"))

    @property
    def n_patches(self):
        return self.nodes.shape[0]

    @staticmethod
    def from_numpy(S, device="cuda"):
        g = lambda a: torch.as_tensor(a, dtype=torch.float64, device=device).contiguous()
        return DeviceSurface(g(S.nodes), g(S.normals), g(S.weights), g(S.verts), g(S.edge_x), g(S.edge_dx))


class DeviceTargets:
    def __init__(self, x, normal=None, self_node=None, side=None):
        self.x, self.normal, self.self_node, self.side = x, normal, self_node, side
        self.c = _Targets(x.shape[0], _ptr(x, torch.float64, "x"), _ptr(normal, torch.float64, "normal"),
                          _ptr(self_node, torch.int64, "self_node"), _ptr(side, torch.int8, "side"))

    @property
    def n_targets(self):
        return self.x.shape[0]

    @staticmethod
    def from_numpy(x, normal=None, self_node=None, side=None, device="cuda"):
        f = lambda a, dt: None if a is None else torch.as_tensor(a, dtype=dt, device=device).contiguous()
        return DeviceTargets(f(x, torch.float64), f(normal, torch.float64), f(self_node, torch.int64),
                             f(side, torch.int8))


class RRQ:
    """One rrq_ctx (constant tables + scratch) for a given discretisation order."""

    def __init__(self, p, eta=1.5, n_omega=32, rho_swap=3.0, all_pairs=False):
        if not torch.cuda.is_available():
            raise RRQError("no CUDA device: the RRQ builder has no CPU path")
        self.lib = load_library()
        self.p, self.n = p, p * p
        prm = _Params(p, p * p, 2 * p, n_omega, eta, rho_swap, int(all_pairs))
        h = ctypes.c_void_p()
        torch.cuda.init()
        st = self.lib.rrq_create(ctypes.byref(prm), ctypes.byref(h))
        if st != 0:
            raise RRQError(f"rrq_create: {st} {self.lib.rrq_last_error(None).decode()}")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.rrq_destroy(self.h)
            self.h = None

    def _check(self, st, what):
        if st != 0:
            raise RRQError(f"{what}: status {st}: {self.lib.rrq_last_error(self.h).decode()}")

    def launch_count(self):
        return int(self.lib.rrq_launch_count(self.h))

    STAGES = ("near_list", "patch_fit", "pair_edge", "qmap", "translate", "contract", "plumbing", "build", "newton", "edge_lines", "target_gamma")

    def set_timing(self, on=True):
        self._check(self.lib.rrq_set_timing(self.h, int(on)), "rrq_set_timing")

    def set_overlap(self, on=True):
        self._check(self.lib.rrq_set_overlap(self.h, int(on)), "rrq_set_overlap")

    def reset_timing(self):
        self._check(self.lib.rrq_reset_timing(self.h), "rrq_reset_timing")

    def timing(self):
        """Accumulated device ms and launch counts per stage + (pairs, swap edges)."""
        import numpy as np
        ms = np.zeros(len(self.STAGES)); n = np.zeros(len(self.STAGES), np.int64); st = np.zeros(2, np.int64)
        self._check(self.lib.rrq_get_timing(self.h, ms.ctypes.data, n.ctypes.data, st.ctypes.data), "rrq_get_timing")
        return dict(ms=dict(zip(self.STAGES, ms.tolist())), launches=dict(zip(self.STAGES, n.tolist())),
                    pairs=int(st[0]), swap_edges=int(st[1]))

    def debug_zeta(self, max_pairs):
        """Test hook: (perm, Z[., 13 n_p]) of the last build sub-chunk."""
        import numpy as np
        npb = self.p * (self.p + 1) // 2
        perm = np.zeros(max_pairs, np.int64); Z = np.zeros((max_pairs, 13 * npb))
        n = ctypes.c_int64(0)
        self._check(self.lib.rrq_debug_zeta(self.h, max_pairs, perm.ctypes.data, Z.ctypes.data, ctypes.byref(n)),
                    "rrq_debug_zeta")
        return perm[: n.value], Z[: n.value]

    def tables(self):
        q = 2 * self.p
        import numpy as np
        t = np.zeros(q); w = np.zeros(q); U = np.zeros((q, q))
        self._check(self.lib.rrq_get_tables(self.h, t.ctypes.data, w.ctypes.data, U.ctypes.data), "rrq_get_tables")
        return t, w, U

    def near_list(self, surf, tgt):
        dev = tgt.x.device
        ptr = torch.zeros(tgt.n_targets + 1, dtype=torch.int64, device=dev)
        n = ctypes.c_int64(0)
        self._check(self.lib.rrq_near_list(self.h, ctypes.byref(surf.c), ctypes.byref(tgt.c), _ptr(ptr), None,
                                           ctypes.byref(n), _stream()), "rrq_near_list(count)")
        pat = torch.empty(max(n.value, 1), dtype=torch.int32, device=dev)
        self._check(self.lib.rrq_near_list(self.h, ctypes.byref(surf.c), ctypes.byref(tgt.c), _ptr(ptr), _ptr(pat),
                                           ctypes.byref(n), _stream()), "rrq_near_list(fill)")
        return ptr, pat[: n.value]

    def fit_bytes(self, n_patches):
        return int(self.lib.rrq_fit_bytes(self.h, n_patches))

    def patch_fit(self, surf):
        nb = self.fit_bytes(surf.n_patches)
        dev = surf.nodes.device
        fit = torch.empty(nb // 8, dtype=torch.float64, device=dev)
        st = torch.zeros(surf.n_patches, dtype=torch.int32, device=dev)
        self._check(self.lib.rrq_patch_fit(self.h, ctypes.byref(surf.c), _ptr(fit), _ptr(st), _stream()),
                    "rrq_patch_fit")
        return fit, st

    def build_correction(self, surf, tgt, pair_ptr, pair_patch, fit, mask=RRQ_ALL, raw=False, row_begin=0,
                         row_end=None, out=None, want_col=True, want_status=True):
        """Returns dict(row_ptr, col_idx, vals=[S, D, S', D'], status) for rows [row_begin, row_end).
        `out` may pass preallocated tensors (same keys) to reuse buffers."""
        if row_end is None:
            row_end = tgt.n_targets
        dev = tgt.x.device
        if out is None:
            npairs = int(pair_ptr[row_end].item() - pair_ptr[row_begin].item())
            nnz = npairs * self.n
            out = dict(row_ptr=torch.empty(row_end - row_begin + 1, dtype=torch.int64, device=dev),
                       col_idx=torch.empty(max(nnz, 1), dtype=torch.int32, device=dev) if want_col else None,
                       vals=[torch.empty(max(nnz, 1), dtype=torch.float64, device=dev) if (mask >> k) & 1 else None
                             for k in range(4)],
                       status=torch.empty(max(npairs, 1), dtype=torch.int32, device=dev) if want_status else None)
        vp4 = (ctypes.c_void_p * 4)(*[ctypes.c_void_p(v.data_ptr()) if v is not None else None for v in out["vals"]])
        m = mask | (RRQ_RAW if raw else 0)
        self._check(self.lib.rrq_build_correction(
            self.h, ctypes.byref(surf.c), ctypes.byref(tgt.c), _ptr(pair_ptr, torch.int64, "pair_ptr"),
            _ptr(pair_patch, torch.int32, "pair_patch"), int(pair_patch.numel()), row_begin, row_end,
            _ptr(fit, torch.float64, "fit"), m, _ptr(out["row_ptr"]) if out.get("row_ptr") is not None else None,
            _ptr(out["col_idx"]) if out.get("col_idx") is not None else None, ctypes.byref(vp4),
            _ptr(out["status"]) if out.get("status") is not None else None, _stream()), "rrq_build_correction")
        return out

    def apply_smooth(self, surf, tx, self_node, density, y, alpha=1.0, beta=0.0):
        """y += alpha S_smooth[density] + beta D_smooth[density] at targets tx (self node skipped)."""
        self._check(self.lib.rrq_apply_smooth(self.h, tx.shape[0], _ptr(tx, torch.float64, "tx"),
                                              _ptr(self_node, torch.int64, "self_node"), ctypes.byref(surf.c),
                                              float(alpha), float(beta), _ptr(density, torch.float64, "density"),
                                              _ptr(y, torch.float64, "y"), _stream()),
                    "rrq_apply_smooth")
        return y

    def apply_correction(self, row_ptr, col_idx, vals, density, y):
        self._check(self.lib.rrq_apply_correction(self.h, row_ptr.numel() - 1, _ptr(row_ptr, torch.int64),
                                                  _ptr(col_idx, torch.int32), _ptr(vals, torch.float64),
                                                  _ptr(density, torch.float64), _ptr(y, torch.float64), _stream()),
                    "rrq_apply_correction")
        return y
