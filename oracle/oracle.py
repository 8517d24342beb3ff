"""ctypes binding of the CPU oracle (oracle/rrq_oracle.c): fp64, plus long-double and quad builds.

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
`--impl reference` legs may import this module.  It imports nothing from paper_2411_08342_b200/.
See the header of rrq_oracle.c for what it computes and the passages it follows.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rrq_oracle.c")

# The oracle in four builds of the same source (rrq_oracle.c header):
#   "d"    fp64, no FMA contraction: THE oracle (its rows are what "oracle" means in the tests);
#   "fma"  fp64 with FMA contraction (-mfma -ffp-contract=fast): a second, equally correct fp64 rounding;
#   "ld"   x87 long double (64-bit significand);
#   "q"    IEEE binary128: the truth reference (same algorithm, same fp64 inputs, ~34 digits).
_BUILDS = {
    "d": ("liboracle.so", ["-frounding-math", "-ffp-contract=off"]),
    "fma": ("liboracle_fma.so", ["-frounding-math", "-mfma", "-ffp-contract=fast"]),
    "ld": ("liboracle_ld.so", ["-DORC_REAL_LD"]),
    "q": ("liboracle_q.so", ["-DORC_REAL_QUAD"]),
}
PRECISIONS = tuple(_BUILDS)
ROUNDING = {"nearest": 0, "up": 1, "down": 2, "zero": 3}


def build(force=False, prec=None):
    """Compile the oracle library of precision `prec` (all four if None); returns the path (or the
    fp64 path when building all)."""
    out = None
    for k in (PRECISIONS if prec is None else (prec,)):
        name, flags = _BUILDS[k]
        lib_path = os.path.join(_HERE, name)
        if force or not os.path.exists(lib_path) or os.path.getmtime(lib_path) < os.path.getmtime(_SRC):
            tmp = lib_path + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", *flags, "-fopenmp", "-fPIC", "-shared", "-Wl,-Bsymbolic",
                                   "-o", tmp, _SRC, "-lquadmath", "-lm"])
            os.replace(tmp, lib_path)
        out = lib_path if out is None or k == "d" else out
    return out


class OrcParams(ctypes.Structure):
    _fields_ = [("p", ctypes.c_int), ("q", ctypes.c_int), ("n_omega", ctypes.c_int),
                ("rho0", ctypes.c_double), ("rounding", ctypes.c_int)]


_libs = {}


def lib(prec="d"):
    if prec not in _libs:
        _libs[prec] = ctypes.CDLL(build(prec=prec))
    return _libs[prec]


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def set_threads(n):
    os.environ["OMP_NUM_THREADS"] = str(n)


# ------------------------------------------------------------------ building blocks (pins)

def gauss_legendre(n):
    x = np.zeros(n); w = np.zeros(n)
    lib().orc_gauss_legendre(ctypes.c_int(n), _p(x), _p(w))
    return x, w


def tables(q):
    t = np.zeros(q); w = np.zeros(q); U = np.zeros((q, q))
    lib().orc_tables(ctypes.c_int(q), _p(t), _p(w), _p(U))
    return t, w, U


def legendre(p, x):
    P = np.zeros((p + 1, p + 1))
    lib().orc_legendre(ctypes.c_int(p), ctypes.c_double(x), ctypes.c_double(np.sqrt(1 - x * x)), _p(P))
    return P


def solid_R(p, X, Y, Z):
    """R_l^m(X,Y,Z) as dict-like array R[l*l+l+m]."""
    out = np.zeros(2 * (p + 1) ** 2)
    lib().orc_solid_R(ctypes.c_int(p), ctypes.c_double(X), ctypes.c_double(Y), ctypes.c_double(Z), _p(out))
    return out[0::2] + 1j * out[1::2]


def harmonics_S(p, x, y, z, hess=True):
    L = (p + 1) ** 2
    S = np.zeros(2 * L); G = np.zeros(6 * L); H = np.zeros(18 * L) if hess else None
    lib().orc_harmonics_S(ctypes.c_int(p), ctypes.c_double(x), ctypes.c_double(y), ctypes.c_double(z),
                          _p(S), _p(G), _p(H))
    S = S[0::2] + 1j * S[1::2]
    G = (G[0::2] + 1j * G[1::2]).reshape(L, 3)
    if hess:
        H = (H[0::2] + 1j * H[1::2]).reshape(L, 3, 3)
    return S, G, H


def qmul(f, g):
    out = np.zeros(4)
    lib().orc_qmul(_p(_c(f, np.float64)), _p(_c(g, np.float64)), _p(out))
    return out


def pinv_qr(A):
    A = _c(A, np.float64)
    m, k = A.shape
    out = np.zeros((k, m))
    st = lib().orc_pinv_qr(ctypes.c_int(m), ctypes.c_int(k), _p(A), _p(out))
    return out, st


def model_integrals(a, b, q):
    I = np.zeros(q); J = np.zeros(q)
    lib().orc_model_integrals(ctypes.c_double(a), ctypes.c_double(b), ctypes.c_int(q), _p(I), _p(J))
    return I, J


def model_integrals_direct(a, b, q):
    I = np.zeros(q); J = np.zeros(q)
    lib().orc_model_integrals_direct(ctypes.c_double(a), ctypes.c_double(b), ctypes.c_int(q), _p(I), _p(J))
    return I, J


def find_t0(C, rp, rho_stop=1e300):
    """C: [q,3] Legendre coefficients of an edge interpolant (reading A4'); rp target -> (t0, converged).
    rho_stop: early stop of reading A12' (default: never)."""
    C = _c(C, np.float64)
    re = ctypes.c_double(); im = ctypes.c_double()
    conv = lib().orc_find_t0(_p(C), ctypes.c_int(C.shape[0]), _p(_c(rp, np.float64)), ctypes.c_double(rho_stop),
                             ctypes.byref(re), ctypes.byref(im))
    return complex(re.value, im.value), bool(conv)


def bernstein_rho(t0):
    lib().orc_bernstein_rho.restype = ctypes.c_double
    return lib().orc_bernstein_rho(ctypes.c_double(t0.real), ctypes.c_double(t0.imag))


# ------------------------------------------------------------------ whole-path entry points

def params(p, q=None, n_omega=32, rho0=3.0, rounding="nearest"):
    return OrcParams(p, q if q is not None else 2 * p, n_omega, rho0, ROUNDING[rounding])


def patch_fit(S, prec="d", rounding="nearest"):
    P, n = S.nodes.shape[:2]
    p, q = S.p, S.q
    np_ = p * (p + 1) // 2
    fit = np.zeros((P, 13 * np_, n))
    st = np.zeros(P, np.int32)
    lib(prec).orc_patch_fit(ctypes.c_int64(P), ctypes.c_int(p), ctypes.c_int(q), _p(_c(S.nodes, np.float64)),
                            _p(_c(S.normals, np.float64)), _p(_c(S.verts, np.float64)),
                            _p(_c(S.edge_x, np.float64)), _p(_c(S.edge_dx, np.float64)), _p(fit), _p(st),
                            ctypes.c_int(ROUNDING[rounding]))
    return fit, st


def near_balls(S):
    """(c_P, R_P, h_P) of every patch (reading A6) -> [P, 5]."""
    ball = np.zeros((S.n_patches, 5))
    lib().orc_near_balls(ctypes.c_int64(S.n_patches), ctypes.c_int(S.p), ctypes.c_int(S.q),
                         _p(_c(S.nodes, np.float64)), _p(_c(S.weights, np.float64)), _p(_c(S.verts, np.float64)),
                         _p(_c(S.edge_x, np.float64)), _p(ball))
    return ball


def near_list(S, tx, self_node, eta, all_pairs=False):
    P = S.n_patches
    T = tx.shape[0]
    ptr = np.zeros(T + 1, np.int64)
    args = [ctypes.c_int64(P), ctypes.c_int(S.p), ctypes.c_int(S.q), _p(_c(S.nodes, np.float64)),
            _p(_c(S.weights, np.float64)), _p(_c(S.verts, np.float64)), _p(_c(S.edge_x, np.float64)),
            ctypes.c_int64(T), _p(_c(tx, np.float64)),
            _p(_c(self_node, np.int64)) if self_node is not None else None,
            ctypes.c_double(eta if np.isfinite(eta) else 1e300), ctypes.c_int(int(all_pairs))]
    lib().orc_near_list(*args, _p(ptr), None)
    pat = np.zeros(int(ptr[-1]), np.int32)
    lib().orc_near_list(*args, _p(ptr), _p(pat))
    return ptr, pat


def build_rows(S, tx, tnormal, self_node, side, pair_target, pair_patch, mask=15, raw=False, n_omega=32,
               rho0=3.0, prec="d", rounding="nearest", zeta=False):
    """-> vals [4, n_pairs, n] (S, D, S', D'), status [n_pairs] (, zeta [n_pairs, 9 np] if zeta: the Step 4-7
    outputs Theta [np] | W [np, 4] | dW [np, 4] per pair).  prec: "d" (the fp64 oracle), "fma", "ld" or "q"
    (truth); rounding: IEEE rounding mode of the whole evaluation ("nearest", "up", "down", "zero")."""
    n = S.n
    npairs = int(pair_target.shape[0])
    vals = np.zeros((4, npairs, n))
    st = np.zeros(npairs, np.int32)
    npb = S.p * (S.p + 1) // 2
    z = np.zeros((npairs, 9 * npb)) if zeta else None
    pr = params(S.p, S.q, n_omega, rho0, rounding)
    lib(prec).orc_build_rows(ctypes.byref(pr), ctypes.c_int64(S.n_patches), _p(_c(S.nodes, np.float64)),
                             _p(_c(S.normals, np.float64)), _p(_c(S.weights, np.float64)),
                             _p(_c(S.verts, np.float64)), _p(_c(S.edge_x, np.float64)),
                             _p(_c(S.edge_dx, np.float64)), _p(_c(tx, np.float64)),
                             _p(_c(tnormal, np.float64)) if tnormal is not None else None,
                             _p(_c(self_node, np.int64)) if self_node is not None else None,
                             _p(_c(side, np.int8)) if side is not None else None,
                             ctypes.c_int64(npairs), _p(_c(pair_target, np.int64)), _p(_c(pair_patch, np.int32)),
                             ctypes.c_uint32(mask), ctypes.c_int(int(raw)), _p(vals), _p(st), _p(z))
    return (vals, st, z) if zeta else (vals, st)


def pair_debug(S, P, x, nu, self_local=-1, side=2, raw=True, n_omega=32, rho0=3.0, prec="d", rounding="nearest"):
    """Intermediates of one pair on patch P.  Returns dict."""
    p, n = S.p, S.n
    np_ = p * (p + 1) // 2
    rows = np.zeros((4, n)); scal = np.zeros(20); W = np.zeros((np_, 4)); dW = np.zeros((np_, 4))
    Th = np.zeros(np_); frame = np.zeros(13)
    pr = params(p, S.q, n_omega, rho0, rounding)
    st = lib(prec).orc_pair_debug(ctypes.byref(pr), _p(_c(S.nodes[P], np.float64)), _p(_c(S.normals[P], np.float64)),
                              _p(_c(S.weights[P], np.float64)), _p(_c(S.verts[P], np.float64)),
                              _p(_c(S.edge_x[P], np.float64)), _p(_c(S.edge_dx[P], np.float64)),
                              _p(_c(x, np.float64)), _p(_c(nu, np.float64)) if nu is not None else None,
                              ctypes.c_int(self_local), ctypes.c_int(side), ctypes.c_int(int(raw)),
                              _p(rows), _p(scal), _p(W), _p(dW), _p(Th), _p(frame))
    return dict(rows=rows, Omega0=scal[0], Omega=scal[1:4], dOmega0=scal[4], dOmega=scal[5:8],
                t0=[complex(scal[8 + 4 * e], scal[9 + 4 * e]) for e in range(3)],
                swap=[int(scal[10 + 4 * e]) for e in range(3)], conv=[int(scal[11 + 4 * e]) for e in range(3)],
                W=W, dW=dW, Theta=Th, origin=frame[:3], Rm=frame[3:12].reshape(3, 3), h=frame[12], status=st)


def pairs_debug(S, P, x, nu=None, self_local=None, side=None, raw=True, n_omega=32, rho0=3.0, prec="d",
                rounding="nearest"):
    """Intermediates of many targets against patch P (patch built once).  Returns dict of arrays: rows
    [T, 4, n], Omega0 [T], Omega [T, 3], dOmega0 [T], dOmega [T, 3], t0 [T, 3] complex, swap/conv [T, 3],
    status [T] (local scaled frame of the patch, as pair_debug)."""
    x = _c(np.atleast_2d(x), np.float64)
    T = x.shape[0]
    n = S.n
    rows = np.zeros((T, 4, n)); scal = np.zeros((T, 20)); st = np.zeros(T, np.int32)
    sl = _c(np.full(T, -1) if self_local is None else self_local, np.int32)
    sd = _c(np.full(T, 2) if side is None else side, np.int32)
    pr = params(S.p, S.q, n_omega, rho0, rounding)
    lib(prec).orc_pairs_debug(ctypes.byref(pr), _p(_c(S.nodes[P], np.float64)), _p(_c(S.normals[P], np.float64)),
                              _p(_c(S.weights[P], np.float64)), _p(_c(S.verts[P], np.float64)),
                              _p(_c(S.edge_x[P], np.float64)), _p(_c(S.edge_dx[P], np.float64)), ctypes.c_int64(T),
                              _p(x), _p(_c(nu, np.float64)) if nu is not None else None, _p(sl), _p(sd),
                              ctypes.c_int(int(raw)), _p(rows), _p(scal), _p(st))
    return dict(rows=rows, Omega0=scal[:, 0], Omega=scal[:, 1:4], dOmega0=scal[:, 4], dOmega=scal[:, 5:8],
                t0=scal[:, 8:20:4] + 1j * scal[:, 9:20:4], swap=scal[:, 10:20:4].astype(int),
                conv=scal[:, 11:20:4].astype(int), status=st)


def pairs_from_ptr(ptr, pat):
    T = ptr.shape[0] - 1
    tgt = np.repeat(np.arange(T, dtype=np.int64), np.diff(ptr))
    return tgt, pat


def near_pairs_for_patches(S, tx, self_node, eta, patches, all_pairs=False, cap=10_000_000):
    """(target, patch) near pairs of the listed patches (reading A6), brute force over targets."""
    sel = np.ascontiguousarray(patches, dtype=np.int32)
    ot = np.zeros(cap, np.int64); op = np.zeros(cap, np.int32)
    lib().orc_near_pairs_for_patches.restype = ctypes.c_int64
    k = lib().orc_near_pairs_for_patches(
        ctypes.c_int(S.p), ctypes.c_int(S.q), _p(_c(S.nodes, np.float64)), _p(_c(S.weights, np.float64)),
        _p(_c(S.verts, np.float64)), _p(_c(S.edge_x, np.float64)), ctypes.c_int64(tx.shape[0]),
        _p(_c(tx, np.float64)), _p(_c(self_node, np.int64)) if self_node is not None else None,
        ctypes.c_double(eta if np.isfinite(eta) else 1e300), ctypes.c_int(int(all_pairs)),
        ctypes.c_int64(sel.size), _p(sel), ctypes.c_int64(cap), _p(ot), _p(op))
    k = min(int(k), cap)
    return ot[:k], op[:k]
