"""Curved triangular patches from exact surface maps.

Every patch P is the image X_P(s,t) of the reference triangle (0,0),(1,0),(0,1).  Nodes are the
collapsed Gauss-Legendre rule (s,t) = (u, v(1-u)), u-major order, weights w_u w_v (1-u)|X_s x X_t|
(SURVEY §8(c) A1).  Edge e runs vertex e -> vertex e+1 (CCW about the outward normal), sampled at the
q Gauss-Legendre parameters tau in (-1,1); edge_dx = dX/dtau.  Derivatives of X are taken by torch
autograd in float64 (exact up to rounding), so every map only has to be written once.
"""
from dataclasses import dataclass
import numpy as np
import torch


@dataclass
class Surface:
    p: int
    q: int
    nodes: np.ndarray      # [P, n, 3]
    normals: np.ndarray    # [P, n, 3]
    weights: np.ndarray    # [P, n]
    verts: np.ndarray      # [P, 3, 3]
    edge_x: np.ndarray     # [P, 3, q, 3]
    edge_dx: np.ndarray    # [P, 3, q, 3]
    uv: np.ndarray         # [n, 2] reference (s, t) of the nodes
    # parameters of the per-patch map, kept so targets can be generated on the exact surface
    kind: str = ""
    pdata: np.ndarray = None
    fmap: object = None     # X = fmap(pdata_rows, s, t) (torch); lets tests evaluate the exact map

    def eval_patch(self, P, s, t):
        """Exact map of patch P at reference points (s, t): X, X_s, X_t  (numpy [k,3] each)."""
        s = np.atleast_1d(np.asarray(s, np.float64))
        t = np.atleast_1d(np.asarray(t, np.float64))
        rows = torch.as_tensor(self.pdata[P:P + 1]).repeat(s.size, 1)
        return _eval_map(self.fmap, rows, s, t)

    @property
    def n_patches(self):
        return self.nodes.shape[0]

    @property
    def n(self):
        return self.nodes.shape[1]


def gauss_legendre_01(n):
    x, w = np.polynomial.legendre.leggauss(n)
    return (x + 1.0) / 2.0, w / 2.0


def collapsed_nodes(p):
    """Collapsed p x p Gauss-Legendre rule on the reference triangle, u-major."""
    u, wu = gauss_legendre_01(p)
    v, wv = gauss_legendre_01(p)
    U, V = np.meshgrid(u, v, indexing="ij")
    WU, WV = np.meshgrid(wu, wv, indexing="ij")
    s = U.ravel()
    t = (V * (1.0 - U)).ravel()
    w = (WU * WV * (1.0 - U)).ravel()
    return s, t, w


def _eval_map(fmap, pdata, s, t):
    """X, X_s, X_t for per-point parameter rows pdata[k] at (s[k], t[k]) (torch autograd)."""
    s = torch.as_tensor(s, dtype=torch.float64).clone().requires_grad_(True)
    t = torch.as_tensor(t, dtype=torch.float64).clone().requires_grad_(True)
    X = fmap(pdata, s, t)
    Xs = torch.empty_like(X)
    Xt = torch.empty_like(X)
    for c in range(3):
        gs, gt = torch.autograd.grad(X[:, c].sum(), (s, t), retain_graph=True)
        Xs[:, c] = gs
        Xt[:, c] = gt
    return X.detach().numpy(), Xs.detach().numpy(), Xt.detach().numpy()


def build_surface(fmap, pdata, p, q, kind=""):
    """Discretise patches X_P = fmap(pdata[P], s, t) (pdata: torch [P, k])."""
    P = pdata.shape[0]
    s0, t0, w0 = collapsed_nodes(p)
    n = s0.size
    rep = pdata.repeat_interleave(n, dim=0)
    X, Xs, Xt = _eval_map(fmap, rep, np.tile(s0, P), np.tile(t0, P))
    cr = np.cross(Xs, Xt)
    J = np.linalg.norm(cr, axis=1)
    nodes = X.reshape(P, n, 3)
    normals = (cr / J[:, None]).reshape(P, n, 3)
    weights = (np.tile(w0, P) * J).reshape(P, n)
    # vertices
    vs = np.array([0.0, 1.0, 0.0])
    vt = np.array([0.0, 0.0, 1.0])
    Xv, _, _ = _eval_map(fmap, pdata.repeat_interleave(3, dim=0), np.tile(vs, P), np.tile(vt, P))
    verts = Xv.reshape(P, 3, 3)
    # edges: e0 v0->v1, e1 v1->v2, e2 v2->v0, tau in (-1,1) Gauss-Legendre
    tau, _ = np.polynomial.legendre.leggauss(q)
    es = np.concatenate([(1 + tau) / 2, (1 - tau) / 2, np.zeros(q)])
    et = np.concatenate([np.zeros(q), (1 + tau) / 2, (1 - tau) / 2])
    dsd = np.concatenate([np.full(q, 0.5), np.full(q, -0.5), np.zeros(q)])
    dtd = np.concatenate([np.zeros(q), np.full(q, 0.5), np.full(q, -0.5)])
    Xe, Xes, Xet = _eval_map(fmap, pdata.repeat_interleave(3 * q, dim=0), np.tile(es, P), np.tile(et, P))
    edge_x = Xe.reshape(P, 3, q, 3)
    edge_dx = (Xes * np.tile(dsd, P)[:, None] + Xet * np.tile(dtd, P)[:, None]).reshape(P, 3, q, 3)
    return Surface(p=p, q=q, nodes=nodes, normals=normals, weights=weights, verts=verts,
                   edge_x=edge_x, edge_dx=edge_dx, uv=np.stack([s0, t0], 1), kind=kind,
                   pdata=pdata.numpy(), fmap=fmap)


# ----------------------------------------------------------------------------- icosahedral spheres

def icosahedron():
    g = (1 + 5 ** 0.5) / 2
    V = []
    for a in (-1, 1):
        for b in (-g, g):
            V += [(0, a, b), (a, b, 0), (b, 0, a)]
    V = np.array(V, dtype=np.float64)
    V /= np.linalg.norm(V, axis=1, keepdims=True)
    el = min(np.linalg.norm(V[i] - V[j]) for i in range(12) for j in range(i + 1, 12))
    F = []
    for i in range(12):
        for j in range(i + 1, 12):
            for k in range(j + 1, 12):
                if all(abs(np.linalg.norm(V[x] - V[y]) - el) < 1e-9 for x, y in ((i, j), (j, k), (i, k))):
                    a, b, c = V[i], V[j], V[k]
                    if np.dot(np.cross(b - a, c - a), a + b + c) < 0:
                        j2, k2 = k, j
                    else:
                        j2, k2 = j, k
                    F.append((i, j2, k2))
    assert len(F) == 20
    return V, np.array(F)


def subdivided_flat_triangles(freq):
    """Frequency-`freq` grid on every flat icosahedron face: 20*freq^2 flat triangles [P,3,3]."""
    V, F = icosahedron()
    tris = []
    for (i, j, k) in F:
        A, B, C = V[i], V[j], V[k]
        P = lambda a, b: A + (a / freq) * (B - A) + (b / freq) * (C - A)
        for a in range(freq):
            for b in range(freq - a):
                tris.append((P(a, b), P(a + 1, b), P(a, b + 1)))
                if a + b <= freq - 2:
                    tris.append((P(a + 1, b), P(a + 1, b + 1), P(a, b + 1)))
    return np.array(tris)


def _radial_map(radius_fn):
    def fmap(pd, s, t):
        a, b, c = pd[:, 0:3], pd[:, 3:6], pd[:, 6:9]
        y = a + s[:, None] * (b - a) + t[:, None] * (c - a)
        xh = y / torch.linalg.norm(y, dim=1, keepdim=True)
        return xh * radius_fn(xh)[:, None]
    return fmap


def make_sphere_surface(freq, p, q, radius_fn=None):
    tris = subdivided_flat_triangles(freq)
    pdata = torch.as_tensor(tris.reshape(-1, 9))
    rf = radius_fn if radius_fn is not None else (lambda xh: torch.ones_like(xh[:, 0]))
    return build_surface(_radial_map(rf), pdata, p, q, kind="sphere")


def make_cap_surface(chord, p, q):
    """One unit-sphere cap: flat equilateral triangle with side `chord` about +z, projected (cfg 5)."""
    rho = chord / 3 ** 0.5
    zc = (1 - rho * rho) ** 0.5
    ang = np.pi / 2 + 2 * np.pi * np.arange(3) / 3
    tri = np.stack([rho * np.cos(ang), rho * np.sin(ang), np.full(3, zc)], 1)
    pdata = torch.as_tensor(tri.reshape(1, 9))
    return build_surface(_radial_map(lambda xh: torch.ones_like(xh[:, 0])), pdata, p, q, kind="cap")


# ----------------------------------------------------------------------------- real spherical harmonics

def real_sph_harm_torch(lmax, xh):
    """Orthonormal real spherical harmonics Y_lm(xh) for unit vectors xh [N,3]; dict (l,m)->tensor.

    Uses Q_l^m(z) = P_l^m(z)/(1-z^2)^{m/2} and sin^m(theta) e^{im phi} = (x+iy)^m, so it is a polynomial
    in the Cartesian components (differentiable by autograd everywhere).  Test-input plumbing only.
    """
    import math
    x, y, z = xh[:, 0], xh[:, 1], xh[:, 2]
    out = {}
    # (x+iy)^m real/imag parts
    cr, ci = [torch.ones_like(x)], [torch.zeros_like(x)]
    for m in range(1, lmax + 1):
        cr.append(cr[-1] * x - ci[-1] * y)
        ci.append(cr[-2] * y + ci[-1] * x)
    for m in range(0, lmax + 1):
        Q = {}
        Q[m] = torch.full_like(z, float(np.prod(np.arange(1, 2 * m, 2))) if m > 0 else 1.0)
        if m + 1 <= lmax:
            Q[m + 1] = (2 * m + 1) * z * Q[m]
        for l in range(m + 2, lmax + 1):
            Q[l] = ((2 * l - 1) * z * Q[l - 1] - (l + m - 1) * Q[l - 2]) / (l - m)
        for l in range(m, lmax + 1):
            N = math.sqrt((2 * l + 1) / (4 * math.pi) * math.factorial(l - m) / math.factorial(l + m))
            if m == 0:
                out[(l, 0)] = N * Q[l]
            else:
                out[(l, m)] = math.sqrt(2) * N * Q[l] * cr[m]
                out[(l, -m)] = math.sqrt(2) * N * Q[l] * ci[m]
    return out


def bumpy_radius_fn(coef, lmax=6, amp=0.2):
    def rf(xh):
        Y = real_sph_harm_torch(lmax, xh)
        r = torch.ones_like(xh[:, 0])
        for (l, m), c in coef.items():
            r = r + amp * c * Y[(l, m)]
        return r
    return rf


# ----------------------------------------------------------------------------- torus

def make_torus_surface(R, r, n_theta, n_phi, p, q):
    """Torus, theta minor (n_theta), phi major (n_phi); each (phi,theta) quad halved along the
    lower-left -> upper-right diagonal.  Parameter order (phi, theta) makes
    X_phi x X_theta the outward normal, so parameter-space CCW is CCW about the outward normal."""
    dphi = 2 * np.pi / n_phi
    dth = 2 * np.pi / n_theta
    pd = []
    for i in range(n_phi):
        for j in range(n_theta):
            LL = (i * dphi, j * dth)
            LR = ((i + 1) * dphi, j * dth)
            UR = ((i + 1) * dphi, (j + 1) * dth)
            UL = (i * dphi, (j + 1) * dth)
            pd.append(LL + LR + UR)
            pd.append(LL + UR + UL)
    pdata = torch.as_tensor(np.array(pd, dtype=np.float64))

    def fmap(pdt, s, t):
        P0, P1, P2 = pdt[:, 0:2], pdt[:, 2:4], pdt[:, 4:6]
        ab = P0 + s[:, None] * (P1 - P0) + t[:, None] * (P2 - P0)
        ph, th = ab[:, 0], ab[:, 1]
        rho = R + r * torch.cos(th)
        return torch.stack([rho * torch.cos(ph), rho * torch.sin(ph), r * torch.sin(th)], 1)

    S = build_surface(fmap, pdata, p, q, kind="torus")
    return S


# Stellarator of PAPER eq (stellarator): r(u, v) = sum_{i=-1..2} sum_{j=-1..1} delta_ij
# [cos v cos((1-i)u + jv), sin v cos((1-i)u + jv), sin((1-i)u + jv)], (u, v) in [0, 2 pi]^2.
STELLARATOR_DELTA = {(-1, -1): 0.17, (-1, 0): 0.11, (0, 0): 1.0, (1, 0): 4.5, (2, 0): -0.25, (0, 1): 0.07,
                     (2, 1): -0.45}


def make_stellarator_surface(n_u, n_v, p, q):
    """The paper's stellarator, the parameter square split into n_u x n_v equal rectangles, each halved
    (P:L1856-1858).  v is the toroidal (major) angle, u the poloidal one; parameter order (v, u) makes
    X_v x X_u the outward normal (checked by tests/test_oracle_stellarator.py: enclosed volume > 0)."""
    dv = 2 * np.pi / n_v
    du = 2 * np.pi / n_u
    pd = []
    for i in range(n_v):
        for j in range(n_u):
            LL = (i * dv, j * du)
            LR = ((i + 1) * dv, j * du)
            UR = ((i + 1) * dv, (j + 1) * du)
            UL = (i * dv, (j + 1) * du)
            pd.append(LL + LR + UR)
            pd.append(LL + UR + UL)
    pdata = torch.as_tensor(np.array(pd, dtype=np.float64))

    def fmap(pdt, s, t):
        P0, P1, P2 = pdt[:, 0:2], pdt[:, 2:4], pdt[:, 4:6]
        ab = P0 + s[:, None] * (P1 - P0) + t[:, None] * (P2 - P0)
        v, u = ab[:, 0], ab[:, 1]
        x = torch.zeros_like(v); y = torch.zeros_like(v); z = torch.zeros_like(v)
        for (i, j), d in STELLARATOR_DELTA.items():
            ang = (1 - i) * u + j * v
            c = torch.cos(ang)
            x = x + d * torch.cos(v) * c
            y = y + d * torch.sin(v) * c
            z = z + d * torch.sin(ang)
        return torch.stack([x, y, z], 1)

    return build_surface(fmap, pdata, p, q, kind="stellarator")


def make_interlocked_tori(n_theta, n_phi, p, q, count=4, a=3.0, b=0.5, shift=4.95):
    """The evaluation-phase boundary of PAPER §5: `count` copies of the torus eq (eq:torus)
    with a = 3, b = 0.5 (omega_c = 0), torus k translated by k * shift along x and, for odd k, rotated by
    90 degrees about the x axis, so adjacent tori interlock with a 0.05 gap (shift 4.95).  Each torus is
    n_theta x n_phi rectangles halved (the same split as make_torus_surface)."""
    dphi = 2 * np.pi / n_phi
    dth = 2 * np.pi / n_theta
    pd = []
    for k in range(count):
        for i in range(n_phi):
            for j in range(n_theta):
                LL = (i * dphi, j * dth)
                LR = ((i + 1) * dphi, j * dth)
                UR = ((i + 1) * dphi, (j + 1) * dth)
                UL = (i * dphi, (j + 1) * dth)
                pd.append(LL + LR + UR + (k,))
                pd.append(LL + UR + UL + (k,))
    pdata = torch.as_tensor(np.array(pd, dtype=np.float64))

    def fmap(pdt, s, t):
        P0, P1, P2 = pdt[:, 0:2], pdt[:, 2:4], pdt[:, 4:6]
        ab = P0 + s[:, None] * (P1 - P0) + t[:, None] * (P2 - P0)
        ph, th = ab[:, 0], ab[:, 1]
        rho = a + b * torch.cos(th)
        x, y, z = rho * torch.cos(ph), rho * torch.sin(ph), b * torch.sin(th)
        odd = (pdt[:, 6] % 2) == 1
        # rotation by +90 degrees about x for odd k: (x, y, z) -> (x, -z, y)
        y2 = torch.where(odd, -z, y)
        z2 = torch.where(odd, y, z)
        return torch.stack([x + shift * pdt[:, 6], y2, z2], 1)

    return build_surface(fmap, pdata, p, q, kind="tori")


def inside_interlocked_tori(x, count=4, a=3.0, b=0.5, shift=4.95):
    """True where x lies inside (or on) one of the tori of make_interlocked_tori."""
    x = np.asarray(x, np.float64)
    inside = np.zeros(x.shape[0], bool)
    for k in range(count):
        px, py, pz = x[:, 0] - shift * k, x[:, 1], x[:, 2]
        if k % 2 == 1:   # undo the rotation: (x, y, z) = (x0, -z0, y0) -> z0 = -y, y0 = z
            py, pz = pz, -py
        dc = np.sqrt(px ** 2 + py ** 2) - a
        inside |= dc ** 2 + pz ** 2 <= b * b
    return inside


def make_flat_surface(tris, p, q):
    """Flat triangles [P,3,3] with the affine map (test geometry)."""
    pdata = torch.as_tensor(np.asarray(tris, np.float64).reshape(-1, 9))

    def fmap(pd, s, t):
        a, b, c = pd[:, 0:3], pd[:, 3:6], pd[:, 6:9]
        return a + s[:, None] * (b - a) + t[:, None] * (c - a)
    return build_surface(fmap, pdata, p, q, kind="flat")
