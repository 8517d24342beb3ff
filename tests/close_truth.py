"""Independent truths for the close-evaluation pins (tests/test_oracle_close.py, tools/close_sweep.py).

Nothing here shares code with the oracle or the CUDA path; everything is mpmath at 30+ digits.

* Flat triangle, density 1: the solid angle Omega_0 by the Van
  Oosterom-Strackee formula, D[1] = -Omega_0/4pi, S'[1] = Omega_0/4pi (nu' = z), D'[1] = -dOmega_0/dz'/4pi,
  and S[1] = (1/4pi) int_T da/|r'-r| by the planar divergence identity div(rho (R-|z|)/|rho|^2) = 1/R:
  S[1] = (1/4pi) sum_e P_e int_e (R - |z|)/(P_e^2 + s^2) ds (P_e the signed distance of the target's
  projection to edge e, s the arclength from its foot point), each edge integral by tanh-sinh quadrature
  split at the foot point.
* Curved patch, density 1: Omega_0 = -sum_e int ((d x u).x'(t)) / (|d| (|d| + u.d)) dt (reading G1, the line
  integral whose exact value is the solid angle when the u-ray misses the patch, reading A8) and the
  Biot-Savart dOmega_0/dnu' = sum_e int nu'.(tau(t) x d(t)) / |d|^3 dt (reading A10), both along the degree
  p~-1 polynomial through the patch's edge samples at the exact Gauss-Legendre parameters (the edge curve
  the method integrates along, reading A4), adaptive tanh-sinh split at the closest point.  The edge curve
  must be that interpolant, not the exact map: near an edge the solid angle moves by ~2 eps / l for a
  normal displacement eps of the edge at lateral distance l (the rounding of the fp64 samples alone
  is worth 1e-9 at l = 1e-8 h)."""
import mpmath as mp
import numpy as np

DPS = 30


def _cross(a, b):
    return [a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]]


def _dot(a, b):
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]


def _mpv(x):
    return [mp.mpf(float(c)) for c in x]


# ------------------------------------------------------------------------------------------- flat
def vos(V, r):
    """Van Oosterom-Strackee signed solid angle of the flat triangle V (3 mp vectors) seen from r."""
    R = [[V[i][a] - r[a] for a in range(3)] for i in range(3)]
    n = [mp.sqrt(_dot(x, x)) for x in R]
    num = _dot(R[0], _cross(R[1], R[2]))
    den = n[0] * n[1] * n[2] + _dot(R[0], R[1]) * n[2] + _dot(R[0], R[2]) * n[1] + _dot(R[1], R[2]) * n[0]
    return 2 * mp.atan2(num, den)


def flat_single_layer_1(V, r):
    """int_T da / |r' - r| for the triangle V in the plane z = 0, CCW about +z."""
    z = abs(r[2])
    tot = mp.mpf(0)
    for e in range(3):
        a, b = V[e], V[(e + 1) % 3]
        L = mp.sqrt((b[0] - a[0]) ** 2 + (b[1] - a[1]) ** 2)
        u = [(b[0] - a[0]) / L, (b[1] - a[1]) / L]
        nout = [u[1], -u[0]]
        P = (a[0] - r[0]) * nout[0] + (a[1] - r[1]) * nout[1]      # > 0 when the projection is inside
        s0 = (r[0] - a[0]) * u[0] + (r[1] - a[1]) * u[1]

        def f(s):
            return (mp.sqrt(P * P + s * s + z * z) - z) / (P * P + s * s)
        pts = [-s0, L - s0]
        if pts[0] < 0 < pts[1]:
            pts = [pts[0], 0, pts[1]]
        tot += P * mp.quad(f, pts)
    return tot


def flat_truths(tri, x):
    """Row sums of the four kernels for density 1 on the flat triangle tri ([3,3], z = 0), target x, nu' = z."""
    with mp.workdps(DPS):
        V = [_mpv(v) for v in tri]
        r = _mpv(x)
        Om = vos(V, r)
        dOm = mp.diff(lambda zz: vos(V, [r[0], r[1], zz]), r[2])
        S1 = flat_single_layer_1(V, r)
        return {"S": float(S1 / (4 * mp.pi)), "D": float(-Om / (4 * mp.pi)), "Sp": float(Om / (4 * mp.pi)),
                "Dp": float(-dOm / (4 * mp.pi))}


# ------------------------------------------------------------------------------------------- curved
class EdgeCurves:
    """The degree q-1 polynomial through each edge's samples at the exact q-point Gauss-Legendre
    parameters (positions and tangent samples), as Legendre series with exact (Gauss) coefficients."""

    def __init__(self, edge_x, edge_dx, verts):
        self.q = edge_x.shape[1]
        with mp.workdps(DPS):
            self.tg, self.wg = self._gl(self.q)
            self.CX = [self._coeffs(edge_x[e]) for e in range(3)]
            self.CT = [self._coeffs(edge_dx[e]) for e in range(3)]
            V = [_mpv(v) for v in verts]
            z = _cross([V[1][i] - V[0][i] for i in range(3)], [V[2][i] - V[0][i] for i in range(3)])
            nz = mp.sqrt(_dot(z, z))
            self.zhat = [c / nz for c in z]       # the patch normal of reading A2 (gauge axis, A8)
        self.edge_x = edge_x

    @staticmethod
    def _gl(n):
        xs, ws = [], []
        for i in range(n):
            t = mp.cos(mp.pi * (n - i - mp.mpf(0.25)) / (n + mp.mpf(0.5)))
            for _ in range(100):
                p0, p1 = mp.mpf(1), t
                for k in range(2, n + 1):
                    p0, p1 = p1, ((2 * k - 1) * t * p1 - (k - 1) * p0) / k
                dp = n * (t * p1 - p0) / (t * t - 1)
                dt = p1 / dp
                t -= dt
                if abs(dt) < mp.mpf(10) ** (-DPS + 3):
                    break
            p0, p1 = mp.mpf(1), t
            for k in range(2, n + 1):
                p0, p1 = p1, ((2 * k - 1) * t * p1 - (k - 1) * p0) / k
            dp = n * (t * p1 - p0) / (t * t - 1)
            xs.append(t)
            ws.append(2 / ((1 - t * t) * dp * dp))
        return xs, ws

    def _coeffs(self, Y):
        q = self.q
        C = [[mp.mpf(0)] * 3 for _ in range(q)]
        for k in range(q):
            Pj = [mp.mpf(1), self.tg[k]]
            for j in range(1, q - 1):
                Pj.append(((2 * j + 1) * self.tg[k] * Pj[j] - j * Pj[j - 1]) / (j + 1))
            for j in range(q):
                f = (2 * j + 1) * self.wg[k] * Pj[j] / 2
                for a in range(3):
                    C[j][a] += f * mp.mpf(float(Y[k][a]))
        return C

    def _eval(self, C, t):
        q = self.q
        x = [C[0][a] for a in range(3)]
        dx = [mp.mpf(0)] * 3
        P0, P1, d0, d1 = mp.mpf(1), t, mp.mpf(0), mp.mpf(1)
        for a in range(3):
            x[a] += C[1][a] * P1
            dx[a] += C[1][a]
        for j in range(1, q - 1):
            P2 = ((2 * j + 1) * t * P1 - j * P0) / (j + 1)
            d2 = d0 + (2 * j + 1) * P1
            for a in range(3):
                x[a] += C[j + 1][a] * P2
                dx[a] += C[j + 1][a] * d2
            P0, P1, d0, d1 = P1, P2, d1, d2
        return x, dx

    def _closest(self, e, r):
        j = int(np.argmin(np.linalg.norm(self.edge_x[e] - np.array([float(c) for c in r])[None], axis=1)))
        t = self.tg[j]
        for _ in range(60):     # Newton on g(t) = (x(t) - r').x'(t), g' = |x'|^2 + (x - r').x''
            X, dX = self._eval(self.CX[e], t)
            hh = mp.mpf(10) ** (-DPS // 2)
            _, dXp = self._eval(self.CX[e], t + hh)
            _, dXm = self._eval(self.CX[e], t - hh)
            ddX = [(dXp[i] - dXm[i]) / (2 * hh) for i in range(3)]
            dd = [X[i] - r[i] for i in range(3)]
            g = _dot(dd, dX)
            gp = _dot(dX, dX) + _dot(dd, ddX)
            dt = g / gp
            t -= dt
            if abs(dt) < mp.mpf(10) ** (-DPS + 5) or abs(t) > 3:
                break
        return t

    def solid_angle(self, x, nu, sg):
        """(Omega_0, dOmega_0/dnu') at target x (global), gauge u = sg * zhat (reading A8)."""
        with mp.workdps(DPS):
            r, nup = _mpv(x), _mpv(nu)
            u = [sg * c for c in self.zhat]
            Om0 = mp.mpf(0)
            dOm0 = mp.mpf(0)
            for e in range(3):
                t = self._closest(e, r)
                pts = [-1, t, 1] if -1 < t < 1 else [-1, 1]

                def f0(s, e=e):
                    xx, dx = self._eval(self.CX[e], s)
                    d = [r[i] - xx[i] for i in range(3)]
                    nd = mp.sqrt(_dot(d, d))
                    return -_dot(_cross(d, u), dx) / (nd * (nd + _dot(u, d)))

                def f1(s, e=e):
                    xx, _ = self._eval(self.CX[e], s)
                    tau, _ = self._eval(self.CT[e], s)
                    d = [r[i] - xx[i] for i in range(3)]
                    nd = mp.sqrt(_dot(d, d))
                    return _dot(nup, _cross(tau, d)) / nd ** 3
                Om0 += mp.quad(f0, pts)
                dOm0 += mp.quad(f1, pts)
            return float(Om0), float(dOm0)
