"""Combined-field BIE solve of the exterior Dirichlet problem on top of the correction builder (SURVEY
§8(f) NEXT(4)):

    u = (S + D)[sigma] in the exterior,   1/2 sigma + (S + D)[sigma] = f on the surface   (eq extdiribie),

discretised as smooth rule + near correction: A sigma = 1/2 sigma + (S + D)_smooth sigma
+ (C_S + C_D) sigma, with the smooth part from rrq_apply_smooth (direct sum; FMM is out of scope) and the
correction rows from rrq_build_correction at the nodes (self targets, principal value, A7).  The linear
system is solved by restarted GMRES (classical Gram-Schmidt applied twice, Givens rotations; one host
synchronisation per iteration) on device vectors; torch supplies only vector arithmetic and dot products (plumbing): every operator
application runs in the library's kernels.  Evaluation at off-surface targets builds their correction
rows the same way (close evaluation)."""
import numpy as np
import torch

from .rrq import RRQ, DeviceSurface, DeviceTargets, RRQ_S, RRQ_D


def gmres(matvec, b, tol=1e-12, restart=60, maxiter=400):
    """Restarted GMRES for A x = b (vectors of any torch device/dtype).  Returns (x, relative residual
    history per inner iteration, iterations)."""
    x = torch.zeros_like(b)
    bnorm = float(torch.linalg.vector_norm(b))
    if bnorm == 0.0:
        return x, [0.0], 0
    hist, it = [], 0
    while it < maxiter:
        r = b - matvec(x)
        beta = float(torch.linalg.vector_norm(r))
        hist.append(beta / bnorm)
        if beta / bnorm < tol:
            break
        m = min(restart, maxiter - it)
        # Krylov basis as one matrix; classical Gram-Schmidt applied twice (CGS2: as stable as modified
        # Gram-Schmidt with reorthogonalisation) so that an iteration costs two matrix-vector products with
        # the basis and ONE host synchronisation (the column of H and the new norm in one transfer)
        Vm = torch.empty((m + 1, b.shape[0]), dtype=b.dtype, device=b.device)
        Vm[0] = r / beta
        H = np.zeros((m + 1, m))
        g = np.zeros(m + 1); g[0] = beta
        cs, sn = np.zeros(m), np.zeros(m)
        k = 0
        for j in range(m):
            w = matvec(Vm[j])
            B = Vm[: j + 1]
            h1 = B @ w
            w = w - B.T @ h1
            h2 = B @ w
            w = w - B.T @ h2
            col = torch.cat([h1 + h2, torch.linalg.vector_norm(w).reshape(1)]).cpu().numpy()
            H[: j + 1, j] = col[: j + 1]
            hn = float(col[j + 1])
            H[j + 1, j] = hn
            for i in range(j):   # previous rotations
                a, c = H[i, j], H[i + 1, j]
                H[i, j], H[i + 1, j] = cs[i] * a + sn[i] * c, -sn[i] * a + cs[i] * c
            den = np.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = (1.0, 0.0) if den == 0 else (H[j, j] / den, H[j + 1, j] / den)
            H[j, j], H[j + 1, j] = den, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            it += 1
            k = j + 1
            hist.append(abs(g[j + 1]) / bnorm)
            if abs(g[j + 1]) / bnorm < tol or hn == 0.0:
                break
            Vm[j + 1] = w / hn
        y = np.linalg.solve(np.triu(H[:k, :k]), g[:k]) if k else np.zeros(0)
        if k:
            x = x + Vm[:k].T @ torch.as_tensor(y, dtype=b.dtype, device=b.device)
    return x, hist, it


class CombinedFieldSolver:
    """Exterior Dirichlet problem for Laplace on a closed surface S (numpy Surface of synth.geometry)."""

    def __init__(self, S, eta=1.5, device="cuda"):
        self.S, self.eta, self.dev = S, eta, device
        self.ctx = RRQ(S.p, eta=eta)
        self.ds = DeviceSurface.from_numpy(S, device)
        N = S.n_patches * S.n
        g = lambda a, dt=torch.float64: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=device)
        self.x = g(S.nodes.reshape(N, 3))
        self.self_node = torch.arange(N, dtype=torch.int64, device=device)
        dt = DeviceTargets(self.x, g(S.normals.reshape(N, 3)), self.self_node,
                           torch.zeros(N, dtype=torch.int8, device=device))
        self.fit, _ = self.ctx.patch_fit(self.ds)
        self.C = self._correction(dt)
        self.N = N

    def _correction(self, dt):
        ptr, pat = self.ctx.near_list(self.ds, dt)
        out = self.ctx.build_correction(self.ds, dt, ptr, pat, self.fit, mask=RRQ_S | RRQ_D, want_status=False)
        vals = out["vals"][0] + out["vals"][1]   # same sparsity: C_S + C_D
        return out["row_ptr"], out["col_idx"], vals

    def _apply(self, C, tx, self_node, sigma, y):
        self.ctx.apply_smooth(self.ds, tx, self_node, sigma, y, alpha=1.0, beta=1.0)
        rp, col, vals = C
        return self.ctx.apply_correction(rp, col, vals, sigma, y)

    def matvec(self, sigma):
        y = 0.5 * sigma
        return self._apply(self.C, self.x, self.self_node, sigma, y)

    def solve(self, f, tol=1e-12, restart=60, maxiter=400):
        f = torch.as_tensor(f, dtype=torch.float64, device=self.dev)
        return gmres(self.matvec, f, tol, restart, maxiter)

    def evaluate(self, sigma, tx_np, side=1):
        """u = (S + D)[sigma] at exterior targets (close ones get their correction rows)."""
        T = tx_np.shape[0]
        tx = torch.as_tensor(np.ascontiguousarray(tx_np), dtype=torch.float64, device=self.dev)
        dt = DeviceTargets(tx, None, None, torch.full((T,), side, dtype=torch.int8, device=self.dev))
        C = self._correction(dt)
        y = torch.zeros(T, dtype=torch.float64, device=self.dev)
        return self._apply(C, tx, None, sigma, y)
