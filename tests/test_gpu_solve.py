"""the combined-field BIE solve of the exterior Dirichlet problem
through the C ABI (correction rows + rrq_apply_smooth), with a manufactured solution u = sum c_j / |x - r_j|,
r_j inside; E_inf of the evaluated solution at close and far exterior targets (eq
relativeerror).  Also the smooth-rule kernel against a numpy direct sum."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth.geometry import make_sphere_surface, make_interlocked_tori


def _exact(rng, inside_pts, scale=1.0):
    c = rng.normal(size=len(inside_pts))
    return lambda x: sum(c[j] / np.linalg.norm(x - inside_pts[j], axis=-1) for j in range(len(inside_pts)))


def test_smooth_kernel_vs_numpy():
    from paper_2411_08342_b200 import RRQ, DeviceSurface
    S = make_sphere_surface(2, 4, 8)
    ctx = RRQ(4)
    ds = DeviceSurface.from_numpy(S)
    xs = S.nodes.reshape(-1, 3); ns = S.normals.reshape(-1, 3); ws = S.weights.reshape(-1)
    rng = np.random.default_rng(0)
    sig = rng.normal(size=xs.shape[0])
    tx = np.concatenate([xs[:50], 1.3 * xs[50:80]])
    sn = np.concatenate([np.arange(50), -np.ones(30, np.int64)])
    d = tx[:, None, :] - xs[None]
    r = np.linalg.norm(d, axis=2)
    r[np.arange(50), np.arange(50)] = np.inf
    ref = (ws * sig / r).sum(1) / (4 * np.pi) * 0.7 + (ws * sig * np.einsum("tjk,jk->tj", d, ns) / r ** 3).sum(1) / (4 * np.pi) * 1.3
    g = lambda a, dt=torch.float64: torch.as_tensor(a, dtype=dt, device="cuda")
    y = ctx.apply_smooth(ds, g(tx), g(sn, torch.int64), g(sig), torch.zeros(80, dtype=torch.float64, device="cuda"),
                         alpha=0.7, beta=1.3).cpu().numpy()
    assert np.abs(y - ref).max() < 1e-12 * np.abs(ref).max()


def test_exterior_dirichlet_sphere_converges():
    e6, e8 = _sphere_solve(4, 6), _sphere_solve(4, 8)
    assert e6 < 1e-5 and e8 < 1e-7 and e8 < e6 / 30    # order-p convergence under p-refinement


def _sphere_solve(freq, p):
    from paper_2411_08342_b200.solve import CombinedFieldSolver
    S = make_sphere_surface(freq, p, 2 * p)
    rng = np.random.default_rng(4)
    src = rng.normal(size=(4, 3)); src = 0.5 * src / np.linalg.norm(src, axis=1, keepdims=True) * rng.random((4, 1))
    u = _exact(rng, src)
    solver = CombinedFieldSolver(S)
    xs = S.nodes.reshape(-1, 3); ns = S.normals.reshape(-1, 3)
    sigma, hist, its = solver.solve(u(xs), tol=1e-13)
    # close targets 10^-1 .. 10^-8 h off the surface above random surface points (not above nodes: the
    # smooth-rule subtraction of the splitting cancels catastrophically within 1e-6 h of a node itself,
    # a property of the splitting P:L1581-1598 that the evaluation grids of the paper never meet) and far ones
    h = 2 * np.pi / (5 * freq)
    q = rng.normal(size=(400, 3)); q /= np.linalg.norm(q, axis=1, keepdims=True)
    close = q * (1 + (10.0 ** -rng.uniform(1, 8, 400) * h))[:, None]
    far = rng.normal(size=(200, 3)); far = far / np.linalg.norm(far, axis=1, keepdims=True) * rng.uniform(1.3, 3, (200, 1))
    tx = np.concatenate([close, far])
    un = solver.evaluate(sigma, tx).cpu().numpy()
    ue = u(tx)
    err = np.abs(un - ue).max() / np.abs(ue).max()
    print(f"sphere freq {freq} p {p}: GMRES {its} iterations, residual {hist[-1]:.1e}, E_inf {err:.2e}")
    assert hist[-1] < 1e-12
    return err


def test_exterior_dirichlet_interlocked_tori():
    """The E4 boundary (four interlocking tori, 12 x 72 each -- the paper's second mesh, P:L1977-1979 --,
    p = 6) with a source inside each torus: solve, then evaluate at the exterior points of a 41^3 grid
    (close and far) as in Table 4 (E_inf 1.41e-6 at p = 6).  The 6 x 36 mesh does not
    resolve the density at the 0.05 gaps (E_inf 0.1 there, 3e-5 away from them)."""
    from paper_2411_08342_b200.solve import CombinedFieldSolver
    from synth.geometry import inside_interlocked_tori
    S = make_interlocked_tori(12, 72, 6, 12)
    rng = np.random.default_rng(6)
    # one source on each torus's core circle (inside the tube)
    src = []
    for k in range(4):
        ph = rng.uniform(0, 2 * np.pi)
        x, y, z = 3 * np.cos(ph), 3 * np.sin(ph), 0.0
        if k % 2:
            y, z = -z, y
        src.append([x + 4.95 * k, y, z])
    u = _exact(rng, np.array(src))
    solver = CombinedFieldSolver(S)
    xs = S.nodes.reshape(-1, 3)
    sigma, hist, its = solver.solve(u(xs), tol=1e-12, restart=120, maxiter=600)
    G = 41
    gx = np.linspace(-5.0, 20.0, G); gy = np.linspace(-6.0, 6.0, G)
    X = np.stack(np.meshgrid(gx, gy, gy, indexing="ij"), -1).reshape(-1, 3)
    X = X[~inside_interlocked_tori(X)]
    un = solver.evaluate(sigma, X).cpu().numpy()
    ue = u(X)
    err = np.abs(un - ue).max() / np.abs(ue).max()
    print(f"tori p 6: GMRES {its} iterations, residual {hist[-1]:.1e}, {X.shape[0]} grid targets, E_inf {err:.2e}")
    assert hist[-1] < 1e-11 and err < 3e-6     # measured 7.5e-7
