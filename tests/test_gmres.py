"""Host logic of the combined-field solve (paper_2411_08342_b200/solve.py): restarted GMRES against a
dense direct solve (CPU, no GPU needed)."""
import numpy as np
import torch

from paper_2411_08342_b200.solve import gmres


def test_gmres_matches_direct_solve():
    rng = np.random.default_rng(0)
    n = 200
    A = np.eye(n) * 0.5 + rng.normal(size=(n, n)) / (4 * np.sqrt(n))   # second-kind-like spectrum
    b = rng.normal(size=n)
    At = torch.as_tensor(A)
    x, hist, its = gmres(lambda v: At @ v, torch.as_tensor(b), tol=1e-13, restart=30)
    xd = np.linalg.solve(A, b)
    assert hist[-1] < 1e-13
    assert np.abs(x.numpy() - xd).max() < 1e-11 * np.abs(xd).max()
    assert its > 30      # restarts exercised
