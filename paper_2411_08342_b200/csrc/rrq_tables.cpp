// Host-side constant tables of the CUDA path, built in __float128 and rounded once to fp64.
//  - Gauss-Legendre nodes / weights on (-1,1) ("the p~ Gauss-Legendre nodes"), by
//    Newton on the three-term recurrence started from Tricomi's asymptotic guess.
//  - U = V^{-1} through the Lagrange basis: row q of U holds the t^q coefficients of
//    L_k(t) = prod_{j!=k} (t - t_j)/(t_k - t_j), expanded by synthetic division of the master
//    polynomial prod_j (t - t_j).  In quad precision every entry is correctly rounded (DESIGN §2 A4).
// Independent of oracle/ (different algorithms; no shared code).
#include <quadmath.h>
#include <cmath>
#include <vector>

namespace rrq_host {

static __float128 legendre_and_deriv(int n, __float128 x, __float128 *dp) {
  __float128 p0 = 1, p1 = x;
  for (int k = 2; k <= n; ++k) {
    __float128 p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
    p0 = p1;
    p1 = p2;
  }
  *dp = n * (p0 - x * p1) / (1 - x * x);
  return p1;
}

void gauss_legendre(int n, double *x, double *w) {
  for (int i = 1; i <= n; ++i) {
    // Tricomi: x_i ~ (1 - (n-1)/(8 n^3)) cos(pi (4i - 1)/(4n + 2)), descending in i
    __float128 th = M_PIq * (4 * i - 1) / (4 * n + 2);
    __float128 xi = (1 - (__float128)(n - 1) / (8.0Q * n * n * n)) * cosq(th);
    __float128 dp = 1;
    for (int it = 0; it < 60; ++it) {
      __float128 p = legendre_and_deriv(n, xi, &dp);
      __float128 dx = p / dp;
      xi -= dx;
      if (fabsq(dx) <= 1e-34Q * (1 + fabsq(xi))) break;
    }
    legendre_and_deriv(n, xi, &dp);
    int k = n - i;  // ascending storage
    x[k] = (double)xi;
    w[k] = (double)(2 / ((1 - xi * xi) * dp * dp));
  }
}

void vandermonde_inverse(int n, const double *t, double *U) {
  std::vector<__float128> master(n + 1, 0), quo(n);
  master[0] = 1;  // coefficients, increasing powers: prod_j (t - t_j)
  for (int j = 0; j < n; ++j) {
    for (int c = j + 1; c >= 1; --c) master[c] = master[c - 1] - (__float128)t[j] * master[c];
    master[0] = -(__float128)t[j] * master[0];
  }
  for (int k = 0; k < n; ++k) {
    // synthetic division: master(t) = (t - t_k) quo(t)
    __float128 tk = t[k];
    quo[n - 1] = master[n];
    for (int c = n - 1; c >= 1; --c) quo[c - 1] = master[c] + tk * quo[c];
    __float128 den = 1;
    for (int j = 0; j < n; ++j)
      if (j != k) den *= (tk - (__float128)t[j]);
    for (int q = 0; q < n; ++q) U[q * n + k] = (double)(quo[q] / den);
  }
}

}  // namespace rrq_host
