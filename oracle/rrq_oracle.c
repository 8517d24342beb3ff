/*
 * rrq_oracle.c -- plain, slow, CPU ORACLE of the recursive reduction quadrature (RRQ) near correction
 * build of Jiang & Zhu, arXiv 2411.08342 ("PAPER.md").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header, table generator or
 * helper with the CUDA path (paper_2411_08342_b200/csrc, include/rrq.h) and imports nothing from it.
 *
 * It follows PAPER.md §4 "Close evaluation of the Laplace double layer potential", Steps 1-8
 * (P:L1397-1509), matrix mode, S / S' / D' (§3.3 Thm 3.3 P:L840-876,
 * §3.6, §3.7), with the readings of the silent / garbled points listed in
 * DESIGN.md §2 (G1-G5, A1-A15).  Every function names the passage
 * it follows.  Plain loops, no blocking, fusion or reordering beyond what the paper states; the
 * negative-k line integrals are computed directly (no conjugate-symmetry shortcut).
 *
 * PRECISION.  The arithmetic type `real` is chosen at compile time:
 *   default        fp64 ("the oracle", liboracle.so; also liboracle_fma.so built with FMA contraction)
 *   ORC_REAL_LD    x87 80-bit long double (liboracle_ld.so)
 *   ORC_REAL_QUAD  IEEE binary128 __float128 (liboracle_q.so): the TRUTH reference of the parity tests,
 *                  i.e. the same algorithm on the same fp64 inputs with ~34-digit arithmetic, constant
 *                  tables (Gauss-Legendre nodes/weights, U = V^{-1}) kept in quad and the Newton
 *                  tolerance scaled to the working precision.
 * Inputs and outputs at the C interface are always fp64 (the outputs are the real results rounded once).
 * The fp64 build can also run under any IEEE rounding mode (orc_params.rounding): the spread of those
 * runs around the truth measures what an fp64 evaluation of this formulation can attain.
 *
 * Citation key: P:Lnnn = /root/reference/PAPER.md line nnn (not read at run time).
 *
 * Pins (tests/test_oracle_*.py, all `-m "not gpu"`): Legendre vs scipy (textbook), solid harmonics
 * vs an independent sympy construction (P:L582 Pi_l^m form), addition theorem, Theorem 3.1 rank,
 * model integrals vs adaptive quadrature and closed forms, t0 closed form on straight edges,
 * Omega_0 vs Van Oosterom-Strackee, per-(l,m) W / Theta vs brute-force 2-form surface integrals
 * (Thm 3.4 / 3.5), D' vs finite differences, fit vs an independent least-squares solve, full
 * operator on the sphere (Gauss law, Y_l^m eigenrelations, Green's identity), close evaluation
 * against closed forms and adaptive quadrature down to 1e-14 h (tests/test_oracle_close.py), and the
 * precision ladder fp64 -> long double -> quad (tests/test_oracle_precision.py).  Parity unpinned:
 * none.
 */
#include <complex.h>
#include <fenv.h>
#include <math.h>
#include <quadmath.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------------------
 * The working precision.
 * ----------------------------------------------------------------------------------------------*/
#if defined(ORC_REAL_QUAD)
typedef __float128 real;
typedef __complex128 cplx;
#define RF(f) f##q
#define ISFIN(x) finiteq(x)
#define NEWTON_TOL 1e-32Q   /* ~ 50 ulp of binary128 */
#define NEWTON_MAXIT 30
#elif defined(ORC_REAL_LD)
typedef long double real;
typedef long double complex cplx;
#define RF(f) f##l
#define ISFIN(x) isfinite(x)
#define NEWTON_TOL 1e-18L   /* ~ 10 ulp of the 64-bit significand */
#define NEWTON_MAXIT 30
#else
typedef double real;
typedef double complex cplx;
#define RF(f) f
#define ISFIN(x) isfinite(x)
#define NEWTON_TOL 1e-15    /* reading A12 */
#define NEWTON_MAXIT 20
#endif
#define SQRT RF(sqrt)
#define FABS RF(fabs)
#define LOG RF(log)
#define ASINH RF(asinh)
#define SINH RF(sinh)
#define COSH RF(cosh)
#define COS RF(cos)
#define SIN RF(sin)
#define ATAN2 RF(atan2)
#define ACOS RF(acos)
#define POW RF(pow)
#define CABS RF(cabs)
#define CSQRT RF(csqrt)
#define CONJ RF(conj)
#define CRE(z) (__real__(z))
#define CIM(z) (__imag__(z))

static inline cplx mkc(real re, real im) {
  cplx z;
  __real__ z = re;
  __imag__ z = im;
  return z;
}
static inline real rmax2(real a, real b) { return a > b ? a : b; }
#define R_PI (ACOS((real)-1))

/* ------------------------------------------------------------------------------------------------
 * Parameters of one run (the discrete choices of DESIGN.md §2: p~ = 2p (A4), rho0 = 3 (A5),
 * n_Omega = 32 (A9), eta (A6)); `rounding`: IEEE rounding mode of the run (0 nearest, 1 upward,
 * 2 downward, 3 toward zero).
 * ----------------------------------------------------------------------------------------------*/
typedef struct {
  int p;          /* harmonic order */
  int q;          /* p~: edge Gauss-Legendre nodes per edge */
  int n_omega;    /* Gauss-Legendre nodes per side of the sinh split (A9) */
  double rho0;    /* Bernstein-ellipse threshold of the swap regime (A5) */
  int rounding;   /* IEEE rounding mode of the whole evaluation */
} orc_params;

static int fe_mode(int r) {
  switch (r) {
    case 1: return FE_UPWARD;
    case 2: return FE_DOWNWARD;
    case 3: return FE_TOWARDZERO;
    default: return FE_TONEAREST;
  }
}

/* ------------------------------------------------------------------------------------------------
 * Quad-precision constant tables.  Gauss-Legendre nodes ("the p~ Gauss-Legendre
 * nodes") and U = V^{-1} are computed in __float128 and rounded once to the working
 * precision (correctly rounded in fp64: DESIGN.md §2, A4).
 * ----------------------------------------------------------------------------------------------*/
static void gl_real(int n, real *x, real *w) {
  for (int i = 0; i < n; ++i) {
    __float128 t = cosq(M_PIq * (n - i - 0.25Q) / (n + 0.5Q)); /* ascending order */
    __float128 dp = 0;
    for (int it = 0; it < 100; ++it) {
      __float128 p0 = 1, p1 = t;
      for (int k = 2; k <= n; ++k) {
        __float128 p2 = ((2 * k - 1) * t * p1 - (k - 1) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      if (n == 1) { p1 = t; p0 = 1; }
      dp = n * (t * p1 - p0) / (t * t - 1);
      __float128 dt = p1 / dp;
      t -= dt;
      if (fabsq(dt) < 1e-33Q) break;
    }
    {
      __float128 p0 = 1, p1 = t;
      for (int k = 2; k <= n; ++k) {
        __float128 p2 = ((2 * k - 1) * t * p1 - (k - 1) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (t * p1 - p0) / (t * t - 1);
    }
    x[i] = (real)t;
    w[i] = (real)(2 / ((1 - t * t) * dp * dp));
  }
}

void orc_gauss_legendre(int n, double *x, double *w) {
  real *xr = malloc(sizeof(real) * n), *wr = malloc(sizeof(real) * n);
  gl_real(n, xr, wr);
  for (int i = 0; i < n; ++i) { x[i] = (double)xr[i]; w[i] = (double)wr[i]; }
  free(xr); free(wr);
}

/* U = V^{-1}, V_{kq} = t_k^q: Gauss-Jordan with partial pivoting in __float128 on the
 * working-precision nodes t (so V is exactly the Vandermonde of the nodes actually used).  U is
 * row-major [q][k]: c~_q = sum_k U[q][k] F_k. */
static void vandermonde_inverse_real(int n, const real *t, real *U) {
  __float128 *M = malloc(sizeof(__float128) * n * 2 * n);
  for (int k = 0; k < n; ++k) {
    __float128 tp = 1;
    for (int q = 0; q < n; ++q) {
      M[k * 2 * n + q] = tp;
      tp *= (__float128)t[k];
    }
    for (int q = 0; q < n; ++q) M[k * 2 * n + n + q] = (q == k);
  }
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (fabsq(M[r * 2 * n + c]) > fabsq(M[piv * 2 * n + c])) piv = r;
    if (piv != c)
      for (int j = 0; j < 2 * n; ++j) {
        __float128 tmp = M[c * 2 * n + j];
        M[c * 2 * n + j] = M[piv * 2 * n + j];
        M[piv * 2 * n + j] = tmp;
      }
    __float128 d = M[c * 2 * n + c];
    for (int j = 0; j < 2 * n; ++j) M[c * 2 * n + j] /= d;
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      __float128 f = M[r * 2 * n + c];
      if (f == 0) continue;
      for (int j = 0; j < 2 * n; ++j) M[r * 2 * n + j] -= f * M[c * 2 * n + j];
    }
  }
  /* M = [I | V^{-1}] with V^{-1}[q][k]: row q of V^{-1} maps samples F_k to coefficient q. */
  for (int q = 0; q < n; ++q)
    for (int k = 0; k < n; ++k) U[q * n + k] = (real)M[q * 2 * n + n + k];
  free(M);
}

void orc_vandermonde_inverse(int n, const double *t, double *U) {
  real *tr = calloc(n, sizeof(real)), *Ur = calloc((size_t)n * n, sizeof(real));
  for (int i = 0; i < n; ++i) tr[i] = t[i];
  vandermonde_inverse_real(n, tr, Ur);
  for (int i = 0; i < n * n; ++i) U[i] = (double)Ur[i];
  free(tr); free(Ur);
}

/* ------------------------------------------------------------------------------------------------
 * Harmonic polynomials.
 * ----------------------------------------------------------------------------------------------*/
static real fact(int n) {
  real f = 1;
  for (int i = 2; i <= n; ++i) f *= i;
  return f;
}

static real binom(int n, int k) {
  if (n < 0 || k < 0 || k > n) return 0;
  return fact(n) / (fact(k) * fact(n - k));
}

/* Associated Legendre P_l^m(x), 0<=m<=l<=p, by the recurrences of P:L338-345 (eq
 * associatelegendrerecurrence) with the diagonal sign of the Rodrigues formula P:L333 (no
 * Condon-Shortley phase, reading G5): P_{l+1}^{l+1} = +(2l+1) sqrt(1-x^2) P_l^l.  `s` is
 * sqrt(1-x^2), passed in so it can be formed accurately.  P[l*(p+1)+m]. */
static void legendre_real(int p, real x, real s, real *P) {
  int L = p + 1;
  for (int i = 0; i < L * L; ++i) P[i] = 0;
  P[0] = 1;
  for (int l = 0; l < p; ++l) {
    P[(l + 1) * L + (l + 1)] = (2 * l + 1) * s * P[l * L + l];
    P[(l + 1) * L + l] = (2 * l + 1) * x * P[l * L + l];
  }
  for (int m = 0; m <= p; ++m)
    for (int l = m + 1; l < p; ++l)
      P[(l + 1) * L + m] = ((2 * l + 1) * x * P[l * L + m] - (l + m) * P[(l - 1) * L + m]) / (l - m + 1);
}

void orc_legendre(int p, double x, double s, double *P) {
  int L = (p + 1) * (p + 1);
  real *Pr = malloc(sizeof(real) * L);
  legendre_real(p, x, s, Pr);
  for (int i = 0; i < L; ++i) P[i] = (double)Pr[i];
  free(Pr);
}

static inline int hidx(int l, int m) { return l * l + l + m; }

/* Regular solid harmonics R_l^m(X,Y,Z) = sqrt((l-m)!/(l+m)!) r^l P_l^m(cos theta) e^{i m phi}
 * (eqs ylmdef, rlmdef), 0<=l<=p, m>=0, and R_l^{-m} := (-1)^m conj(R_l^m) (reading G5).
 * Output R[hidx(l,m)], -l<=m<=l. */
static void solid_R_real(int p, real X, real Y, real Z, cplx *R) {
  int L = p + 1;
  for (int i = 0; i < L * L; ++i) R[i] = 0;
  R[0] = 1;
  real rho = SQRT(X * X + Y * Y);
  real r = SQRT(X * X + Y * Y + Z * Z);
  if (r == 0) return;
  real ct = Z / r, st = rho / r, phi = ATAN2(Y, X);
  real *P = malloc(sizeof(real) * L * L);
  legendre_real(p, ct, st, P);
  for (int l = 0; l <= p; ++l) {
    real rl = POW(r, (real)l);
    for (int m = 0; m <= l; ++m) {
      real N = SQRT(fact(l - m) / fact(l + m));
      real a = N * rl * P[l * L + m];
      cplx v = mkc(a * COS(m * phi), a * SIN(m * phi));
      R[hidx(l, m)] = v;
      if (m > 0) R[hidx(l, -m)] = ((m & 1) ? -1 : 1) * CONJ(v);
    }
  }
  free(P);
}

void orc_solid_R(int p, double X, double Y, double Z, double *out) {
  int L = (p + 1) * (p + 1);
  cplx *R = malloc(sizeof(cplx) * L);
  solid_R_real(p, X, Y, Z, R);
  for (int k = 0; k < L; ++k) { out[2 * k] = (double)CRE(R[k]); out[2 * k + 1] = (double)CIM(R[k]); }
  free(R);
}

static inline cplx Rget(const cplx *R, int l, int m) {
  if (l < 0 || m > l || m < -l) return 0;
  return R[hidx(l, m)];
}

/* First derivatives of R_l^m (reading A3, no-CS): dZ R_l^m = sqrt((l-m)(l+m)) R_{l-1}^m,
 * (dX + i dY) R_l^m = -sqrt((l-m)(l-m-1)) R_{l-1}^{m+1}, (dX - i dY) R_l^m = +sqrt((l+m)(l+m-1))
 * R_{l-1}^{m-1}.  Written as up to two terms (coef, l-1, m').  a = 0,1,2 for X,Y,Z. */
typedef struct { cplx c; int l, m; } term_t;

static int dR_terms(int l, int m, int a, term_t *t) {
  real cp = (l - m) * (real)(l - m - 1) > 0 ? SQRT((l - m) * (real)(l - m - 1)) : 0;
  real cm = (l + m) * (real)(l + m - 1) > 0 ? SQRT((l + m) * (real)(l + m - 1)) : 0;
  if (a == 2) {
    real cz = (l - m) * (real)(l + m) > 0 ? SQRT((l - m) * (real)(l + m)) : 0;
    t[0].c = cz; t[0].l = l - 1; t[0].m = m;
    return 1;
  }
  /* D+ = -cp R_{l-1}^{m+1}, D- = cm R_{l-1}^{m-1};  dX = (D+ + D-)/2, dY = (D+ - D-)/(2i) */
  if (a == 0) {
    t[0].c = -cp / 2; t[0].l = l - 1; t[0].m = m + 1;
    t[1].c = cm / 2;  t[1].l = l - 1; t[1].m = m - 1;
  } else {
    t[0].c = mkc(0, cp / 2); t[0].l = l - 1; t[0].m = m + 1;   /* -cp/(2i) = i cp/2 */
    t[1].c = mkc(0, cm / 2); t[1].l = l - 1; t[1].m = m - 1;   /* -cm/(2i) = i cm/2 */
  }
  return 2;
}

static cplx dR(const cplx *R, int l, int m, int a) {
  term_t t[2];
  int nt = dR_terms(l, m, a, t);
  cplx s = 0;
  for (int i = 0; i < nt; ++i) s += t[i].c * Rget(R, t[i].l, t[i].m);
  return s;
}

static cplx d2R(const cplx *R, int l, int m, int a, int b) {
  term_t t[2];
  int nt = dR_terms(l, m, a, t);
  cplx s = 0;
  for (int i = 0; i < nt; ++i)
    if (t[i].l >= 0 && t[i].m <= t[i].l && t[i].m >= -t[i].l) s += t[i].c * dR(R, t[i].l, t[i].m, b);
  return s;
}

/* S^{(l,m)}(x,y,z) = R_l^m(y,z,x) (eq slmdef).  Hence dS/dx = (dZ R), dS/dy = (dX R),
 * dS/dz = (dY R), all evaluated at (y,z,x).  AX[a] = R-axis of S-axis a. */
static const int AX[3] = {2, 0, 1};

typedef struct {
  int p;
  cplx *S;   /* [(p+1)^2]      S^{(l,m)}          */
  cplx *G;   /* [(p+1)^2][3]   grad S^{(l,m)}     */
  cplx *H;   /* [(p+1)^2][3][3] Hess S^{(l,m)} (NULL if not requested) */
} htab_t;

static void htab_alloc(htab_t *h, int p, int with_hess) {
  int L = (p + 1) * (p + 1);
  h->p = p;
  h->S = malloc(sizeof(cplx) * L);
  h->G = malloc(sizeof(cplx) * L * 3);
  h->H = with_hess ? malloc(sizeof(cplx) * L * 9) : NULL;
}
static void htab_free(htab_t *h) { free(h->S); free(h->G); free(h->H); }

static void htab_eval(htab_t *h, real x, real y, real z) {
  int p = h->p;
  cplx *R = malloc(sizeof(cplx) * (p + 1) * (p + 1));
  solid_R_real(p, y, z, x, R);
  for (int l = 0; l <= p; ++l)
    for (int m = -l; m <= l; ++m) {
      int k = hidx(l, m);
      h->S[k] = R[k];
      for (int a = 0; a < 3; ++a) h->G[3 * k + a] = dR(R, l, m, AX[a]);
      if (h->H)
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) h->H[9 * k + 3 * a + b] = d2R(R, l, m, AX[a], AX[b]);
    }
  free(R);
}

/* Test hook: S, grad S, Hess S at one point, interleaved re/im. */
void orc_harmonics_S(int p, double x, double y, double z, double *S, double *G, double *Hs) {
  htab_t h;
  htab_alloc(&h, p, Hs != NULL);
  htab_eval(&h, x, y, z);
  int L = (p + 1) * (p + 1);
  for (int k = 0; k < L; ++k) {
    S[2 * k] = (double)CRE(h.S[k]); S[2 * k + 1] = (double)CIM(h.S[k]);
    for (int a = 0; a < 3; ++a) { G[6 * k + 2 * a] = (double)CRE(h.G[3 * k + a]); G[6 * k + 2 * a + 1] = (double)CIM(h.G[3 * k + a]); }
    if (Hs)
      for (int a = 0; a < 9; ++a) { Hs[18 * k + 2 * a] = (double)CRE(h.H[9 * k + a]); Hs[18 * k + 2 * a + 1] = (double)CIM(h.H[9 * k + a]); }
  }
  htab_free(&h);
}

/* T_{jk,lm} = C(l+m, j+k)^{1/2} C(l-m, j-k)^{1/2} (eq tjklmdef), zero out of range. */
static real Tjklm(int j, int k, int l, int m) { return SQRT(binom(l + m, j + k) * binom(l - m, j - k)); }
/* C_{j,l} = (j-2)!(l-j)!/(l-1)! and D_{j,l} = (j-1)!(l-j)!/l!. */
static real Cjl(int j, int l) { return fact(j - 2) * fact(l - j) / fact(l - 1); }
static real Djl(int j, int l) { return fact(j - 1) * fact(l - j) / fact(l); }

/* (l,m), 1<=m<=l<=p -> basis index (P:L465-466 enumerates l=1..p, m=1..l). */
static inline int lmidx(int l, int m) { return l * (l - 1) / 2 + (m - 1); }

/* ------------------------------------------------------------------------------------------------
 * Quaternions (eq qprule): fg = (f0 g0 - f.g, f0 g + g0 f + f x g), complex components.
 * ----------------------------------------------------------------------------------------------*/
typedef struct { cplx s, v[3]; } quat;

static quat qmul(quat f, quat g) {
  quat r;
  r.s = f.s * g.s - (f.v[0] * g.v[0] + f.v[1] * g.v[1] + f.v[2] * g.v[2]);
  cplx c[3] = {f.v[1] * g.v[2] - f.v[2] * g.v[1], f.v[2] * g.v[0] - f.v[0] * g.v[2], f.v[0] * g.v[1] - f.v[1] * g.v[0]};
  for (int a = 0; a < 3; ++a) r.v[a] = f.s * g.v[a] + g.s * f.v[a] + c[a];
  return r;
}
static quat qzero(void) { quat r; r.s = 0; r.v[0] = r.v[1] = r.v[2] = 0; return r; }
static quat qvec(cplx a, cplx b, cplx c) { quat r; r.s = 0; r.v[0] = a; r.v[1] = b; r.v[2] = c; return r; }
static quat qscale(quat f, cplx a) { quat r; r.s = a * f.s; for (int i = 0; i < 3; ++i) r.v[i] = a * f.v[i]; return r; }
static quat qadd(quat f, quat g) { quat r; r.s = f.s + g.s; for (int i = 0; i < 3; ++i) r.v[i] = f.v[i] + g.v[i]; return r; }

/* Test hook: quaternion product on real quaternions. */
void orc_qmul(const double *f, const double *g, double *out) {
  quat a = {f[0], {f[1], f[2], f[3]}}, b = {g[0], {g[1], g[2], g[3]}};
  quat r = qmul(a, b);
  out[0] = (double)CRE(r.s);
  for (int i = 0; i < 3; ++i) out[1 + i] = (double)CRE(r.v[i]);
}

/* ------------------------------------------------------------------------------------------------
 * Dense least squares: Moore-Penrose pseudo-inverse by Householder QR (reading A1).
 * A is m x k row-major (m >= k), Aplus is k x m row-major.  Returns 1 if rank deficient.
 * ----------------------------------------------------------------------------------------------*/
static int pinv_qr_real(int m, int k, const real *A, real *Aplus) {
  real *W = malloc(sizeof(real) * m * k);
  real *V = calloc((size_t)m * k, sizeof(real)); /* reflector vectors, column j in V[:,j] */
  real *beta = calloc(k, sizeof(real));
  memcpy(W, A, sizeof(real) * m * k);
  int deficient = 0;
  real rmax = 0;
  for (int j = 0; j < k; ++j) {
    real nrm = 0;
    for (int i = j; i < m; ++i) nrm += W[i * k + j] * W[i * k + j];
    nrm = SQRT(nrm);
    real alpha = (W[j * k + j] > 0) ? -nrm : nrm;
    for (int i = j; i < m; ++i) V[i * k + j] = W[i * k + j];
    V[j * k + j] -= alpha;
    real b = 0;
    for (int i = j; i < m; ++i) b += V[i * k + j] * V[i * k + j];
    beta[j] = b;
    if (b > 0)
      for (int c = j; c < k; ++c) {
        real s = 0;
        for (int i = j; i < m; ++i) s += V[i * k + j] * W[i * k + c];
        s = 2 * s / b;
        for (int i = j; i < m; ++i) W[i * k + c] -= s * V[i * k + j];
      }
    if (FABS(W[j * k + j]) > rmax) rmax = FABS(W[j * k + j]);
  }
  for (int j = 0; j < k; ++j)
    if (!(FABS(W[j * k + j]) > (real)1e-13 * rmax)) deficient = 1;
  /* Q^T e_c for each column c, first k rows; then R^{-1} by back substitution. */
  real *e = malloc(sizeof(real) * m);
  for (int c = 0; c < m; ++c) {
    for (int i = 0; i < m; ++i) e[i] = (i == c);
    for (int j = 0; j < k; ++j) {
      if (beta[j] <= 0) continue;
      real s = 0;
      for (int i = j; i < m; ++i) s += V[i * k + j] * e[i];
      s = 2 * s / beta[j];
      for (int i = j; i < m; ++i) e[i] -= s * V[i * k + j];
    }
    for (int r = k - 1; r >= 0; --r) {
      real s = e[r];
      for (int cc = r + 1; cc < k; ++cc) s -= W[r * k + cc] * e[cc];
      e[r] = s / W[r * k + r];
    }
    for (int r = 0; r < k; ++r) Aplus[r * m + c] = e[r];
  }
  free(e); free(W); free(V); free(beta);
  return deficient;
}

int orc_pinv_qr(int m, int k, const double *A, double *Aplus) {
  real *Ar = calloc((size_t)m * k, sizeof(real)), *Pr = calloc((size_t)m * k, sizeof(real));
  for (int i = 0; i < m * k; ++i) Ar[i] = A[i];
  int st = pinv_qr_real(m, k, Ar, Pr);
  for (int i = 0; i < m * k; ++i) Aplus[i] = (double)Pr[i];
  free(Ar); free(Pr);
  return st;
}

/* ------------------------------------------------------------------------------------------------
 * Patch: local frame (reading A2), fit operators (Steps 1-2 in matrix mode, reading A1; P:L715-746,
 * P:L846-865), edge tables (Step 3).
 * ----------------------------------------------------------------------------------------------*/
typedef struct {
  int p, q, n, np;
  real o[3], Rm[3][3], h;     /* local = Rm (x - o) / h */
  real *xl, *nl;              /* [n][3] local nodes, normals */
  real vl[3][3];              /* local vertices */
  real *yl, *tl;              /* [3q][3] local edge samples, tangents d y / d t */
  real *C;                    /* [3][q][3] Legendre coefficients of each edge interpolant (A4, A4') */
  real zlo, zhi;
  cplx *g;                    /* [3q][(p+1)^2][3] Hess S^{(j,k)}(y) tau */
  cplx *e;                    /* [3q][(p+1)^2][3] grad S^{(j,k)}(y) x tau */
  real *fit;                  /* [13 np][n]: P_D (4np), P_Sp (4np), P_Sd (np), P_Sg (4np) */
  int status;
} patch_t;

static void cross3(const real *a, const real *b, real *c) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}
static real dot3(const real *a, const real *b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static real norm3(const real *a) { return SQRT(dot3(a, a)); }

/* Reading A2: origin = vertex centroid, z = normalise((v1-v0) x (v2-v0)), e1 = normalise(v1-v0),
 * e2 = z x e1, coordinates scaled by 1/h_P (h_P = max vertex chord, A6). */
static void patch_frame(const double *verts, real o[3], real Rm[3][3], real *h) {
  real v0[3], v1[3], v2[3];
  for (int i = 0; i < 3; ++i) { v0[i] = verts[i]; v1[i] = verts[3 + i]; v2[i] = verts[6 + i]; }
  real a[3], b[3], z[3], e1[3], e2[3];
  for (int i = 0; i < 3; ++i) { o[i] = (v0[i] + v1[i] + v2[i]) / 3; a[i] = v1[i] - v0[i]; b[i] = v2[i] - v0[i]; }
  cross3(a, b, z);
  real nz = norm3(z), na = norm3(a);
  for (int i = 0; i < 3; ++i) { z[i] /= nz; e1[i] = a[i] / na; }
  cross3(z, e1, e2);
  for (int i = 0; i < 3; ++i) { Rm[0][i] = e1[i]; Rm[1][i] = e2[i]; Rm[2][i] = z[i]; }
  real c = 0;
  for (int e = 0; e < 3; ++e) {
    real d[3];
    for (int i = 0; i < 3; ++i) d[i] = (real)verts[3 * ((e + 1) % 3) + i] - (real)verts[3 * e + i];
    real l = norm3(d);
    if (l > c) c = l;
  }
  *h = c;
}

static void to_local(const patch_t *P, const double *x, real *y) {
  real d[3] = {(real)x[0] - P->o[0], (real)x[1] - P->o[1], (real)x[2] - P->o[2]};
  for (int r = 0; r < 3; ++r) y[r] = dot3(P->Rm[r], d) / P->h;
}
static void rot_local(const patch_t *P, const double *v, real *y) {
  real vr[3] = {v[0], v[1], v[2]};
  for (int r = 0; r < 3; ++r) y[r] = dot3(P->Rm[r], vr);
}

static void patch_build(patch_t *P, const orc_params *pr, const double *nodes, const double *normals,
                        const double *verts, const double *edge_x, const double *edge_dx, int want_fit) {
  int p = pr->p, q = pr->q, n = p * p, np = p * (p + 1) / 2, L = (p + 1) * (p + 1);
  P->p = p; P->q = q; P->n = n; P->np = np;
  patch_frame(verts, P->o, P->Rm, &P->h);
  P->xl = malloc(sizeof(real) * n * 3);
  P->nl = malloc(sizeof(real) * n * 3);
  P->yl = malloc(sizeof(real) * 3 * q * 3);
  P->tl = malloc(sizeof(real) * 3 * q * 3);
  P->C = malloc(sizeof(real) * 3 * q * 3);
  for (int i = 0; i < n; ++i) { to_local(P, nodes + 3 * i, P->xl + 3 * i); rot_local(P, normals + 3 * i, P->nl + 3 * i); }
  for (int v = 0; v < 3; ++v) to_local(P, verts + 3 * v, P->vl[v]);
  for (int k = 0; k < 3 * q; ++k) {
    to_local(P, edge_x + 3 * k, P->yl + 3 * k);
    rot_local(P, edge_dx + 3 * k, P->tl + 3 * k);
    for (int a = 0; a < 3; ++a) P->tl[3 * k + a] /= P->h;
  }
  /* Edge interpolants (reading A4): the degree q-1 interpolant of the samples, held as a Legendre
   * series x(t) = sum_j C_j P_j(t) (reading A4': same polynomial as the monomial form c~ = U y of
   * P:L1231, but evaluated without the cond(V) amplification of monomials).  Gauss-Legendre exactness
   * gives the discrete transform C_j = (2j+1)/2 sum_k W_k P_j(t_k) y_k. */
  {
    real tg[64], wg[64];
    gl_real(q, tg, wg);
    for (int e = 0; e < 3; ++e)
      for (int a = 0; a < 3; ++a)
        for (int j = 0; j < q; ++j) P->C[(e * q + j) * 3 + a] = 0;
    for (int k = 0; k < q; ++k) {
      real Pj[64];
      Pj[0] = 1;
      if (q > 1) Pj[1] = tg[k];
      for (int j = 1; j + 1 < q; ++j) Pj[j + 1] = ((2 * j + 1) * tg[k] * Pj[j] - j * Pj[j - 1]) / (j + 1);
      for (int e = 0; e < 3; ++e)
        for (int j = 0; j < q; ++j)
          for (int a = 0; a < 3; ++a)
            P->C[(e * q + j) * 3 + a] += (real)0.5 * (2 * j + 1) * wg[k] * Pj[j] * P->yl[3 * (e * q + k) + a];
    }
  }
  /* height range of nodes, vertices, edge samples (reading A8) */
  P->zlo = 1e300; P->zhi = -1e300;
  for (int i = 0; i < n; ++i) { real z = P->xl[3 * i + 2]; if (z < P->zlo) P->zlo = z; if (z > P->zhi) P->zhi = z; }
  for (int v = 0; v < 3; ++v) { real z = P->vl[v][2]; if (z < P->zlo) P->zlo = z; if (z > P->zhi) P->zhi = z; }
  for (int k = 0; k < 3 * q; ++k) { real z = P->yl[3 * k + 2]; if (z < P->zlo) P->zlo = z; if (z > P->zhi) P->zhi = z; }

  /* Step 3: harmonics at the 3 p~ edge nodes. */
  P->g = malloc(sizeof(cplx) * 3 * q * L * 3);
  P->e = malloc(sizeof(cplx) * 3 * q * L * 3);
  htab_t ht;
  htab_alloc(&ht, p, 1);
  for (int k = 0; k < 3 * q; ++k) {
    htab_eval(&ht, P->yl[3 * k], P->yl[3 * k + 1], P->yl[3 * k + 2]);
    const real *t = P->tl + 3 * k;
    for (int j = 0; j <= p; ++j)
      for (int kk = -j; kk <= j; ++kk) {
        int hk = hidx(j, kk);
        cplx *gg = P->g + ((size_t)k * L + hk) * 3, *ee = P->e + ((size_t)k * L + hk) * 3;
        for (int a = 0; a < 3; ++a) {
          gg[a] = 0;
          for (int b = 0; b < 3; ++b) gg[a] += ht.H[9 * hk + 3 * a + b] * t[b]; /* d(grad S)/dt */
        }
        const cplx *G = ht.G + 3 * hk;
        ee[0] = G[1] * t[2] - G[2] * t[1];
        ee[1] = G[2] * t[0] - G[0] * t[2];
        ee[2] = G[0] * t[1] - G[1] * t[0];
      }
  }
  htab_free(&ht);

  P->fit = NULL;
  P->status = 0;
  if (!want_fit) return;
  /* Steps 1-2: F_{i,lm} = grad H^{(l,m)}(x_i), H^{(l,m)} = sqrt(2) Im S^{(l,m)} (G5). */
  const real s2 = SQRT((real)2);
  real *F = malloc(sizeof(real) * 3 * n * np);  /* F[a][i][lm] */
  real *Hm = malloc(sizeof(real) * n * np);
  htab_t hn;
  htab_alloc(&hn, p, 0);
  for (int i = 0; i < n; ++i) {
    htab_eval(&hn, P->xl[3 * i], P->xl[3 * i + 1], P->xl[3 * i + 2]);
    for (int l = 1; l <= p; ++l)
      for (int m = 1; m <= l; ++m) {
        int c = lmidx(l, m), hk = hidx(l, m);
        for (int a = 0; a < 3; ++a) F[(a * n + i) * np + c] = s2 * CIM(hn.G[3 * hk + a]);
        Hm[i * np + c] = s2 * CIM(hn.S[hk]);
      }
  }
  htab_free(&hn);
  /* A: 4n x 4np block matrix of P:L729-735 (eq dlpdensitylinearsystem2). */
  int M4 = 4 * n, K4 = 4 * np;
  real *A = calloc((size_t)M4 * K4, sizeof(real));
  /* block (r, c) of [[0,-F1,-F2,-F3],[F1,0,-F3,F2],[F2,F3,0,-F1],[F3,-F2,F1,0]] */
  const int blk[4][4] = {{0, -1, -2, -3}, {1, 0, -3, 2}, {2, 3, 0, -1}, {3, -2, 1, 0}};
  for (int br = 0; br < 4; ++br)
    for (int bc = 0; bc < 4; ++bc) {
      int s = blk[br][bc];
      if (s == 0) continue;
      int a = abs(s) - 1;
      real sg = s > 0 ? 1 : -1;
      for (int i = 0; i < n; ++i)
        for (int c = 0; c < np; ++c) A[(size_t)(br * n + i) * K4 + bc * np + c] = sg * F[(a * n + i) * np + c];
    }
  real *Ap = malloc(sizeof(real) * K4 * M4);
  int st = pinv_qr_real(M4, K4, A, Ap);
  /* B_{i,lm} = grad H^{(l,m)}(x_i) . nu_i */
  real *B = malloc(sizeof(real) * n * np), *Bp = malloc(sizeof(real) * np * n);
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < np; ++c) {
      real s = 0;
      for (int a = 0; a < 3; ++a) s += F[(a * n + i) * np + c] * P->nl[3 * i + a];
      B[i * np + c] = s;
    }
  st |= pinv_qr_real(n, np, B, Bp);
  real *fit = calloc((size_t)13 * np * n, sizeof(real));
  real *PD = fit, *PSp = fit + 4 * np * n, *PSd = fit + 8 * np * n, *PSg = fit + 9 * np * n;
  for (int r = 0; r < K4; ++r)
    for (int i = 0; i < n; ++i) {
      PD[r * n + i] = Ap[r * M4 + i];  /* RHS (mu, 0, 0, 0) */
      real s = 0;                       /* RHS (0, sigma nu) */
      for (int a = 0; a < 3; ++a) s += P->nl[3 * i + a] * Ap[r * M4 + (a + 1) * n + i];
      PSp[r * n + i] = s;
    }
  for (int r = 0; r < np; ++r)
    for (int i = 0; i < n; ++i) PSd[r * n + i] = Bp[r * n + i];
  /* P_Sg = P_D Hm P_Sd : rho = sum_lm H d at the nodes, then the quaternion fit of (rho, 0)
   * (P:L857-865). */
  real *HP = malloc(sizeof(real) * n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      real s = 0;
      for (int c = 0; c < np; ++c) s += Hm[i * np + c] * PSd[c * n + j];
      HP[i * n + j] = s;
    }
  for (int r = 0; r < K4; ++r)
    for (int j = 0; j < n; ++j) {
      real s = 0;
      for (int i = 0; i < n; ++i) s += PD[r * n + i] * HP[i * n + j];
      PSg[r * n + j] = s;
    }
  P->fit = fit;
  P->status = st;
  free(F); free(Hm); free(A); free(Ap); free(B); free(Bp); free(HP);
}

static void patch_free(patch_t *P) {
  free(P->xl); free(P->nl); free(P->yl); free(P->tl); free(P->C); free(P->g); free(P->e); free(P->fit);
}

/* ------------------------------------------------------------------------------------------------
 * Singularity-swap quadrature per edge (Step 5; readings A4, A5, A11, A12).
 * ----------------------------------------------------------------------------------------------*/
/* x(t), x'(t), x''(t) of the Legendre series C (reading A4'), complex t: Bonnet's recurrence
 * (j+1)P_{j+1} = (2j+1) t P_j - j P_{j-1} and P'_{j+1} = P'_{j-1} + (2j+1) P_j,
 * P''_{j+1} = P''_{j-1} + (2j+1) P'_j. */
static void edge_eval(const real *C, int q, cplx t, cplx *x, cplx *dx, cplx *ddx) {
  cplx P0 = 1, P1 = t, d0 = 0, d1 = 1, e0 = 0, e1 = 0;
  for (int a = 0; a < 3; ++a) {
    x[a] = C[a] * P0;
    dx[a] = 0;
    ddx[a] = 0;
  }
  if (q > 1)
    for (int a = 0; a < 3; ++a) { x[a] += C[3 + a] * P1; dx[a] += C[3 + a] * d1; }
  for (int j = 1; j + 1 < q; ++j) {
    cplx P2 = ((2 * j + 1) * t * P1 - j * P0) / (real)(j + 1);
    cplx d2 = d0 + (2 * j + 1) * P1;
    cplx e2 = e0 + (2 * j + 1) * d1;
    for (int a = 0; a < 3; ++a) {
      real c = C[(j + 1) * 3 + a];
      x[a] += c * P2;
      dx[a] += c * d2;
      ddx[a] += c * e2;
    }
    P0 = P1; P1 = P2; d0 = d1; d1 = d2; e0 = e1; e1 = e2;
  }
}

/* Bernstein ellipse parameter rho(t0) = |t0 + sqrt(t0^2 - 1)|, branch with rho >= 1 (reading A5). */
static real bernstein_rho_real(real re, real im) {
  cplx t = mkc(re, im);
  cplx s = CSQRT(t * t - 1);
  real r1 = CABS(t + s), r2 = CABS(t - s);
  return r1 > r2 ? r1 : r2;
}

double orc_bernstein_rho(double re, double im) { return (double)bernstein_rho_real(re, im); }

/* Reading A12: complex root t0 of sum_c (x_c(t) - r'_c)^2 = 0 (eq complexparameter).
 * Returns 1 if converged.  Im t0 >= 0.  Reading A12': the iteration also stops (as converged) once,
 * after at least one complex step, the step is below 1e-3 |t| and rho(t) > rho_stop (= 2 rho0): the
 * root is then certainly outside the swap ellipse, so the regime decision is already fixed and t0 is
 * not used by the plain rule.  Reading A12'': it also stops once the iteration is in its quadratic
 * regime (|dt| < 0.1 |dt_prev|) and the predicted next step C |dt|^2, C ~ |dt| / |dt_prev|^2, is below the
 * tolerance NEWTON_TOL (1 + |t|): the updated t is then already converged (Newton's quadratic
 * convergence).  NEWTON_TOL = 1e-15 in fp64 (A12), scaled to the working precision otherwise. */
static int find_t0_real(const real *C, int q, const real *rp, real rho_stop, real *t0re, real *t0im) {
  cplx x[3], dx[3], ddx[3];
  /* chord projection */
  edge_eval(C, q, -1, x, dx, ddx);
  real A[3] = {CRE(x[0]), CRE(x[1]), CRE(x[2])};
  edge_eval(C, q, 1, x, dx, ddx);
  real Bv[3] = {CRE(x[0]), CRE(x[1]), CRE(x[2])};
  real ab[3] = {Bv[0] - A[0], Bv[1] - A[1], Bv[2] - A[2]}, ar[3] = {rp[0] - A[0], rp[1] - A[1], rp[2] - A[2]};
  real tc = -1 + 2 * dot3(ar, ab) / dot3(ab, ab);
  /* 3 real Newton steps on g(t) = (x(t) - r').x'(t) */
  for (int it = 0; it < 3; ++it) {
    edge_eval(C, q, tc, x, dx, ddx);
    real g = 0, gp = 0;
    for (int a = 0; a < 3; ++a) {
      real xr = CRE(x[a]) - rp[a];
      g += xr * CRE(dx[a]);
      gp += CRE(dx[a]) * CRE(dx[a]) + xr * CRE(ddx[a]);
    }
    if (!(gp > 0)) break;
    tc -= g / gp;
  }
  /* quadratic-model guess t_c + i sqrt(2 f / f''), f = |x - r'|^2, f'' = 2 (|x'|^2 + (x-r').x'') */
  edge_eval(C, q, tc, x, dx, ddx);
  real f = 0, dd = 0, xp2 = 0;
  for (int a = 0; a < 3; ++a) {
    real xr = CRE(x[a]) - rp[a];
    f += xr * xr;
    dd += CRE(dx[a]) * CRE(dx[a]) + xr * CRE(ddx[a]);
    xp2 += CRE(dx[a]) * CRE(dx[a]);
  }
  if (!(dd > 0)) dd = xp2;
  cplx t = mkc(tc, SQRT(f / dd));
  int conv = 0;
  real dprev = 0;
  for (int it = 0; it < NEWTON_MAXIT; ++it) {
    edge_eval(C, q, t, x, dx, ddx);
    cplx F = 0, Fp = 0;
    for (int a = 0; a < 3; ++a) {
      cplx xr = x[a] - rp[a];
      F += xr * xr;
      Fp += 2 * xr * dx[a];
    }
    cplx dt = F / Fp;
    t -= dt;
    const real ad = CABS(dt), tol = NEWTON_TOL * (1 + CABS(t));
    if (ad < tol) { conv = 1; break; }
    if (dprev > 0 && ad < (real)0.1 * dprev && ad * ad * ad < tol * dprev * dprev) { conv = 1; break; }   /* A12'' */
    if (it >= 1 && ad < (real)1e-3 * CABS(t) && bernstein_rho_real(CRE(t), CIM(t)) > rho_stop) { conv = 1; break; }
    dprev = ad;
  }
  if (CIM(t) < 0) t = CONJ(t);
  *t0re = CRE(t);
  *t0im = CIM(t);
  return conv && ISFIN(CRE(t)) && ISFIN(CIM(t));
}

int orc_find_t0(const double *C, int q, const double *rp, double rho_stop, double *t0re, double *t0im) {
  real Cr[64 * 3], rr[3] = {rp[0], rp[1], rp[2]}, a, b;
  for (int i = 0; i < 3 * q; ++i) Cr[i] = C[i];
  int conv = find_t0_real(Cr, q, rr, rho_stop, &a, &b);
  *t0re = (double)a;
  *t0im = (double)b;
  return conv;
}

/* Model integrals (reading A11, App. A.4): with a = Re t0, b = |Im t0|, Q(t) = (t-a)^2 + b^2,
 * I_k = int_{-1}^{1} t^k Q^{-1/2} dt, J_k = int t^k Q^{-3/2} dt, k = 0..q-1, by upward recurrences
 * ("calculated by a recurrence relation").  I_0 and J_0 in cancellation-free form. */
static void model_integrals_real(real a, real b, int q, real *Iv, real *Jv) {
  real Q1 = (1 - a) * (1 - a) + b * b, Qm = (1 + a) * (1 + a) + b * b;
  real s1 = SQRT(Q1), sm = SQRT(Qm);
  real I0, J0;
  if (FABS(a) <= 1) {
    I0 = ASINH((1 - a) / b) + ASINH((1 + a) / b);
    J0 = ((1 - a) / s1 + (1 + a) / sm) / (b * b);
  } else {
    real aa = FABS(a), u = aa + 1, v = aa - 1;
    real su = SQRT(u * u + b * b), sv = SQRT(v * v + b * b);
    I0 = LOG((u + su) / (v + sv));
    J0 = 4 * aa / (su * sv * (u * sv + v * su));
  }
  Iv[0] = I0;
  Jv[0] = J0;
  real a2b2 = a * a + b * b;
  for (int k = 1; k < q; ++k) {
    real sgn = ((k - 1) & 1) ? -1 : 1;                 /* (-1)^{k-1} */
    real beta = s1 - sgn * sm;                         /* [t^{k-1} sqrt(Q)]_{-1}^{1} */
    real gam = 1 / s1 - sgn / sm;                      /* [t^{k-1} Q^{-1/2}]_{-1}^{1} */
    if (k == 1) {
      Iv[1] = beta + a * Iv[0];
      Jv[1] = a * Jv[0] - gam;
    } else {
      Iv[k] = (beta + (2 * k - 1) * a * Iv[k - 1] - (k - 1) * a2b2 * Iv[k - 2]) / k;
      Jv[k] = a * Jv[k - 1] - gam + (k - 1) * Iv[k - 2];
    }
  }
}

void orc_model_integrals(double a, double b, int q, double *Iv, double *Jv) {
  real Ir[64], Jr[64];
  model_integrals_real(a, b, q, Ir, Jr);
  for (int k = 0; k < q; ++k) { Iv[k] = (double)Ir[k]; Jv[k] = (double)Jr[k]; }
}

/* Reading A11': where t0 lies outside the Bernstein ellipse rho = RHO_DIRECT the upward recurrences
 * amplify rounding (App. B.8: 1e-10..2e-7 near rho0 = 3 at p~ = 20), while the model integrands
 * t^k |t - t0|^{-m} are analytic inside that ellipse; there the same integrals are evaluated by an
 * N_DIRECT-point Gauss-Legendre rule (error ~ rho^{-2 N_DIRECT} < 1e-17).  Inside it, the recurrences
 * (accurate to ~1e-14 for |t0| <~ 1.1) are used. */
#define RHO_DIRECT 1.6
#define N_DIRECT 48
static void model_integrals_direct_real(real a, real b, int q, const real *x, const real *w, real *Iv, real *Jv) {
  for (int k = 0; k < q; ++k) { Iv[k] = 0; Jv[k] = 0; }
  for (int j = 0; j < N_DIRECT; ++j) {
    real Qv = (x[j] - a) * (x[j] - a) + b * b;
    real r1 = w[j] / SQRT(Qv), r3 = r1 / Qv, tk = 1;
    for (int k = 0; k < q; ++k) {
      Iv[k] += tk * r1;
      Jv[k] += tk * r3;
      tk *= x[j];
    }
  }
}

void orc_model_integrals_direct(double a, double b, int q, double *Iv, double *Jv) {
  real Ir[64], Jr[64], x[N_DIRECT], w[N_DIRECT];
  gl_real(N_DIRECT, x, w);
  model_integrals_direct_real(a, b, q, x, w, Ir, Jr);
  for (int k = 0; k < q; ++k) { Iv[k] = (double)Ir[k]; Jv[k] = (double)Jr[k]; }
}

/* Per-edge quadrature data for one target. */
typedef struct {
  real w1[64], w3[64];     /* omega^{(1)}_k, omega^{(3)}_k (q <= 64) */
  real om0;                /* this edge's contribution to Omega_0 */
  real t0re, t0im;
  int swap, conv;
} edgeq_t;

/* Constant tables of one run, in the working precision. */
typedef struct {
  real tgl[64], wgl[64], U[64 * 64], xo[256], wo[256], xd[N_DIRECT], wd[N_DIRECT];
} tables_t;

static void tables_init(tables_t *T, const orc_params *pr) {
  gl_real(pr->q, T->tgl, T->wgl);
  vandermonde_inverse_real(pr->q, T->tgl, T->U);
  gl_real(pr->n_omega, T->xo, T->wo);
  gl_real(N_DIRECT, T->xd, T->wd);
}

/* Step 5 for edge e: regime, t0, weights omega^{(m)}_k = [M^T U]_k |t_k - t0|^m / |d_k|^m
 * in the swap regime, w_k / |d_k|^m in the plain regime (readings A4, A5); and Omega_0's edge
 * integral by the sinh-split rule (reading A9) or plain Gauss-Legendre. */
static void edge_quadrature(const patch_t *P, const orc_params *pr, const tables_t *T, int e, const real *rp,
                            const real *u, edgeq_t *E) {
  int q = P->q;
  const real *C = P->C + e * q * 3;
  const real rho0 = pr->rho0;
  real t0r, t0i;
  int conv = find_t0_real(C, q, rp, 2 * rho0, &t0r, &t0i);
  E->t0re = t0r; E->t0im = t0i; E->conv = conv;
  E->swap = conv && (bernstein_rho_real(t0r, t0i) < rho0);
  real dn[64];
  for (int k = 0; k < q; ++k) {
    const real *y = P->yl + 3 * (e * q + k);
    real d[3] = {rp[0] - y[0], rp[1] - y[1], rp[2] - y[2]};
    dn[k] = norm3(d);
  }
  if (E->swap) {
    real Iv[64], Jv[64];
    if (bernstein_rho_real(t0r, t0i) >= (real)RHO_DIRECT) model_integrals_direct_real(t0r, FABS(t0i), q, T->xd, T->wd, Iv, Jv);
    else model_integrals_real(t0r, FABS(t0i), q, Iv, Jv);
    for (int k = 0; k < q; ++k) {
      real mu1 = 0, mu3 = 0;
      for (int c = 0; c < q; ++c) { mu1 += Iv[c] * T->U[c * q + k]; mu3 += Jv[c] * T->U[c * q + k]; }
      real tt = SQRT((T->tgl[k] - t0r) * (T->tgl[k] - t0r) + t0i * t0i);
      real r1 = tt / dn[k];
      E->w1[k] = mu1 * r1;
      E->w3[k] = mu3 * r1 * r1 * r1;
    }
    /* Omega_0 on this edge: t = a + b sinh(s), n_Omega GL nodes on each side of a (reading A9) */
    real a = t0r < -1 ? -1 : (t0r > 1 ? 1 : t0r), b = FABS(t0i);
    real sR = ASINH((1 - a) / b), sL = ASINH((-1 - a) / b);
    real acc = 0;
    for (int side = 0; side < 2; ++side) {
      real lo = side ? 0 : sL, hi = side ? sR : 0;
      if (hi <= lo) continue;
      for (int j = 0; j < pr->n_omega; ++j) {
        real s = lo + (hi - lo) * (T->xo[j] + 1) / 2, W = (hi - lo) / 2 * T->wo[j];
        real t = a + b * SINH(s), dt = b * COSH(s);
        cplx x[3], dx[3], ddx[3];
        edge_eval(C, q, t, x, dx, ddx);
        real d[3] = {rp[0] - CRE(x[0]), rp[1] - CRE(x[1]), rp[2] - CRE(x[2])};
        real tau[3] = {CRE(dx[0]), CRE(dx[1]), CRE(dx[2])};
        real dxu[3];
        cross3(d, u, dxu);
        real nd = norm3(d);
        acc += W * dt * (-(dot3(dxu, tau)) / (nd * (nd + dot3(u, d))));
      }
    }
    E->om0 = acc;
  } else {
    real acc = 0;
    for (int k = 0; k < q; ++k) {
      E->w1[k] = T->wgl[k] / dn[k];
      E->w3[k] = T->wgl[k] / (dn[k] * dn[k] * dn[k]);
      const real *y = P->yl + 3 * (e * q + k), *tau = P->tl + 3 * (e * q + k);
      real d[3] = {rp[0] - y[0], rp[1] - y[1], rp[2] - y[2]}, dxu[3];
      cross3(d, u, dxu);
      acc += T->wgl[k] * (-(dot3(dxu, tau)) / (dn[k] * (dn[k] + dot3(u, d))));
    }
    E->om0 = acc;
  }
}

/* Reading A8: gauge u = sigma_P z (local frame), Dirac string r' + s u (s > 0) must miss P. */
static real gauge_sign(const patch_t *P, const real *rp, int side, int is_self) {
  if (is_self) return -1;
  real z = rp[2] - P->vl[0][2];
  if (z > P->zhi + (real)0.1) return 1;   /* h_P = 1 in local scaled units */
  if (z < P->zlo - (real)0.1) return -1;
  /* barycentric coordinates of the projection in the vertex triangle */
  const real *a = P->vl[0], *b = P->vl[1], *c = P->vl[2];
  real det = (b[0] - a[0]) * (c[1] - a[1]) - (c[0] - a[0]) * (b[1] - a[1]);
  real l1 = ((rp[0] - a[0]) * (c[1] - a[1]) - (c[0] - a[0]) * (rp[1] - a[1])) / det;
  real l2 = ((b[0] - a[0]) * (rp[1] - a[1]) - (rp[0] - a[0]) * (b[1] - a[1])) / det;
  real l0 = 1 - l1 - l2;
  real mn = l0 < l1 ? l0 : l1;
  if (l2 < mn) mn = l2;
  if (mn >= (real)-0.25 && side != 2) return side > 0 ? 1 : -1;  /* side == 2: flag absent */
  real mid = (P->zlo + P->zhi) / 2;
  return (z - mid > 0) ? 1 : -1;
}

/* ------------------------------------------------------------------------------------------------
 * One (target, patch) pair: Steps 4-8 for S, D, S', D' in matrix mode.
 * rows[4][n] (S, D, S', D') in GLOBAL units; dbg (optional) receives intermediates.
 * ----------------------------------------------------------------------------------------------*/
typedef struct {
  real om0, om[3], dom0, dom[3];
  real t0[3][2];
  int swap[3], conv[3];
  double *W, *dW, *Th;     /* [np][4], [np][4], [np] (rounded to fp64) */
} pair_dbg;

static int pair_rows(const patch_t *P, const orc_params *pr, const tables_t *T, const double *x_glob,
                     const double *nu_glob, int self_local, int side, unsigned mask, int raw, const double *nodes_glob,
                     const double *normals_glob, const double *weights_glob, real *rows, pair_dbg *dbg) {
  int p = P->p, q = P->q, n = P->n, np = P->np, L = (p + 1) * (p + 1);
  const real inv4pi = 1 / (4 * R_PI), s2 = SQRT((real)2);
  int is_self = self_local >= 0;
  int status = 0;
  real rp[3], nup[3] = {0, 0, 0};
  to_local(P, x_glob, rp);
  if (nu_glob) rot_local(P, nu_glob, nup);

  /* Step 4: S, grad S, Hess S at the target. */
  htab_t ht;
  htab_alloc(&ht, p, 1);
  htab_eval(&ht, rp[0], rp[1], rp[2]);

  /* gauge (A8) and Step 5 per edge */
  real sg = gauge_sign(P, rp, side, is_self);
  real u[3] = {0, 0, sg};
  edgeq_t E[3];
  for (int e = 0; e < 3; ++e) {
    edge_quadrature(P, pr, T, e, rp, u, &E[e]);
    if (!E[e].conv) status |= 1;
  }

  /* Step 6: line integrals (P:L1196-1211 eq lineintegrals, P:L1362-1376 eq dprimelineintegrals). */
  real Om0 = 0, Om[3] = {0, 0, 0}, dOm0 = 0, dOm[3] = {0, 0, 0};
  quat *Qt = malloc(sizeof(quat) * L), *dQt = malloc(sizeof(quat) * L);
  cplx *Vt = malloc(sizeof(cplx) * L);
  for (int k = 0; k < L; ++k) { Qt[k] = qzero(); dQt[k] = qzero(); Vt[k] = 0; }
  for (int e = 0; e < 3; ++e) {
    Om0 += E[e].om0;
    for (int kk = 0; kk < q; ++kk) {
      int kap = e * q + kk;
      const real *y = P->yl + 3 * kap, *tau = P->tl + 3 * kap;
      real d[3] = {rp[0] - y[0], rp[1] - y[1], rp[2] - y[2]};
      real w1 = E[e].w1[kk], w3 = E[e].w3[kk];
      real nd = dot3(nup, d);
      for (int a = 0; a < 3; ++a) {
        Om[a] -= w1 * tau[a];            /* Omega = - int dr / |r' - r| */
        dOm[a] += w3 * nd * tau[a];      /* dOmega/dnu' = int (nu'.(r'-r)) dr / |r'-r|^3 */
      }
      real txd[3];
      cross3(tau, d, txd);
      dOm0 += w3 * dot3(nup, txd);       /* Biot-Savart form of dOmega_0/dnu' (reading A10) */
      quat qd = qvec(d[0], d[1], d[2]);
      quat qb = qvec(w1 * nup[0] - w3 * nd * d[0], w1 * nup[1] - w3 * nd * d[1], w1 * nup[2] - w3 * nd * d[2]);
      for (int j = 1; j <= p; ++j)
        for (int k = -j; k <= j; ++k) {
          int hk = hidx(j, k);
          const cplx *gg = P->g + ((size_t)kap * L + hk) * 3, *ee = P->e + ((size_t)kap * L + hk) * 3;
          if (j >= 2) {
            quat qg = qvec(gg[0], gg[1], gg[2]);
            /* Q^{(j,k)} = int (0, (r'-r)/|r'-r|)(0, d grad S^{(j,k)})  (eq qjkdef2) */
            Qt[hk] = qadd(Qt[hk], qscale(qmul(qd, qg), w1));
            /* dQ/dnu' */
            dQt[hk] = qadd(dQt[hk], qmul(qb, qg));
          }
          /* V^{(j,k)} = int (1/|r'-r|) [(r'-r) x grad S^{(j,k)}] . dr  (eq vjkdef) */
          Vt[hk] += w1 * (d[0] * ee[0] + d[1] * ee[1] + d[2] * ee[2]);
        }
    }
  }
  /* reading G1: Omega_0 := solid angle = - sum of the printed omega_0 (the sign is folded into the
   * edge integrand above).  Reading A7: self targets use u = -z and the principal value shift. */
  if (is_self) Om0 -= 2 * R_PI;

  /* Step 7: translation (P:L1263-1268 eq cdlp1dintegral, reading G2). */
  real *Wr = calloc(np * 4, sizeof(real)), *dWr = calloc(np * 4, sizeof(real)), *Th = calloc(np, sizeof(real));
  quat Omq = {Om0, {Om[0], Om[1], Om[2]}}, dOmq = {dOm0, {dOm[0], dOm[1], dOm[2]}};
  for (int l = 1; l <= p; ++l)
    for (int m = 1; m <= l; ++m) {
      quat lam = qzero(), dlam = qzero();
      cplx th = 0;
      for (int j = 1; j <= l; ++j)
        for (int k = -j; k <= j; ++k) {
          int mk = m - k, lj = l - j;
          if (mk > lj || mk < -lj) continue;
          real Tv = Tjklm(j, k, l, m);
          if (Tv == 0) continue;
          int hk = hidx(j, k), hs = hidx(lj, mk);
          cplx Sv = ht.S[hs];
          cplx nuGS = nup[0] * ht.G[3 * hs] + nup[1] * ht.G[3 * hs + 1] + nup[2] * ht.G[3 * hs + 2];
          if (j >= 2) {
            real cT = Cjl(j, l) * Tv;
            lam = qadd(lam, qscale(Qt[hk], cT * Sv));
            dlam = qadd(dlam, qadd(qscale(dQt[hk], cT * Sv), qscale(Qt[hk], cT * nuGS)));
          }
          th += Djl(j, l) * Tv * Vt[hk] * Sv;
        }
      int hl = hidx(l, m);
      const cplx *GS = ht.G + 3 * hl, *HS = ht.H + 9 * hl;
      quat gq = qvec(GS[0], GS[1], GS[2]);
      cplx hn[3];
      for (int a = 0; a < 3; ++a) hn[a] = HS[3 * a] * nup[0] + HS[3 * a + 1] * nup[1] + HS[3 * a + 2] * nup[2];
      quat hq = qvec(hn[0], hn[1], hn[2]);
      quat gam = qmul(Omq, gq);                                  /* I[gamma] * 4 pi, omega first */
      quat dgam = qadd(qmul(dOmq, gq), qmul(Omq, hq));
      quat tot = qscale(qadd(lam, gam), inv4pi), dtot = qscale(qadd(dlam, dgam), inv4pi);
      int c = lmidx(l, m);
      /* W = -sqrt(2) Im(I[lambda_1] + I[gamma]) (eq wlmdef) */
      Wr[4 * c] = -s2 * CIM(tot.s);
      dWr[4 * c] = -s2 * CIM(dtot.s);
      for (int a = 0; a < 3; ++a) { Wr[4 * c + 1 + a] = -s2 * CIM(tot.v[a]); dWr[4 * c + 1 + a] = -s2 * CIM(dtot.v[a]); }
      /* Theta = sqrt(2) Im I[theta_1],  I[theta_1] = (1/4pi)[sum D T V S + S(r') Omega_0] (G2) */
      Th[c] = s2 * CIM(inv4pi * (th + ht.S[hl] * Om0));
    }

  /* Step 8, matrix mode (reading G3 for S'; Thm 3.3 for S). */
  const real *PD = P->fit, *PSp = P->fit + 4 * np * n, *PSd = P->fit + 8 * np * n, *PSg = P->fit + 9 * np * n;
  real *rS = rows, *rD = rows + n, *rSp = rows + 2 * n, *rDp = rows + 3 * n;
  for (int i = 0; i < 4 * n; ++i) rows[i] = 0;
  for (int c = 0; c < np; ++c) {
    real zW[4] = {Wr[4 * c], -Wr[4 * c + 1], -Wr[4 * c + 2], -Wr[4 * c + 3]};
    real zdW[4] = {dWr[4 * c], -dWr[4 * c + 1], -dWr[4 * c + 2], -dWr[4 * c + 3]};
    const real *Wv = Wr + 4 * c + 1;
    real nxW[3];
    cross3(nup, Wv, nxW);
    real zS[4] = {-dot3(nup, Wv), -Wr[4 * c] * nup[0] - nxW[0], -Wr[4 * c] * nup[1] - nxW[1],
                  -Wr[4 * c] * nup[2] - nxW[2]};
    for (int b = 0; b < 4; ++b) {
      const real *pd = PD + (b * np + c) * n, *psp = PSp + (b * np + c) * n, *psg = PSg + (b * np + c) * n;
      for (int i = 0; i < n; ++i) {
        rD[i] += zW[b] * pd[i];
        rDp[i] += zdW[b] * pd[i];
        rSp[i] += zS[b] * psp[i];
        rS[i] += zW[b] * psg[i];
      }
    }
    for (int i = 0; i < n; ++i) rS[i] += Th[c] * PSd[c * n + i];
  }
  /* back to global units (reading A2): S rows scale with h, D' rows with 1/h */
  for (int i = 0; i < n; ++i) { rS[i] *= P->h; rDp[i] /= P->h; }

  /* smooth-rule subtraction (reading A14), skipping the self node */
  if (!raw)
    for (int i = 0; i < n; ++i) {
      if (i == self_local) continue;
      const double *x = nodes_glob + 3 * i, *nu = normals_glob + 3 * i;
      real d[3] = {(real)x_glob[0] - x[0], (real)x_glob[1] - x[1], (real)x_glob[2] - x[2]};
      real nur[3] = {nu[0], nu[1], nu[2]};
      real r = norm3(d), r3 = r * r * r, w = weights_glob[i];
      real dn = dot3(d, nur);
      rS[i] -= inv4pi / r * w;
      rD[i] -= inv4pi * dn / r3 * w;
      if (nu_glob) {
        real nug[3] = {nu_glob[0], nu_glob[1], nu_glob[2]};
        real dnp = dot3(d, nug);
        rSp[i] -= -inv4pi * dnp / r3 * w;
        rDp[i] -= inv4pi * (dot3(nur, nug) / r3 - 3 * dn * dnp / (r3 * r * r)) * w;
      }
    }
  if (!(mask & 1)) for (int i = 0; i < n; ++i) rS[i] = 0;
  if (!(mask & 2)) for (int i = 0; i < n; ++i) rD[i] = 0;
  if (!(mask & 4)) for (int i = 0; i < n; ++i) rSp[i] = 0;
  if (!(mask & 8)) for (int i = 0; i < n; ++i) rDp[i] = 0;
  for (int i = 0; i < 4 * n; ++i)
    if (!ISFIN(rows[i])) status |= 2;

  if (dbg) {
    dbg->om0 = Om0; dbg->dom0 = dOm0;
    for (int a = 0; a < 3; ++a) { dbg->om[a] = Om[a]; dbg->dom[a] = dOm[a]; }
    for (int e = 0; e < 3; ++e) { dbg->t0[e][0] = E[e].t0re; dbg->t0[e][1] = E[e].t0im; dbg->swap[e] = E[e].swap; dbg->conv[e] = E[e].conv; }
    if (dbg->W) for (int i = 0; i < 4 * np; ++i) dbg->W[i] = (double)Wr[i];
    if (dbg->dW) for (int i = 0; i < 4 * np; ++i) dbg->dW[i] = (double)dWr[i];
    if (dbg->Th) for (int i = 0; i < np; ++i) dbg->Th[i] = (double)Th[i];
  }
  free(Qt); free(dQt); free(Vt); free(Wr); free(dWr); free(Th);
  htab_free(&ht);
  return status;
}

/* ------------------------------------------------------------------------------------------------
 * Public oracle entry points (called from tests via ctypes).  Inputs and outputs are fp64.
 * ----------------------------------------------------------------------------------------------*/

/* Fit block of each patch, [P][13 np][n] (P_D, P_Sp, P_Sd, P_Sg, local scaled frame). */
void orc_patch_fit(int64_t n_patches, int p, int q, const double *nodes, const double *normals, const double *verts,
                   const double *edge_x, const double *edge_dx, double *fit_out, int32_t *status, int rounding) {
  orc_params pr = {p, q, 32, 3.0, rounding};
  int n = p * p, np = p * (p + 1) / 2;
  const int mode = fe_mode(rounding);
#pragma omp parallel
  {
    const int saved = fegetround();
    fesetround(mode);
#pragma omp for schedule(dynamic)
    for (int64_t P = 0; P < n_patches; ++P) {
      patch_t pt;
      patch_build(&pt, &pr, nodes + P * n * 3, normals + P * n * 3, verts + P * 9, edge_x + P * 3 * q * 3,
                  edge_dx + P * 3 * q * 3, 1);
      for (int i = 0; i < 13 * np * n; ++i) fit_out[P * 13 * np * n + i] = (double)pt.fit[i];
      if (status) status[P] = pt.status;
      patch_free(&pt);
    }
    fesetround(saved);
  }
}

/* Rows of pairs (pair_target[k], pair_patch[k]) for S, D, S', D' -> vals[4][n_pairs][n]; status
 * bit0 Newton fallback, bit1 nonfinite, bit2 rank-deficient patch fit; zeta (optional) [n_pairs][9 np]:
 * the Step 4-7 outputs Theta, W, dW of each pair (local scaled frame).  Pairs are processed
 * patch by patch (Steps 1-3 once per patch).  The whole evaluation runs in the IEEE
 * rounding mode prm->rounding (each OpenMP thread sets and restores its own mode). */
void orc_build_rows(const orc_params *prm, int64_t n_patches, const double *nodes, const double *normals,
                    const double *weights, const double *verts, const double *edge_x, const double *edge_dx,
                    const double *tx, const double *tnormal, const int64_t *self_node, const int8_t *side,
                    int64_t n_pairs, const int64_t *pair_target, const int32_t *pair_patch, uint32_t mask, int raw,
                    double *vals, int32_t *pair_status, double *zeta) {
  orc_params pr = *prm;
  int p = pr.p, q = pr.q, n = p * p;
  tables_t *T = malloc(sizeof(tables_t));
  tables_init(T, &pr);
  /* group pairs by patch (stable) */
  int64_t *cnt = calloc(n_patches + 1, sizeof(int64_t)), *ord = malloc(sizeof(int64_t) * (n_pairs + 1));
  for (int64_t k = 0; k < n_pairs; ++k) cnt[pair_patch[k] + 1]++;
  for (int64_t P = 0; P < n_patches; ++P) cnt[P + 1] += cnt[P];
  int64_t *fill = malloc(sizeof(int64_t) * (n_patches + 1));
  memcpy(fill, cnt, sizeof(int64_t) * (n_patches + 1));
  for (int64_t k = 0; k < n_pairs; ++k) ord[fill[pair_patch[k]]++] = k;
  free(fill);
  const int mode = fe_mode(pr.rounding);
#pragma omp parallel
  {
    const int saved = fegetround();
    fesetround(mode);
#pragma omp for schedule(dynamic)
    for (int64_t P = 0; P < n_patches; ++P) {
      if (cnt[P + 1] == cnt[P]) continue;
      patch_t pt;
      patch_build(&pt, &pr, nodes + P * n * 3, normals + P * n * 3, verts + P * 9, edge_x + P * 3 * q * 3,
                  edge_dx + P * 3 * q * 3, 1);
      real *rows = malloc(sizeof(real) * 4 * n);
      for (int64_t s = cnt[P]; s < cnt[P + 1]; ++s) {
        int64_t k = ord[s], t = pair_target[k];
        int self_local = -1;
        if (self_node && self_node[t] >= 0 && self_node[t] / n == P) self_local = (int)(self_node[t] % n);
        int sd = side ? side[t] : 2;
        pair_dbg dbg, *dp = NULL;
        if (zeta) {   /* Steps 4-7 output of this pair: Theta [np], W [np][4], dW [np][4] */
          const int np = pt.np;
          dbg.Th = zeta + (size_t)k * 9 * np;
          dbg.W = dbg.Th + np;
          dbg.dW = dbg.W + 4 * np;
          dp = &dbg;
        }
        int st = pair_rows(&pt, &pr, T, tx + 3 * t, tnormal ? tnormal + 3 * t : NULL, self_local, sd, mask, raw,
                           nodes + P * n * 3, normals + P * n * 3, weights + P * n, rows, dp);
        if (pt.status) st |= 4;
        for (int kk = 0; kk < 4; ++kk)
          for (int i = 0; i < n; ++i) vals[((size_t)kk * n_pairs + k) * n + i] = (double)rows[kk * n + i];
        if (pair_status) pair_status[k] = st;
      }
      free(rows);
      patch_free(&pt);
    }
    fesetround(saved);
  }
  free(cnt); free(ord); free(T);
}

/* Debug entry for one pair: intermediates (Omega_0, Omega, derivatives, t0, regimes, W, dW, Theta),
 * frame (o, Rm, h) and the 4 rows.  out layout documented in oracle/oracle.py. */
int orc_pair_debug(const orc_params *prm, const double *nodes, const double *normals, const double *weights,
                   const double *verts, const double *edge_x, const double *edge_dx, const double *x,
                   const double *nu, int self_local, int side, int raw, double *rows, double *scal, double *W,
                   double *dW, double *Th, double *frame) {
  orc_params pr = *prm;
  const int saved = fegetround();
  fesetround(fe_mode(pr.rounding));
  tables_t *T = malloc(sizeof(tables_t));
  tables_init(T, &pr);
  patch_t pt;
  patch_build(&pt, &pr, nodes, normals, verts, edge_x, edge_dx, 1);
  pair_dbg dbg;
  dbg.W = W; dbg.dW = dW; dbg.Th = Th;
  int n = pt.n;
  real *rr = malloc(sizeof(real) * 4 * n);
  int st = pair_rows(&pt, &pr, T, x, nu, self_local, side, 15u, raw, nodes, normals, weights, rr, &dbg);
  for (int i = 0; i < 4 * n; ++i) rows[i] = (double)rr[i];
  free(rr);
  scal[0] = (double)dbg.om0;
  for (int a = 0; a < 3; ++a) scal[1 + a] = (double)dbg.om[a];
  scal[4] = (double)dbg.dom0;
  for (int a = 0; a < 3; ++a) scal[5 + a] = (double)dbg.dom[a];
  for (int e = 0; e < 3; ++e) {
    scal[8 + 4 * e] = (double)dbg.t0[e][0];
    scal[9 + 4 * e] = (double)dbg.t0[e][1];
    scal[10 + 4 * e] = dbg.swap[e];
    scal[11 + 4 * e] = dbg.conv[e];
  }
  if (frame) {
    for (int a = 0; a < 3; ++a) frame[a] = (double)pt.o[a];
    for (int a = 0; a < 9; ++a) frame[3 + a] = (double)pt.Rm[a / 3][a % 3];
    frame[12] = (double)pt.h;
  }
  patch_free(&pt);
  free(T);
  fesetround(saved);
  return st;
}

/* Batched debug entry: many targets against ONE patch (the patch, its fit and edge tables built once).
 * Per target: rows [4][n] and scal[20] as in orc_pair_debug (Omega_0, Omega, dOmega_0, dOmega, t0/regime
 * per edge); self_local[i] < 0 for non-self targets, side[i] as in orc_pair_debug, nu may be NULL. */
void orc_pairs_debug(const orc_params *prm, const double *nodes, const double *normals, const double *weights,
                     const double *verts, const double *edge_x, const double *edge_dx, int64_t n_targets,
                     const double *x, const double *nu, const int32_t *self_local, const int32_t *side, int raw,
                     double *rows, double *scal, int32_t *status) {
  orc_params pr = *prm;
  tables_t *T = malloc(sizeof(tables_t));
  tables_init(T, &pr);
  patch_t pt;
  patch_build(&pt, &pr, nodes, normals, verts, edge_x, edge_dx, 1);
  const int n = pt.n;
#pragma omp parallel
  {
    const int saved = fegetround();
    fesetround(fe_mode(pr.rounding));
    real *rr = malloc(sizeof(real) * 4 * n);
#pragma omp for schedule(dynamic)
    for (int64_t i = 0; i < n_targets; ++i) {
      pair_dbg dbg;
      dbg.W = dbg.dW = dbg.Th = NULL;
      int st = pair_rows(&pt, &pr, T, x + 3 * i, nu ? nu + 3 * i : NULL, self_local ? self_local[i] : -1,
                         side ? side[i] : 2, 15u, raw, nodes, normals, weights, rr, &dbg);
      for (int k = 0; k < 4 * n; ++k) rows[i * 4 * n + k] = (double)rr[k];
      double *sc = scal + i * 20;
      sc[0] = (double)dbg.om0;
      for (int a = 0; a < 3; ++a) sc[1 + a] = (double)dbg.om[a];
      sc[4] = (double)dbg.dom0;
      for (int a = 0; a < 3; ++a) sc[5 + a] = (double)dbg.dom[a];
      for (int e = 0; e < 3; ++e) {
        sc[8 + 4 * e] = (double)dbg.t0[e][0];
        sc[9 + 4 * e] = (double)dbg.t0[e][1];
        sc[10 + 4 * e] = dbg.swap[e];
        sc[11 + 4 * e] = dbg.conv[e];
      }
      if (status) status[i] = st;
    }
    free(rr);
    fesetround(saved);
  }
  patch_free(&pt);
  free(T);
}

/* ------------------------------------------------------------------------------------------------
 * Near list (reading A6), fp64 in every build (integer work: the decision is taken in the kernel's
 * precision).  Balls: c_P = sum_i w_i x_i / sum_i w_i summed sequentially over i,
 * R_P = max distance of nodes, vertices and edge samples from c_P, h_P = max vertex chord; every
 * product and sum is a separately rounded IEEE operation (no contraction: -ffp-contract=off), the
 * order the CUDA path reproduces with __dmul_rn / __dadd_rn.
 * ----------------------------------------------------------------------------------------------*/
#pragma GCC push_options
#pragma GCC optimize("fp-contract=off")
static double dnorm3(double a, double b, double c) { return sqrt(a * a + b * b + c * c); }

static void near_ball(int n, int q, const double *nodes, const double *weights, const double *verts,
                      const double *edge_x, double *ball) {
  double c[3] = {0, 0, 0}, ws = 0;
  for (int i = 0; i < n; ++i) {
    double w = weights[i];
    ws += w;
    for (int a = 0; a < 3; ++a) c[a] += w * nodes[i * 3 + a];
  }
  for (int a = 0; a < 3; ++a) c[a] /= ws;
  double R = 0;
  for (int i = 0; i < n; ++i) {
    double r = dnorm3(nodes[i * 3] - c[0], nodes[i * 3 + 1] - c[1], nodes[i * 3 + 2] - c[2]);
    if (r > R) R = r;
  }
  for (int v = 0; v < 3; ++v) {
    double r = dnorm3(verts[3 * v] - c[0], verts[3 * v + 1] - c[1], verts[3 * v + 2] - c[2]);
    if (r > R) R = r;
  }
  for (int k = 0; k < 3 * q; ++k) {
    const double *y = edge_x + k * 3;
    double r = dnorm3(y[0] - c[0], y[1] - c[1], y[2] - c[2]);
    if (r > R) R = r;
  }
  double h = 0;
  for (int e = 0; e < 3; ++e) {
    const double *a = verts + 3 * e, *b = verts + 3 * ((e + 1) % 3);
    double l = dnorm3(b[0] - a[0], b[1] - a[1], b[2] - a[2]);
    if (l > h) h = l;
  }
  ball[0] = c[0]; ball[1] = c[1]; ball[2] = c[2]; ball[3] = R; ball[4] = h;
}

/* Test hook: the balls (c, R, h) of all patches. */
void orc_near_balls(int64_t n_patches, int p, int q, const double *nodes, const double *weights, const double *verts,
                    const double *edge_x, double *ball) {
  int n = p * p;
  for (int64_t P = 0; P < n_patches; ++P)
    near_ball(n, q, nodes + P * n * 3, weights + P * n, verts + P * 9, edge_x + P * 3 * q * 3, ball + P * 5);
}

static int near_test(const double *tx, const double *b, double eta) {
  return dnorm3(tx[0] - b[0], tx[1] - b[1], tx[2] - b[2]) <= b[3] + eta * b[4];
}

/* near(t, P) iff |t - c_P| <= R_P + eta h_P, or t is a node of P; all pairs if all_pairs.  Brute force
 * O(N_T N_P).  Two-phase: counts into pair_ptr (size T+1, exclusive scan), then fill if pair_patch !=
 * NULL. */
void orc_near_list(int64_t n_patches, int p, int q, const double *nodes, const double *weights, const double *verts,
                   const double *edge_x, int64_t n_targets, const double *tx, const int64_t *self_node, double eta,
                   int all_pairs, int64_t *pair_ptr, int32_t *pair_patch) {
  int n = p * p;
  double *ball = malloc(sizeof(double) * n_patches * 5);
  orc_near_balls(n_patches, p, q, nodes, weights, verts, edge_x, ball);
  int fill = pair_patch != NULL;
  if (!fill) pair_ptr[0] = 0;
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < n_targets; ++t) {
    int64_t k = fill ? pair_ptr[t] : 0, c = 0;
    for (int64_t P = 0; P < n_patches; ++P) {
      int near = all_pairs || near_test(tx + 3 * t, ball + P * 5, eta) ||
                 (self_node && self_node[t] >= 0 && self_node[t] / n == P);
      if (near) {
        if (fill) pair_patch[k++] = (int32_t)P;
        c++;
      }
    }
    if (!fill) pair_ptr[t + 1] = c;
  }
  if (!fill)
    for (int64_t t = 0; t < n_targets; ++t) pair_ptr[t + 1] += pair_ptr[t];
  free(ball);
}

#pragma GCC pop_options

/* Test hook: the q-point U table and GL nodes/weights (rounded to fp64). */
void orc_tables(int q, double *t, double *w, double *U) {
  real *tr = malloc(sizeof(real) * q), *wr = malloc(sizeof(real) * q), *Ur = malloc(sizeof(real) * q * q);
  gl_real(q, tr, wr);
  vandermonde_inverse_real(q, tr, Ur);
  for (int i = 0; i < q; ++i) { t[i] = (double)tr[i]; w[i] = (double)wr[i]; }
  for (int i = 0; i < q * q; ++i) U[i] = (double)Ur[i];
  free(tr); free(wr); free(Ur);
}

/* Near pairs restricted to a list of patches (same rule as orc_near_list, reading A6), brute force
 * over all targets; used to draw bounded samples.  Returns the number of pairs written (<= cap);
 * out_t / out_p receive (target, patch) in patch-list order, targets ascending. */
int64_t orc_near_pairs_for_patches(int p, int q, const double *nodes, const double *weights, const double *verts,
                                   const double *edge_x, int64_t n_targets, const double *tx, const int64_t *self_node,
                                   double eta, int all_pairs, int64_t n_sel, const int32_t *sel, int64_t cap,
                                   int64_t *out_t, int32_t *out_p) {
  int n = p * p;
  int64_t k = 0;
  for (int64_t s = 0; s < n_sel; ++s) {
    int64_t P = sel[s];
    double b[5];
    near_ball(n, q, nodes + P * n * 3, weights + P * n, verts + P * 9, edge_x + P * 3 * q * 3, b);
    for (int64_t t = 0; t < n_targets; ++t) {
      int near = all_pairs || near_test(tx + 3 * t, b, eta) || (self_node && self_node[t] >= 0 && self_node[t] / n == P);
      if (near) {
        if (k < cap) { out_t[k] = t; out_p[k] = (int32_t)P; }
        ++k;
      }
    }
  }
  return k;
}
