// Device-side building blocks of the RRQ near-correction builder (sm_100a, fp64).
// Complex arithmetic, regular solid harmonics R_l^m by the Cartesian three-term recurrence, their
// first/second derivatives (reading A3), quaternion products.  Independent of oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rrq {

// |(a, b, c)| with separately rounded IEEE operations in a fixed order (no FMA contraction): the near-list
// arithmetic shared in definition (not in code) with the CPU oracle's near balls.
__device__ __forceinline__ double norm3_rn(double a, double b, double c) {
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)), __dmul_rn(c, c)));
}


constexpr double kPi = 3.14159265358979323846264338327950288;

struct cd {
  double x, y;
};
__device__ __forceinline__ cd mk(double x, double y) { return cd{x, y}; }
__device__ __forceinline__ cd operator+(cd a, cd b) { return cd{a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ cd operator-(cd a, cd b) { return cd{a.x - b.x, a.y - b.y}; }
__device__ __forceinline__ cd operator*(cd a, cd b) { return cd{a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
__device__ __forceinline__ cd operator*(double s, cd a) { return cd{s * a.x, s * a.y}; }
__device__ __forceinline__ cd conj(cd a) { return cd{a.x, -a.y}; }
// 1/sqrt(x) and 1/x for finite x > 0 (resp. x != 0): the SFU's 64-bit seed (MUFU.RSQ64H / RCP64H, ~2^-22)
// and two Newton steps (error ~2^-80 before the final rounding): a few DFMAs instead of the IEEE library
// routines with their slow-path calls.  Results are within 1 ulp of the correctly rounded value.
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  return y * fma(-hx * y, y, 1.5);
}
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * fma(-x, y, 2.0);
  return y * fma(-x, y, 2.0);
}
__device__ __forceinline__ cd cdiv(cd a, cd b) {
  double s = rcp_nr(b.x * b.x + b.y * b.y);
  return cd{(a.x * b.x + a.y * b.y) * s, (a.y * b.x - a.x * b.y) * s};
}
// acc += a * b
__device__ __forceinline__ void cfma(cd &acc, cd a, cd b) {
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
}

template <int P>
struct Dims {
  static constexpr int Q = 2 * P;                 // p~ = 2p edge nodes (reading A4)
  static constexpr int E = 3 * Q;                 // edge nodes per patch
  static constexpr int N = P * P;                 // nodes per patch (reading A1)
  static constexpr int NP = P * (P + 1) / 2;      // basis functions
  static constexpr int NS = (P + 1) * (P + 2) / 2;// (l, m >= 0), l <= p
  static constexpr int NQ = NS - 3;               // (j, k >= 0), 2 <= j <= p
  static constexpr int NV = NS - 1;               // (j, k >= 0), 1 <= j <= p
  static constexpr int NZ = 13 * NP;              // per-pair contraction vector
  static constexpr int K = 3 * E;                 // GEMM depth of the line-integral maps: k = axis E + kappa
  static constexpr int CQP = (2 * NQ + 7) / 8 * 8;// Q columns of one quaternion component (jk, re/im), padded
  static constexpr int NCQ = 4 * CQP;             // Q columns, component-major (scalar, x, y, z)
  static constexpr int NV8 = (2 * NV + 7) / 8 * 8;// V columns (jk, re/im), padded
  static constexpr int NCP = NCQ + NV8;           // whole 8-wide DMMA tiles
  static constexpr int NCS = NCP + ((4 - NCP % 16) + 16) % 16; // row stride == 4 (mod 16): conflict-free B frags
  // k_qmap runs the columns in two passes (register budget): half 0 = Q components scalar, x; half 1 = Q
  // components y, z and the V columns.  M is stored as two blocks [K][NCSH0] | [K][NCSH1] (rows == 4 mod 16)
  static constexpr int NCH0 = 2 * CQP, NCH1 = 2 * CQP + NV8;
  static constexpr int NCSH0 = NCH0 + ((4 - NCH0 % 16) + 16) % 16, NCSH1 = NCH1 + ((4 - NCH1 % 16) + 16) % 16;
};

// (l, m >= 0) -> flat index
__host__ __device__ constexpr int sidx(int l, int m) { return l * (l + 1) / 2 + m; }
__host__ __device__ constexpr int qidx(int j, int k) { return j * (j + 1) / 2 - 3 + k; }
__host__ __device__ constexpr int vidx(int j, int k) { return j * (j + 1) / 2 - 1 + k; }
// (l, m), 1 <= m <= l  -> c-layout index
__host__ __device__ constexpr int lmidx(int l, int m) { return l * (l - 1) / 2 + (m - 1); }

// Per-patch block layout in the fit buffer (doubles).
template <int P>
struct Layout {
  using D = Dims<P>;
  static constexpr int HDR = 0;       // o[3] Rm[9] h zlo zhi vl[9] cP[3] RP hP  (32 slots)
  static constexpr int YL = 32;       // [E][3] local scaled edge samples
  static constexpr int TL = YL + 3 * D::E;   // [E][3] local scaled tangents
  static constexpr int CM = TL + 3 * D::E;   // [3][Q][3] monomial coefficients of the edge interpolants
  static constexpr int NF = D::N + ((4 - D::N % 16) + 16) % 16;   // fit-operator row stride == 4 (mod 16)
  static constexpr int FIT = CM + 9 * D::Q;  // [13 NP][NF]: P_D (4NP) P_Sp (4NP) P_Sd (NP) P_Sg (4NP)
  static constexpr int MQ = (FIT + 13 * D::NP * NF + 3) / 4 * 4;   // GEMM operand of the Q / V maps:
  static constexpr int MQ1 = MQ + D::K * D::NCSH0;                  //   [K][NCSH0] (half 0) | [K][NCSH1] (half 1)
  static constexpr int END = MQ1 + D::K * D::NCSH1;
  static constexpr int STRIDE = (END + 31) / 32 * 32;
};
enum { H_O = 0, H_RM = 3, H_H = 12, H_ZLO = 13, H_ZHI = 14, H_VL = 15, H_CP = 24, H_RP = 27, H_HP = 28 };

// Constant tables uploaded by rrq_create (device global memory).
struct Tables {
  const double *tgl, *wgl;   // [q]
  const double *U;           // [q][q]  c~_c = sum_k U[c][k] F_k
  const double *xo, *wo;     // [n_omega] GL on (-1,1)
  const double *sqb;         // [41][41] sqrt(binomial(n, k))
  const double *xd, *wd;     // [N_DIRECT] Gauss-Legendre rule of the direct model integrals (A11')
  const double *xdp;         // [N_DIRECT][q] powers x_j^k
  const double *hc;          // [HC_SIZE] harmonic coefficients (see below)
};
constexpr int kNDirect = 48;       // reading A11'
constexpr double kRhoDirect = 1.6;

// Harmonic coefficient table (host-built by rrq_create, copied to shared memory by the kernels that use
// it), so no square root is taken on the hot path:
//   HC_DC + 3 (l*l + l + m) + {0,1,2} = sqrt((l-m)(l+m)), sqrt((l-m)(l-m-1)), sqrt((l+m)(l+m-1))  (|m|<=l<=14)
//   HC_DG + m  = sqrt((2m-1)/(2m)),  HC_SB + m = sqrt(2m+1)                                       (m <= 14)
//   HC_RA + sidx(l,m) = (2l+1)/sqrt((l+1+m)(l+1-m)),  HC_RB + sidx(l,m) = sqrt((l+m)(l-m))/sqrt((l+1+m)(l+1-m))
constexpr int HC_LMAX = 14;
// The l-ordered derivative block comes last, so a kernel instantiated for order P stages only the first
// hc_size(P) entries in shared memory.
constexpr int HC_DG = 0, HC_SB = HC_DG + HC_LMAX + 1, HC_RA = HC_SB + HC_LMAX + 1,
              HC_RB = HC_RA + (HC_LMAX + 1) * (HC_LMAX + 2) / 2, HC_DC = HC_RB + (HC_LMAX + 1) * (HC_LMAX + 2) / 2,
              HC_SIZE = HC_DC + 3 * (HC_LMAX + 1) * (HC_LMAX + 1);
__host__ __device__ constexpr int hc_size(int P) { return (HC_DC + 3 * (P + 1) * (P + 1) + 1) / 2 * 2; }

// R_l^m(X,Y,Z), 0 <= m <= l <= P (no Condon-Shortley phase, reading G5) by the Cartesian recurrences
//  R_m^m = sqrt((2m-1)/(2m)) (X + iY) R_{m-1}^{m-1},  R_{m+1}^m = sqrt(2m+1) Z R_m^m,
//  R_{l+1}^m = [(2l+1) Z R_l^m - sqrt((l+m)(l-m)) r^2 R_{l-1}^m] / sqrt((l+1+m)(l+1-m)),
// which follow from P:L338-345 and P:L347-360 multiplied through by r^l (no trig, valid at r = 0).
template <int P>
__device__ __noinline__ void r_column(double X, double Y, double Z, int m, cd *R, const double *hc) {
  double r2 = X * X + Y * Y + Z * Z;
  cd rmm = mk(1.0, 0.0);
  for (int k = 1; k <= m; ++k) rmm = hc[HC_DG + k] * (mk(X, Y) * rmm);
  R[sidx(m, m)] = rmm;
  if (m + 1 <= P) {
    cd a = hc[HC_SB + m] * Z * rmm;
    R[sidx(m + 1, m)] = a;
    cd b = rmm;
    for (int l = m + 1; l < P; ++l) {
      const double ra = hc[HC_RA + sidx(l, m)], rb = hc[HC_RB + sidx(l, m)];
      cd c = (ra * Z) * a - (rb * r2) * b;
      R[sidx(l + 1, m)] = c;
      b = a;
      a = c;
    }
  }
}

template <int P>
__device__ __forceinline__ void r_table(double X, double Y, double Z, cd *R, const double *hc) {
#pragma unroll 1
  for (int m = 0; m <= P; ++m) r_column<P>(X, Y, Z, m, R, hc);
}

// R_l^m for any -l <= m <= l from the m >= 0 table: R_l^{-m} = (-1)^m conj(R_l^m).
__device__ __forceinline__ cd rget(const cd *R, int l, int m) {
  if (l < 0 || m > l || m < -l) return mk(0.0, 0.0);
  if (m >= 0) return R[sidx(l, m)];
  cd v = R[sidx(l, -m)];
  return (((-m) & 1) ? -1.0 : 1.0) * conj(v);
}

// Derivative of R_l^m along R-axis a (0 = X, 1 = Y, 2 = Z) as <= 2 terms (coef, l-1, m') (reading A3).
struct Term {
  cd c;
  int m;
};
__device__ __forceinline__ int dterms(int l, int m, int a, Term *t, const double *hc) {
  const double *dc = hc + HC_DC + 3 * (l * l + l + m);
  if (a == 2) {
    t[0].c = mk(dc[0], 0.0);
    t[0].m = m;
    return 1;
  }
  const double cp = dc[1], cm = dc[2];
  if (a == 0) {  // dX = (D+ + D-)/2, D+ = -cp R^{m+1}, D- = cm R^{m-1}
    t[0].c = mk(-0.5 * cp, 0.0);
    t[1].c = mk(0.5 * cm, 0.0);
  } else {       // dY = (D+ - D-)/(2i) = i (D- - D+)/2
    t[0].c = mk(0.0, 0.5 * cp);
    t[1].c = mk(0.0, 0.5 * cm);
  }
  t[0].m = m + 1;
  t[1].m = m - 1;
  return 2;
}

__device__ __noinline__ cd dR(const cd *R, int l, int m, int a, const double *hc) {
  Term t[2];
  int n = dterms(l, m, a, t, hc);
  cd s = mk(0.0, 0.0);
  for (int i = 0; i < n; ++i) cfma(s, t[i].c, rget(R, l - 1, t[i].m));
  return s;
}

__device__ __noinline__ cd d2R(const cd *R, int l, int m, int a, int b, const double *hc) {
  Term t[2];
  int n = dterms(l, m, a, t, hc);
  cd s = mk(0.0, 0.0);
  for (int i = 0; i < n; ++i)
    if (t[i].m <= l - 1 && t[i].m >= -(l - 1)) cfma(s, t[i].c, dR(R, l - 1, t[i].m, b, hc));
  return s;
}

// S^{(l,m)}(x,y,z) = R_l^m(y,z,x): S-axis x,y,z -> R-axis Z, X, Y.
__device__ __forceinline__ int sax(int a) { return a == 0 ? 2 : a - 1; }

// grad S^{(l,m)} at the point whose R table is R (any m).
__device__ __noinline__ void gradS(const cd *R, int l, int m, cd g[3], const double *hc) {
  for (int a = 0; a < 3; ++a) g[a] = dR(R, l, m, sax(a), hc);
}
// (Hess S^{(l,m)}) v
__device__ __noinline__ void hessS_v(const cd *R, int l, int m, const double v[3], cd out[3], const double *hc) {
  for (int a = 0; a < 3; ++a) {
    cd s = mk(0.0, 0.0);
    for (int b = 0; b < 3; ++b) {
      cd h = d2R(R, l, m, sax(a), sax(b), hc);
      s = s + v[b] * h;
    }
    out[a] = s;
  }
}

// Inline gradient of S^{(l,m)} from the R table (reading A3 rules with S(x,y,z) = R(y,z,x)):
//   dS/dx = dZ R = cz R_{l-1}^m,  dS/dy = dX R = (cm R_{l-1}^{m-1} - cp R_{l-1}^{m+1})/2,
//   dS/dz = dY R = i (cp R_{l-1}^{m+1} + cm R_{l-1}^{m-1})/2.
__device__ __forceinline__ void grad_fast(const cd *R, int l, int m, const double *hc, cd g[3]) {
  const double *dc = hc + HC_DC + 3 * (l * l + l + m);
  const cd r0 = rget(R, l - 1, m), rp = rget(R, l - 1, m + 1), rm = rget(R, l - 1, m - 1);
  g[0] = dc[0] * r0;
  g[1] = 0.5 * (dc[2] * rm - dc[1] * rp);
  const cd t = 0.5 * (dc[1] * rp + dc[2] * rm);
  g[2] = mk(-t.y, t.x);
}
// GS table entry for any m from the m >= 0 table: grad S^{(l,-m)} = (-1)^m conj(grad S^{(l,m)}).
__device__ __forceinline__ void gget(const cd (*GS)[3], int l, int m, cd g[3]) {
  if (l < 0 || m > l || m < -l) { g[0] = g[1] = g[2] = mk(0, 0); return; }
  if (m >= 0) { g[0] = GS[sidx(l, m)][0]; g[1] = GS[sidx(l, m)][1]; g[2] = GS[sidx(l, m)][2]; return; }
  const double sg = ((-m) & 1) ? -1.0 : 1.0;
  for (int a = 0; a < 3; ++a) g[a] = sg * conj(GS[sidx(l, -m)][a]);
}
// (Hess S^{(l,m)}) v = grad (v . grad S^{(l,m)}) with v . grad S^{(l,m)} = v_x cz S^{(l-1,m)} +
// cp b+ S^{(l-1,m+1)} + cm b- S^{(l-1,m-1)},  b+- = (-+ v_y + i v_z)/2   (same rules, applied twice).
__device__ __forceinline__ void hess_fast(const cd (*GS)[3], int l, int m, const double v[3], const double *hc,
                                          cd out[3]) {
  const double *dc = hc + HC_DC + 3 * (l * l + l + m);
  const cd bp = (0.5 * dc[1]) * mk(-v[1], v[2]), bm = (0.5 * dc[2]) * mk(v[1], v[2]);
  const double b0 = v[0] * dc[0];
  cd g0[3], gp[3], gm[3];
  gget(GS, l - 1, m, g0);
  gget(GS, l - 1, m + 1, gp);
  gget(GS, l - 1, m - 1, gm);
  for (int a = 0; a < 3; ++a) out[a] = b0 * g0[a] + bp * gp[a] + bm * gm[a];
}

// Complex quaternion.
struct cq {
  cd s, v[3];
};
__device__ __forceinline__ cq qzero() {
  cq r;
  r.s = mk(0, 0);
  r.v[0] = r.v[1] = r.v[2] = mk(0, 0);
  return r;
}

// One 32-byte global store (STG.256, sm_100): p must be 32-byte aligned.
__device__ __forceinline__ void st_global_256(double *p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

__device__ __forceinline__ double dot3(const double *a, const double *b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
__device__ __forceinline__ void cross3(const double *a, const double *b, double *c) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}

// Inverse of the triangular index t(l) = l (l + 1) / 2: the l with t(l) <= e < t(l + 1) (e < 2^20; the float
// square root is exact on the perfect squares 8 t(l) + 1 = (2l + 1)^2 that decide the floor).
__device__ __forceinline__ int tri_inv(int e) { return (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// Warp sums of 8 values at once by a reduce-scatter butterfly (9 shuffles instead of 8 x 5): on return
// lane L holds the sum of value 4 b4 + 2 b3 + b2 (b = bits of L), i.e. value (L >> 2) & 7 ... for L in 0..31
// the value index is ((L >> 4) & 1) * 4 + ((L >> 3) & 1) * 2 + ((L >> 2) & 1).
__device__ __forceinline__ double warp_sum8(const double (&v)[8], int lane) {
  const bool b4 = (lane >> 4) & 1, b3 = (lane >> 3) & 1, b2 = (lane >> 2) & 1;
  double w[4], x[2];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double keep = b4 ? v[4 + j] : v[j], send = b4 ? v[j] : v[4 + j];
    w[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const double keep = b3 ? w[2 + j] : w[j], send = b3 ? w[j] : w[2 + j];
    x[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  double y = (b2 ? x[1] : x[0]) + __shfl_xor_sync(0xffffffffu, b2 ? x[0] : x[1], 4);
  y += __shfl_xor_sync(0xffffffffu, y, 2);
  y += __shfl_xor_sync(0xffffffffu, y, 1);
  return y;
}

}  // namespace rrq
