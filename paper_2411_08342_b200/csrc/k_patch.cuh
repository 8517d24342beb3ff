// Per-patch kernels: frame + edge geometry (reading A2, A4), near balls (A6), Step-3 edge tables
// (P:L1436-1440), and the least-squares fit operators (Steps 1-2 in matrix mode, reading A1;
// P:L715-746) by a CTA-level Householder QR.
#pragma once
#include "rrq_device.cuh"

namespace rrq {

// Near ball of patch P (reading A6): c_P = sum w x / sum w, R_P = max |x - c_P| over nodes, vertices
// and edge samples, h_P = max vertex chord.  One thread per patch.  balls[P] = (c, R, h).
// The near list is integer output decided in floating point, so the decision is taken in one fixed
// arithmetic on both sides: sums sequential over the nodes, every product, sum, quotient
// and square root a separately rounded IEEE operation (__dmul_rn/__dadd_rn/__ddiv_rn/__dsqrt_rn, no FMA
// contraction) -- the CPU oracle, compiled with -ffp-contract=off, does the same in the same
// order, so both produce the same bits.
__global__ void k_patch_balls(int64_t n_patches, int n, int q, const double *__restrict__ nodes,
                              const double *__restrict__ weights, const double *__restrict__ verts,
                              const double *__restrict__ edge_x, double *__restrict__ balls) {
  const int64_t P = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (P >= n_patches) return;
  const double *x = nodes + P * n * 3, *w = weights + P * n;
  double c0 = 0, c1 = 0, c2 = 0, ws = 0;
  for (int i = 0; i < n; ++i) {
    const double wi = w[i];
    ws = __dadd_rn(ws, wi);
    c0 = __dadd_rn(c0, __dmul_rn(wi, x[3 * i]));
    c1 = __dadd_rn(c1, __dmul_rn(wi, x[3 * i + 1]));
    c2 = __dadd_rn(c2, __dmul_rn(wi, x[3 * i + 2]));
  }
  c0 = __ddiv_rn(c0, ws);
  c1 = __ddiv_rn(c1, ws);
  c2 = __ddiv_rn(c2, ws);
  double R = 0;
  for (int i = 0; i < n + 3 + 3 * q; ++i) {
    const double *y = i < n ? x + 3 * i : (i < n + 3 ? verts + P * 9 + 3 * (i - n) : edge_x + (P * 3 * q + (i - n - 3)) * 3);
    const double r = norm3_rn(__dsub_rn(y[0], c0), __dsub_rn(y[1], c1), __dsub_rn(y[2], c2));
    if (r > R) R = r;
  }
  double h = 0;
  for (int e = 0; e < 3; ++e) {
    const double *a = verts + P * 9 + 3 * e, *b = verts + P * 9 + 3 * ((e + 1) % 3);
    const double l = norm3_rn(__dsub_rn(b[0], a[0]), __dsub_rn(b[1], a[1]), __dsub_rn(b[2], a[2]));
    if (l > h) h = l;
  }
  double *o = balls + P * 5;
  o[0] = c0; o[1] = c1; o[2] = c2; o[3] = R; o[4] = h;
}

// Frame, local edge samples / tangents, Legendre coefficients of the edge interpolants (A4'), height range.
// One CTA (128 threads) per patch.
template <int P>
__global__ void k_patch_geom(int64_t n_patches, const double *__restrict__ nodes, const double *__restrict__ verts,
                             const double *__restrict__ edge_x, const double *__restrict__ edge_dx,
                             const double *__restrict__ balls, Tables T, double *__restrict__ fit) {
  using D = Dims<P>;
  using L = Layout<P>;
  int64_t Pp = blockIdx.x;
  if (Pp >= n_patches) return;
  double *blk = fit + Pp * (int64_t)L::STRIDE;
  __shared__ double fr[13];
  __shared__ double red[2][128];
  const double *v = verts + Pp * 9;
  if (threadIdx.x == 0) {
    double a[3], b[3], z[3], e1[3], e2[3];
    for (int i = 0; i < 3; ++i) {
      fr[i] = (v[i] + v[3 + i] + v[6 + i]) / 3.0;
      a[i] = v[3 + i] - v[i];
      b[i] = v[6 + i] - v[i];
    }
    cross3(a, b, z);
    double nz = sqrt(dot3(z, z)), na = sqrt(dot3(a, a));
    for (int i = 0; i < 3; ++i) { z[i] /= nz; e1[i] = a[i] / na; }
    cross3(z, e1, e2);
    for (int i = 0; i < 3; ++i) { fr[3 + i] = e1[i]; fr[6 + i] = e2[i]; fr[9 + i] = z[i]; }
    fr[12] = balls[Pp * 5 + 4];   // h_P = max vertex chord
  }
  __syncthreads();
  const double *o = fr, *Rm = fr + 3;
  double invh = 1.0 / fr[12];
  auto loc = [&](const double *x, double *y) {
    double d[3] = {x[0] - o[0], x[1] - o[1], x[2] - o[2]};
    for (int r = 0; r < 3; ++r) y[r] = (Rm[3 * r] * d[0] + Rm[3 * r + 1] * d[1] + Rm[3 * r + 2] * d[2]) * invh;
  };
  double zlo = 1e300, zhi = -1e300;
  for (int k = threadIdx.x; k < D::E; k += blockDim.x) {
    double y[3], t[3];
    loc(edge_x + (Pp * D::E + k) * 3, y);
    const double *dx = edge_dx + (Pp * D::E + k) * 3;
    for (int r = 0; r < 3; ++r) t[r] = (Rm[3 * r] * dx[0] + Rm[3 * r + 1] * dx[1] + Rm[3 * r + 2] * dx[2]) * invh;
    for (int r = 0; r < 3; ++r) { blk[L::YL + 3 * k + r] = y[r]; blk[L::TL + 3 * k + r] = t[r]; }
    zlo = fmin(zlo, y[2]); zhi = fmax(zhi, y[2]);
  }
  for (int i = threadIdx.x; i < D::N; i += blockDim.x) {
    double y[3];
    loc(nodes + (Pp * D::N + i) * 3, y);
    zlo = fmin(zlo, y[2]); zhi = fmax(zhi, y[2]);
  }
  if (threadIdx.x < 3) {
    double y[3];
    loc(v + 3 * threadIdx.x, y);
    for (int r = 0; r < 3; ++r) blk[L::HDR + H_VL + 3 * threadIdx.x + r] = y[r];
    zlo = fmin(zlo, y[2]); zhi = fmax(zhi, y[2]);
  }
  red[0][threadIdx.x] = zlo;
  red[1][threadIdx.x] = zhi;
  __syncthreads();
  // Edge interpolants as Legendre series x(t) = sum_j C_j P_j(t) (reading A4'): by Gauss-Legendre
  // exactness C_j = (2j+1)/2 sum_k w_k P_j(t_k) y_k.  Thread (e, j, a).
  for (int t = threadIdx.x; t < 9 * D::Q; t += blockDim.x) {
    int e = t / (3 * D::Q), j = (t / 3) % D::Q, a = t % 3;
    double s = 0;
    for (int k = 0; k < D::Q; ++k) {
      double tk = T.tgl[k], p0 = 1.0, p1 = tk, pj = 1.0;
      if (j == 1) pj = tk;
      for (int i = 1; i < j; ++i) {
        double p2 = ((2 * i + 1) * tk * p1 - i * p0) / (i + 1);
        p0 = p1;
        p1 = p2;
        pj = p2;
      }
      s += T.wgl[k] * pj * blk[L::YL + 3 * (e * D::Q + k) + a];
    }
    blk[L::CM + t] = 0.5 * (2 * j + 1) * s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double lo = 1e300, hi = -1e300;
    for (int i = 0; i < blockDim.x; ++i) { lo = fmin(lo, red[0][i]); hi = fmax(hi, red[1][i]); }
    for (int i = 0; i < 3; ++i) blk[L::HDR + H_O + i] = fr[i];
    for (int i = 0; i < 9; ++i) blk[L::HDR + H_RM + i] = fr[3 + i];
    blk[L::HDR + H_H] = fr[12];
    blk[L::HDR + H_ZLO] = lo;
    blk[L::HDR + H_ZHI] = hi;
    for (int i = 0; i < 3; ++i) blk[L::HDR + H_CP + i] = balls[Pp * 5 + i];
    blk[L::HDR + H_RP] = balls[Pp * 5 + 3];
    blk[L::HDR + H_HP] = balls[Pp * 5 + 4];
  }
}

// Step 3: at each edge node y_kappa the tables g^{(j,k)} = Hess S^{(j,k)}(y) tau
// (2<=j<=p, eq qjkdef2) and e^{(j,k)} = grad S^{(j,k)}(y) x tau (1<=j<=p, eq vjkdef), k >= 0, written as
// the rows (kappa, axis) of the per-patch GEMM operand M of the line-integral maps (Step 6):
//   Q^{(j,k)} = sum_kappa (0, a_kappa)(0, g) = (-a.g, a x g),  V^{(j,k)} = sum_kappa a_kappa . e,
// so that [Q | V](pair) = a(pair) M with a = (omega1_kappa d_kappa) flattened (k = 3 kappa + axis), and
// dQ(pair) = b(pair) M[:, Q cols] with b = omega1 nu' - omega3 (nu'.d) d.
// Columns: Q block 8 jk + 2 comp + re/im (comp 0..3 = scalar, x, y, z), then V block 8 NQ + 2 jk + re/im.
// The columns of (j,k) carry k_translate's operand scaling v_lambda(j,k) (Q) / v_theta(j,k) (V) (TrCfg), so
// k_qmap stores its accumulators as they are.
// One thread per (patch, edge node); it owns rows 3 kappa .. 3 kappa + 2.
template <int P>
struct EdgeTabCfg {
  using D = Dims<P>;
  static constexpr int NB = 8;                                   // edge nodes per round
  static constexpr int THREADS = 128;
  // shared: per node of the round: R [NS] | GS [NS][3] | H [NQ][3] | EV [NV][3] (complex), y, tau
  static constexpr int NODE = (D::NS + 3 * D::NS + 3 * D::NQ + 3 * D::NV) * 2 + 6;
  static constexpr size_t SMEM = (size_t)NB * NODE * sizeof(double);
};

// CTA per patch, rounds of NB edge nodes: thread per node builds R (r_table) and the gradient table in
// shared memory, threads over (node, (j,k)) build g = Hess S tau and e = grad S x tau, then the CTA writes
// the NB x 3 rows of M column-fastest (coalesced whole rows; zero blocks and padding included).
template <int P>
__global__ void __launch_bounds__(EdgeTabCfg<P>::THREADS) k_edge_tables(int64_t n_patches, const double *__restrict__ hc,
                                                                        const double *__restrict__ vlam,
                                                                        const double *__restrict__ vth,
                                                                        double *__restrict__ fit) {
  using D = Dims<P>;
  using L = Layout<P>;
  using C = EdgeTabCfg<P>;
  constexpr int NS = D::NS, NQ = D::NQ, NV = D::NV, E = D::E, NB = C::NB, CQP = D::CQP;
  extern __shared__ __align__(16) double es[];
  const int64_t Pp = blockIdx.x;
  if (Pp >= n_patches) return;
  double *blk = fit + Pp * (int64_t)L::STRIDE;
  double *M = blk + L::MQ, *M1 = blk + L::MQ1;
  for (int n0 = 0; n0 < E; n0 += NB) {
    const int nb = E - n0 < NB ? E - n0 : NB;   // nodes in this round
    __syncthreads();
    // thread per node: R and grad tables (written to shared memory directly)
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
      double *nd = es + i * C::NODE;
      cd *R = reinterpret_cast<cd *>(nd), *GS = R + NS;
      double *yt = nd + C::NODE - 6;
      const int kap = n0 + i;
      for (int a = 0; a < 3; ++a) { yt[a] = blk[L::YL + 3 * kap + a]; yt[3 + a] = blk[L::TL + 3 * kap + a]; }
      r_table<P>(yt[1], yt[2], yt[0], R, hc);
      for (int j = 0; j <= P; ++j)
        for (int k = 0; k <= j; ++k) grad_fast(R, j, k, hc, reinterpret_cast<cd(*)[3]>(GS)[sidx(j, k)]);
    }
    __syncthreads();
    // threads over (node, (j,k)): hessian along tau (j >= 2) and grad x tau, pre-scaled by v_lambda / v_theta
    for (int w = threadIdx.x; w < nb * NV; w += blockDim.x) {
      const int i = w / NV, v = w % NV;
      double *nd = es + i * C::NODE;
      const cd(*GS)[3] = reinterpret_cast<const cd(*)[3]>(reinterpret_cast<cd *>(nd) + NS);
      cd *H = reinterpret_cast<cd *>(nd) + 4 * NS, *EV = H + 3 * NQ;
      const double *t = nd + C::NODE - 3;
      int j = 1;
      while (vidx(j + 1, 0) <= v) ++j;
      const int k = v - vidx(j, 0);
      const cd *g = GS[sidx(j, k)];
      const double sv = vth[v];
      EV[3 * v + 0] = sv * (g[1] * mk(t[2], 0) - g[2] * mk(t[1], 0));
      EV[3 * v + 1] = sv * (g[2] * mk(t[0], 0) - g[0] * mk(t[2], 0));
      EV[3 * v + 2] = sv * (g[0] * mk(t[1], 0) - g[1] * mk(t[0], 0));
      if (j >= 2) {
        cd h[3];
        hess_fast(GS, j, k, t, hc, h);
        const int q = qidx(j, k);
        const double sq = vlam[q];
        for (int a = 0; a < 3; ++a) H[3 * q + a] = sq * h[a];
      }
    }
    __syncthreads();
    // rows k = axis E + kappa of M, column-fastest over the round's NB x 3 rows; columns [0, NCH0) go to
    // half 0 (row stride NCSH0), the rest to half 1 (row stride NCSH1) -- k_qmap's two column passes
    for (int w = threadIdx.x; w < 3 * nb * D::NCP; w += blockDim.x) {
      const int r = w / D::NCP, col = w % D::NCP, axis = r / nb, i = r % nb;
      const cd *H = reinterpret_cast<const cd *>(es + i * C::NODE) + 4 * NS, *EV = H + 3 * NQ;
      double val = 0.0;
      if (col < D::NCQ) {
        // Q columns: component c = col / CQP, entry q, re/im.  Scalar part -a.g; vector parts a x g with
        // the zero block (axis c-1 of component c)
        const int c = col / CQP, wq = col % CQP, q = wq >> 1, ri = wq & 1;
        if (q < NQ) {
          const cd *h = H + 3 * q;
          auto hv = [&](int b) { return ri ? h[b].y : h[b].x; };
          if (c == 0) val = -hv(axis);
          else {
            // component c = 1..3 (x, y, z), cc = c - 1: (a x g)_cc = a_{cc+1} g_{cc+2} - a_{cc+2} g_{cc+1}
            const int cc = c - 1, p1 = (cc + 1) % 3, p2 = (cc + 2) % 3;
            if (axis == p1) val = hv(p2);
            else if (axis == p2) val = -hv(p1);
          }
        }
      } else {
        const int wv = col - D::NCQ, v = wv >> 1, ri = wv & 1;
        if (v < NV) val = ri ? EV[3 * v + axis].y : EV[3 * v + axis].x;
      }
      if (col < D::NCH0) M[(int64_t)(axis * E + n0 + i) * D::NCSH0 + col] = val;
      else M1[(int64_t)(axis * E + n0 + i) * D::NCSH1 + (col - D::NCH0)] = val;
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Fit operators, quaternion form.  The 4n x 4n_p real system of P:L729-735 is the real representation
// of left multiplication by the n x n_p quaternion matrix F_{i,lm} = (0, grad H^{(l,m)}(x_i)) (eq qprule;
// the block pattern [[0,-F1,-F2,-F3],[F1,0,-F3,F2],...] is exactly that representation), and the real
// representation is a *-homomorphism, so A^+ = rep(F^+) with F^+ the quaternion Moore-Penrose inverse.
// F^+ comes from a quaternion Householder QR (H = I - v v^H / beta, v_1 = u (|x_1| + ||x||),
// u = x_1/|x_1|, H x = -u ||x|| e_1) held entirely in shared memory (4x fewer flops than the real QR),
// then P_D[b n_p + lm][i] = (F^+_{lm,i})_b and P_Sp[b n_p + lm][i] = (F^+_{lm,i} (0, nu_i))_b.
// The scalar system B = grad H . nu uses a real Householder QR in shared memory.
// One CTA (256 threads) per patch, persistent over patches.
// ------------------------------------------------------------------------------------------------
struct qd {
  double s, x, y, z;
};
__device__ __forceinline__ qd qmul_(qd a, qd b) {
  return qd{a.s * b.s - a.x * b.x - a.y * b.y - a.z * b.z, a.s * b.x + b.s * a.x + a.y * b.z - a.z * b.y,
            a.s * b.y + b.s * a.y + a.z * b.x - a.x * b.z, a.s * b.z + b.s * a.z + a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ qd qconjmul_(qd a, qd b) {   // conj(a) b
  return qmul_(qd{a.s, -a.x, -a.y, -a.z}, b);
}
__device__ __forceinline__ qd qld(const double *p) { return qd{p[0], p[1], p[2], p[3]}; }
__device__ __forceinline__ void qst(double *p, qd a) { p[0] = a.s; p[1] = a.x; p[2] = a.y; p[3] = a.z; }

template <int P>
struct FitCfg {
  using D = Dims<P>;
  static constexpr int N = D::N, NP = D::NP;
  // shared: Fq [NP][N][4] | rd [NP][4] | beta [NP] | rdb [NP] | betab [NP] | xl,nl [N][3] | sh [64] |
  // vd [NP][4] | cn2 [NP + 1]
  static constexpr size_t FQ = (size_t)NP * N * 4, RD = 4 * NP;
  // p >= 12: the quaternion matrix (359 KB at p = 12) lives in the CTA's global workspace (L2-resident)
  static constexpr bool FQ_GLOBAL = FQ * sizeof(double) > 160 * 1024;
  static constexpr size_t SMEM_D = (FQ_GLOBAL ? 0 : FQ) + RD + 3 * NP + 6 * N + 64 + 4 * NP + NP + 1;
  static constexpr size_t SMEM = SMEM_D * sizeof(double);
  static constexpr int MINB = FQ_GLOBAL ? 1 : (2 * SMEM <= 227 * 1024 ? 2 : 1);   // CTAs per SM
  // per-CTA global workspace (doubles): W [N][N][4] | Xs [N][N] | B [NP][N] | Hm [N][NP] (| Fq)
  static constexpr int64_t WS = (int64_t)N * N * 4 + (int64_t)N * N + 2 * (int64_t)N * NP + (FQ_GLOBAL ? (int64_t)FQ : 0);
};

template <int P>
__global__ void __launch_bounds__(256, FitCfg<P>::MINB) k_patch_fit_q(int64_t n_patches, const double *__restrict__ nodes,
                                                     const double *__restrict__ normals,
                                                     const double *__restrict__ hc, double *__restrict__ fit,
                                                     double *__restrict__ work, int32_t *__restrict__ status) {
  using D = Dims<P>;
  using L = Layout<P>;
  using FC = FitCfg<P>;
  constexpr int N = D::N, NP = D::NP;
  extern __shared__ double fs[];
  double *Fq = FC::FQ_GLOBAL ? work + blockIdx.x * FC::WS + (FC::WS - (int64_t)FC::FQ) : fs;   // Fq[(lm N + i) 4 + comp]
  double *rd = FC::FQ_GLOBAL ? fs : Fq + FC::FQ;   // [NP][4] diagonal of R
  double *beta = rd + FC::RD;           // [NP]
  double *rdb = beta + NP, *betab = rdb + NP;
  double *xl = betab + NP, *nl = xl + 3 * N;
  double *sh = nl + 3 * N;              // [32] reductions
  double *vd = sh + 64, *cn2 = vd + 4 * NP;   // QR pivots v_j, squared column norms
  double *W = work + blockIdx.x * FC::WS;       // [N][N][4]: Q^H e_c
  double *Xs = W + (int64_t)N * N * 4;          // [N][N] real workspace (B system)
  double *Bm = Xs + (int64_t)N * N;             // [NP][N] column-major real B
  double *Hm = Bm + (int64_t)NP * N;            // [N][NP]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  long long ph_t = clock64();
  for (int64_t Pp = blockIdx.x; Pp < n_patches; Pp += gridDim.x) {
    double *blk = fit + Pp * (int64_t)L::STRIDE;
    const double *o = blk + L::HDR + H_O, *Rm = blk + L::HDR + H_RM;
    const double invh = 1.0 / blk[L::HDR + H_H];
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      const double *x = nodes + (Pp * N + i) * 3, *nu = normals + (Pp * N + i) * 3;
      const double d[3] = {x[0] - o[0], x[1] - o[1], x[2] - o[2]};
      for (int r = 0; r < 3; ++r) {
        xl[3 * i + r] = (Rm[3 * r] * d[0] + Rm[3 * r + 1] * d[1] + Rm[3 * r + 2] * d[2]) * invh;
        nl[3 * i + r] = Rm[3 * r] * nu[0] + Rm[3 * r + 1] * nu[1] + Rm[3 * r + 2] * nu[2];
      }
    }
    __syncthreads();
    // F_{i,lm} = (0, grad H), H = sqrt2 Im S; B = grad H . nu; Hm = H(x_i)
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      cd R[D::NS];
      r_table<P>(xl[3 * i + 1], xl[3 * i + 2], xl[3 * i], R, hc);
      for (int l = 1; l <= P; ++l)
        for (int m = 1; m <= l; ++m) {
          cd g[3];
          grad_fast(R, l, m, hc, g);
          const int c = lmidx(l, m);
          const double gx = 1.4142135623730950488 * g[0].y, gy = 1.4142135623730950488 * g[1].y,
                       gz = 1.4142135623730950488 * g[2].y;
          qst(Fq + ((size_t)c * N + i) * 4, qd{0.0, gx, gy, gz});
          Bm[(size_t)c * N + i] = gx * nl[3 * i] + gy * nl[3 * i + 1] + gz * nl[3 * i + 2];
          Hm[(size_t)i * NP + c] = 1.4142135623730950488 * R[sidx(l, m)].y;
        }
    }
    __syncthreads();
    RRQ_PHASE_MARK(8);
    // ---- quaternion Householder QR of Fq (N x NP), one barrier per column: every thread derives column j's
    // reflector (u, |x_1|, ||x||) itself from the squared norm cn2[j] that warp 0 left when it updated column
    // j in step j - 1; the pivot entry v_j = u (|x_1| + ||x||) is kept in registers during the step and
    // written back (vd) after the loop
    if (warp == 0) {
      double s2 = 0;
      for (int i = lane; i < N; i += 32) {
        const qd a = qld(Fq + (size_t)i * 4);
        s2 += a.s * a.s + a.x * a.x + a.y * a.y + a.z * a.z;
      }
      s2 = warp_sum(s2);
      if (lane == 0) cn2[0] = s2;
    }
    __syncthreads();
    for (int j = 0; j < NP; ++j) {
      const double nrm = sqrt(cn2[j]);
      const qd x1 = qld(Fq + ((size_t)j * N + j) * 4);
      const double a = sqrt(x1.s * x1.s + x1.x * x1.x + x1.y * x1.y + x1.z * x1.z);
      const qd u = a > 0 ? qd{x1.s / a, x1.x / a, x1.y / a, x1.z / a} : qd{1, 0, 0, 0};
      const double f = a + nrm;
      const qd vj = {u.s * f, u.x * f, u.y * f, u.z * f};
      const double bj = nrm * (nrm + a);
      if (threadIdx.x == 0) {
        qst(vd + 4 * j, vj);
        qst(rd + 4 * j, qd{-u.s * nrm, -u.x * nrm, -u.y * nrm, -u.z * nrm});
        beta[j] = bj;
      }
      // two columns per warp per pass (c0 and c0 + nw) so their reductions interleave
      for (int c0 = j + 1 + warp; c0 < NP; c0 += 2 * nw) {
        const int c1 = c0 + nw;
        const bool two = c1 < NP;
        double s2 = 0;
        if (bj > 0) {
          qd t0 = {0, 0, 0, 0}, t1 = {0, 0, 0, 0};
          for (int i = j + lane; i < N; i += 32) {
            const qd vi = i == j ? vj : qld(Fq + ((size_t)j * N + i) * 4);
            const qd p0 = qconjmul_(vi, qld(Fq + ((size_t)c0 * N + i) * 4));
            t0.s += p0.s; t0.x += p0.x; t0.y += p0.y; t0.z += p0.z;
            if (two) {
              const qd p1 = qconjmul_(vi, qld(Fq + ((size_t)c1 * N + i) * 4));
              t1.s += p1.s; t1.x += p1.x; t1.y += p1.y; t1.z += p1.z;
            }
          }
          const double ib = 1.0 / bj;
          t0.s = warp_sum(t0.s) * ib; t0.x = warp_sum(t0.x) * ib; t0.y = warp_sum(t0.y) * ib; t0.z = warp_sum(t0.z) * ib;
          if (two) {
            t1.s = warp_sum(t1.s) * ib; t1.x = warp_sum(t1.x) * ib; t1.y = warp_sum(t1.y) * ib; t1.z = warp_sum(t1.z) * ib;
          }
          for (int i = j + lane; i < N; i += 32) {
            const qd vi = i == j ? vj : qld(Fq + ((size_t)j * N + i) * 4);
            double *y = Fq + ((size_t)c0 * N + i) * 4;
            const qd vt = qmul_(vi, t0);
            const qd yn = {y[0] - vt.s, y[1] - vt.x, y[2] - vt.y, y[3] - vt.z};
            qst(y, yn);
            if (c0 == j + 1 && i > j) s2 += yn.s * yn.s + yn.x * yn.x + yn.y * yn.y + yn.z * yn.z;
            if (two) {
              double *y1 = Fq + ((size_t)c1 * N + i) * 4;
              const qd vt1 = qmul_(vi, t1);
              qst(y1, qd{y1[0] - vt1.s, y1[1] - vt1.x, y1[2] - vt1.y, y1[3] - vt1.z});
            }
          }
        } else if (c0 == j + 1) {
          for (int i = j + 1 + lane; i < N; i += 32) {
            const qd yn = qld(Fq + ((size_t)c0 * N + i) * 4);
            s2 += yn.s * yn.s + yn.x * yn.x + yn.y * yn.y + yn.z * yn.z;
          }
        }
        if (c0 == j + 1) {
          s2 = warp_sum(s2);
          if (lane == 0) cn2[j + 1] = s2;
        }
      }
      __syncthreads();
    }
    for (int j = threadIdx.x; j < NP; j += blockDim.x) qst(Fq + ((size_t)j * N + j) * 4, qld(vd + 4 * j));
    __syncthreads();
    RRQ_PHASE_MARK(9);
    // ---- Q^H e_c (warp per two or four columns, the columns in registers: entry i = lane + 32 u), the first
    // NP entries stored for the back substitution
    {
      // 2 under the 128-register bound, 1 at p >= 12 (NU = 5, 7 quaternions per column)
      constexpr int NU = (N + 31) / 32, CW = FC::FQ_GLOBAL ? 1 : (FC::MINB == 2 ? 2 : 4);
      for (int c0 = CW * warp; c0 < N; c0 += CW * nw) {
        qd y[CW][NU];
#pragma unroll
        for (int h = 0; h < CW; ++h)
#pragma unroll
          for (int u = 0; u < NU; ++u) y[h][u] = qd{lane + 32 * u == c0 + h ? 1.0 : 0.0, 0, 0, 0};
        for (int j = 0; j < NP; ++j) {
          const double bj = beta[j];
          if (!(bj > 0)) continue;
          qd v[NU];
          qd t[CW];
#pragma unroll
          for (int h = 0; h < CW; ++h) t[h] = qd{0, 0, 0, 0};
#pragma unroll
          for (int u = 0; u < NU; ++u) {
            const int i = lane + 32 * u;
            v[u] = (i >= j && i < N) ? qld(Fq + ((size_t)j * N + i) * 4) : qd{0, 0, 0, 0};
#pragma unroll
            for (int h = 0; h < CW; ++h) {
              const qd p = qconjmul_(v[u], y[h][u]);
              t[h].s += p.s; t[h].x += p.x; t[h].y += p.y; t[h].z += p.z;
            }
          }
          const double ib = 1.0 / bj;
#pragma unroll
          for (int h = 0; h < CW; ++h) {
            t[h].s = warp_sum(t[h].s) * ib; t[h].x = warp_sum(t[h].x) * ib;
            t[h].y = warp_sum(t[h].y) * ib; t[h].z = warp_sum(t[h].z) * ib;
          }
#pragma unroll
          for (int u = 0; u < NU; ++u)
#pragma unroll
            for (int h = 0; h < CW; ++h) {
              const qd vt = qmul_(v[u], t[h]);
              y[h][u].s -= vt.s; y[h][u].x -= vt.x; y[h][u].y -= vt.y; y[h][u].z -= vt.z;
            }
        }
#pragma unroll
        for (int h = 0; h < CW; ++h) {
          if (c0 + h >= N) continue;
          double *w = W + (size_t)(c0 + h) * N * 4;
#pragma unroll
          for (int u = 0; u < NU; ++u)
            if (lane + 32 * u < NP) qst(w + 4 * (lane + 32 * u), y[h][u]);
        }
      }
    }
    __syncthreads();
    RRQ_PHASE_MARK(10);
    // ---- back substitution R x = (Q^H e_c)[0:NP], column-oriented with four threads per column c: thread g
    // keeps s_k (k = g mod 4) in registers; for r = NP-1 .. 0 the owner of r forms x_r = rd_r^{-1} s_r,
    // broadcasts it to the column's threads, and each subtracts R_kr x_r from its s_k, k < r
    constexpr int NF = L::NF;   // row stride of the fit operators
    double *PD = blk + L::FIT, *PSp = PD + 4 * NP * NF, *PSd = PD + 8 * NP * NF, *PSg = PD + 9 * NP * NF;
    {
      constexpr int G = 4, NR = (NP + G - 1) / G;
      const int g = threadIdx.x & (G - 1), cpb = blockDim.x / G;
      for (int cb = 0; cb < N; cb += cpb) {
        const int c = cb + threadIdx.x / G;
        const bool ok = c < N;
        const double *w = W + (size_t)(ok ? c : 0) * N * 4;
        qd sk[NR];
#pragma unroll
        for (int u = 0; u < NR; ++u) {
          const int k = g + G * u;
          sk[u] = (ok && k < NP) ? qld(w + 4 * k) : qd{0, 0, 0, 0};
        }
        const double n0 = ok ? nl[3 * c] : 0.0, n1 = ok ? nl[3 * c + 1] : 0.0, n2 = ok ? nl[3 * c + 2] : 0.0;
#pragma unroll
        for (int r = NP - 1; r >= 0; --r) {
          const int ow = r % G, ur = r / G;
          qd x = {0, 0, 0, 0};
          if (g == ow) {
            const qd d = qld(rd + 4 * r);
            const double idn = 1.0 / (d.s * d.s + d.x * d.x + d.y * d.y + d.z * d.z);
            const qd q = qconjmul_(d, sk[ur]);
            x = qd{q.s * idn, q.x * idn, q.y * idn, q.z * idn};
            if (ok) {
              // P_D (RHS (mu,0)) and P_Sp (RHS (0, sigma nu))
              PD[(0 * NP + r) * NF + c] = x.s;
              PD[(1 * NP + r) * NF + c] = x.x;
              PD[(2 * NP + r) * NF + c] = x.y;
              PD[(3 * NP + r) * NF + c] = x.z;
              const qd sp = qmul_(x, qd{0.0, n0, n1, n2});
              PSp[(0 * NP + r) * NF + c] = sp.s;
              PSp[(1 * NP + r) * NF + c] = sp.x;
              PSp[(2 * NP + r) * NF + c] = sp.y;
              PSp[(3 * NP + r) * NF + c] = sp.z;
            }
          }
          const int src = (lane & ~(G - 1)) | ow;
          x.s = __shfl_sync(0xffffffffu, x.s, src); x.x = __shfl_sync(0xffffffffu, x.x, src);
          x.y = __shfl_sync(0xffffffffu, x.y, src); x.z = __shfl_sync(0xffffffffu, x.z, src);
#pragma unroll
          for (int u = 0; u < NR; ++u) {
            const int k = g + G * u;
            if (G * u < r && k < r) {
              const qd p = qmul_(qld(Fq + ((size_t)r * N + k) * 4), x);
              sk[u].s -= p.s; sk[u].x -= p.x; sk[u].y -= p.y; sk[u].z -= p.z;
            }
          }
        }
      }
    }
    __syncthreads();
    RRQ_PHASE_MARK(11);
    // ---- the real part runs in shared memory (the Fq space is free now): B, then Xs, Hm (then HP over Xs)
    double *const sBm = Fq, *const sXs = Fq + (size_t)NP * N, *const sHm = sXs + (size_t)N * N;
    for (int i = threadIdx.x; i < NP * N; i += blockDim.x) {
      sBm[i] = Bm[i];
      sHm[i] = Hm[i];
    }
    __syncthreads();
    // ---- real Householder QR of B (N x NP, column-major in sBm) -> P_Sd = B^+; one barrier per column as
    // in the quaternion QR (cn2: squared norms from warp 0, pivots kept in registers, written back after)
    if (warp == 0) {
      double s2 = 0;
      for (int i = lane; i < N; i += 32) s2 += sBm[i] * sBm[i];
      s2 = warp_sum(s2);
      if (lane == 0) cn2[0] = s2;
    }
    __syncthreads();
    for (int j = 0; j < NP; ++j) {
      const double nrm = sqrt(cn2[j]), ajj = sBm[(size_t)j * N + j];
      const double alpha = ajj > 0 ? -nrm : nrm;
      const double vj = ajj - alpha, bj = nrm * (nrm + fabs(ajj));
      if (threadIdx.x == 0) {
        vd[j] = vj;
        rdb[j] = alpha;
        betab[j] = bj;
      }
      for (int c0 = j + 1 + warp; c0 < NP; c0 += 2 * nw) {   // two columns per pass, as above
        const int c1 = c0 + nw;
        const bool two = c1 < NP;
        double s2 = 0;
        if (bj > 0) {
          double t0 = 0, t1 = 0;
          for (int i = j + lane; i < N; i += 32) {
            const double vi = i == j ? vj : sBm[(size_t)j * N + i];
            t0 += vi * sBm[(size_t)c0 * N + i];
            if (two) t1 += vi * sBm[(size_t)c1 * N + i];
          }
          t0 = warp_sum(t0) / bj;
          if (two) t1 = warp_sum(t1) / bj;
          for (int i = j + lane; i < N; i += 32) {
            const double vi = i == j ? vj : sBm[(size_t)j * N + i];
            const double yn = sBm[(size_t)c0 * N + i] - t0 * vi;
            sBm[(size_t)c0 * N + i] = yn;
            if (c0 == j + 1 && i > j) s2 += yn * yn;
            if (two) sBm[(size_t)c1 * N + i] -= t1 * vi;
          }
        } else if (c0 == j + 1) {
          for (int i = j + 1 + lane; i < N; i += 32) s2 += sBm[(size_t)c0 * N + i] * sBm[(size_t)c0 * N + i];
        }
        if (c0 == j + 1) {
          s2 = warp_sum(s2);
          if (lane == 0) cn2[j + 1] = s2;
        }
      }
      __syncthreads();
    }
    for (int j = threadIdx.x; j < NP; j += blockDim.x) sBm[(size_t)j * N + j] = vd[j];
    __syncthreads();
    RRQ_PHASE_MARK(12);
    {   // Q_B^T e_c, four columns per warp in registers (entry i = lane + 32 u)
      constexpr int NU = (N + 31) / 32, CW = 4;
      for (int c0 = CW * warp; c0 < N; c0 += CW * nw) {
        double y[CW][NU];
#pragma unroll
        for (int h = 0; h < CW; ++h)
#pragma unroll
          for (int u = 0; u < NU; ++u) y[h][u] = lane + 32 * u == c0 + h ? 1.0 : 0.0;
        for (int j = 0; j < NP; ++j) {
          const double bj = betab[j];
          if (!(bj > 0)) continue;
          double v[NU], t[CW];
#pragma unroll
          for (int h = 0; h < CW; ++h) t[h] = 0;
#pragma unroll
          for (int u = 0; u < NU; ++u) {
            const int i = lane + 32 * u;
            v[u] = (i >= j && i < N) ? sBm[(size_t)j * N + i] : 0.0;
#pragma unroll
            for (int h = 0; h < CW; ++h) t[h] = fma(v[u], y[h][u], t[h]);
          }
          const double ib = 1.0 / bj;
#pragma unroll
          for (int h = 0; h < CW; ++h) t[h] = warp_sum(t[h]) * ib;
#pragma unroll
          for (int u = 0; u < NU; ++u)
#pragma unroll
            for (int h = 0; h < CW; ++h) y[h][u] = fma(-t[h], v[u], y[h][u]);
        }
#pragma unroll
        for (int h = 0; h < CW; ++h) {
          if (c0 + h >= N) continue;
          double *w = sXs + (size_t)(c0 + h) * N;
#pragma unroll
          for (int u = 0; u < NU; ++u)
            if (lane + 32 * u < N) w[lane + 32 * u] = y[h][u];
        }
      }
    }
    __syncthreads();
    RRQ_PHASE_MARK(13);
    for (int c = threadIdx.x; c < N; c += blockDim.x) {
      double *w = sXs + (size_t)c * N;
      for (int r = NP - 1; r >= 0; --r) {
        double s = w[r];
        for (int k = r + 1; k < NP; ++k) s -= sBm[(size_t)k * N + r] * w[k];
        w[r] = s / rdb[r];
        PSd[r * NF + c] = w[r];
      }
    }
    __syncthreads();
    RRQ_PHASE_MARK(14);
    // ---- P_Sg = P_D (sHm P_Sd); HP over the (now dead) Xs
    double *HP = sXs;
    for (int t = threadIdx.x; t < N * N; t += blockDim.x) {
      const int i = t / N, j = t % N;
      double s = 0;
      for (int c = 0; c < NP; ++c) s += sHm[(size_t)i * NP + c] * PSd[c * NF + j];
      HP[t] = s;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 4 * NP * N; t += blockDim.x) {
      const int r = t / N, j = t % N;
      double s = 0;
      for (int i = 0; i < N; ++i) s += PD[r * NF + i] * HP[(size_t)i * N + j];
      PSg[r * NF + j] = s;
    }
    if (threadIdx.x == 0 && status) {
      double rmax = 0, rmin = 1e300, bmax = 0, bmin = 1e300;
      for (int j = 0; j < NP; ++j) {
        const qd d = qld(rd + 4 * j);
        const double a = sqrt(d.s * d.s + d.x * d.x + d.y * d.y + d.z * d.z);
        rmax = fmax(rmax, a); rmin = fmin(rmin, a);
        bmax = fmax(bmax, fabs(rdb[j])); bmin = fmin(bmin, fabs(rdb[j]));
      }
      status[Pp] = (rmin <= 1e-13 * rmax || bmin <= 1e-13 * bmax) ? 1 : 0;
    }
    __syncthreads();
    RRQ_PHASE_MARK(15);
  }
}

template <int P>
constexpr int64_t fit_workspace_doubles() {
  using D = Dims<P>;
  constexpr int64_t M4 = 4 * D::N, K4 = 4 * D::NP;
  return M4 * K4 + M4 * M4 + K4 * M4 + 3 * D::N * D::NP + D::N * D::NP + 2 * D::N * D::N;
}

}  // namespace rrq
