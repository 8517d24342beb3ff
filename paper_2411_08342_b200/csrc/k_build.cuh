// The per-pair hot path: Steps 4-7 -> contraction vector Z, then Step 8 in matrix
// mode + smooth-rule subtraction (reading A14) -> CSR weights.
//
// k_pair_zeta: one warp per (target, patch) pair, pairs visited patch-major so a CTA's warps share
//   one patch's edge tables in L1/L2.  Lanes split: the R_l^m columns (m), the harmonic derivative
//   table, the 9 (edge, component) polynomial evaluations of the complex Newton solve, the 3p~ edge
//   nodes (weights, Omega, dOmega), the 2 n_Omega sinh-rule nodes, the 2 NQ + NV line-integral maps
//   Q, dQ, V, and the NP translations.
// k_contract: per patch, a CTA contracts TILE pairs' Z rows with the patch's fit operators
//   (register-blocked over pairs), subtracts the smooth rule and stores n contiguous fp64 per pair.
#pragma once
#include "rrq_device.cuh"

namespace rrq {

__device__ __forceinline__ cd csqrt_(cd z) {
  double r = hypot(z.x, z.y);
  if (r == 0) return mk(0, 0);
  double a = sqrt(0.5 * (r + fabs(z.x)));
  double b = 0.5 * z.y / a;
  if (z.x >= 0) return mk(a, b);
  return mk(fabs(b), z.y >= 0 ? a : -a);
}

// Bernstein ellipse parameter (reading A5)
__device__ __forceinline__ double bernstein_rho(double re, double im) {
  cd t = mk(re, im);
  cd s = csqrt_(t * t - mk(1.0, 0.0));
  double r1 = cabs_(t + s), r2 = cabs_(t - s);
  return fmax(r1, r2);
}

// Model integrals I_k, J_k (reading A11): upward recurrences, cancellation-free I_0, J_0.
template <int Q>
__device__ void model_integrals(double a, double b, double *I, double *J) {
  double Q1 = (1 - a) * (1 - a) + b * b, Qm = (1 + a) * (1 + a) + b * b;
  double s1 = sqrt(Q1), sm = sqrt(Qm);
  if (fabs(a) <= 1.0) {
    I[0] = asinh((1 - a) / b) + asinh((1 + a) / b);
    J[0] = ((1 - a) / s1 + (1 + a) / sm) / (b * b);
  } else {
    double aa = fabs(a), u = aa + 1, v = aa - 1;
    double su = sqrt(u * u + b * b), sv = sqrt(v * v + b * b);
    I[0] = log((u + su) / (v + sv));
    J[0] = 4 * aa / (su * sv * (u * sv + v * su));
  }
  double a2b2 = a * a + b * b, is1 = 1.0 / s1, ism = 1.0 / sm;
  for (int k = 1; k < Q; ++k) {
    double sg = ((k - 1) & 1) ? -1.0 : 1.0;
    double beta = s1 - sg * sm, gam = is1 - sg * ism;
    if (k == 1) {
      I[1] = beta + a * I[0];
      J[1] = a * J[0] - gam;
    } else {
      I[k] = (beta + (2 * k - 1) * a * I[k - 1] - (k - 1) * a2b2 * I[k - 2]) / k;
      J[k] = a * J[k - 1] - gam + (k - 1) * I[k - 2];
    }
  }
}

template <int P>
struct WarpScratch {
  using D = Dims<P>;
  cd R[D::NS];        // R_l^m at (y', z', x'): S^{(l,m)}(r') for m >= 0
  cd GS[D::NS][3];    // grad S^{(l,m)}(r')
  cd NG[D::NS];       // nu' . grad S^{(l,m)}(r')
  cd HN[D::NS][3];    // Hess S^{(l,m)}(r') nu'
  double a[D::E][3];  // omega1_k d_k
  double b[D::E][3];  // omega1_k nu' - omega3_k (nu'.d_k) d_k
  double I[3][D::Q], J[3][D::Q];
  double Qv[D::NQ][8], dQ[D::NQ][8], V[D::NV][2];
  double t0[3][2];
  double Om[4], dOm[4];   // (Omega_0, Omega), (dOmega_0, dOmega)
  double r13[2][kNDirect];
  int swap[3], conv[3], direct[3];
};

struct SmemTables {
  int q, n_omega;
};

// Legendre-series edge interpolant (reading A4'): value and derivatives of component c at t, by
// Bonnet's recurrence and P'_{j+1} = P'_{j-1} + (2j+1) P_j, P''_{j+1} = P''_{j-1} + (2j+1) P'_j.
template <int Q>
__device__ __forceinline__ void leg_r(const double *C, int c, double t, double &v, double &d1, double &d2) {
  double P0 = 1, P1 = t, a0 = 0, a1 = 1, b0 = 0, b1 = 0;
  v = C[c] + C[3 + c] * t;
  d1 = C[3 + c];
  d2 = 0;
#pragma unroll
  for (int j = 1; j + 1 < Q; ++j) {
    double P2 = ((2 * j + 1) * t * P1 - j * P0) * (1.0 / (j + 1));
    double a2 = a0 + (2 * j + 1) * P1, b2 = b0 + (2 * j + 1) * a1;
    double cc = C[3 * (j + 1) + c];
    v = fma(cc, P2, v);
    d1 = fma(cc, a2, d1);
    d2 = fma(cc, b2, d2);
    P0 = P1; P1 = P2; a0 = a1; a1 = a2; b0 = b1; b1 = b2;
  }
}
template <int Q>
__device__ __forceinline__ void leg_c(const double *C, int c, cd t, cd &v, cd &d1) {
  cd P0 = mk(1, 0), P1 = t, a0 = mk(0, 0), a1 = mk(1, 0);
  v = mk(C[c], 0) + C[3 + c] * t;
  d1 = mk(C[3 + c], 0);
#pragma unroll
  for (int j = 1; j + 1 < Q; ++j) {
    cd P2 = (1.0 / (j + 1)) * ((2.0 * j + 1) * (t * P1) - (double)j * P0);
    cd a2 = a0 + (2.0 * j + 1) * P1;
    double cc = C[3 * (j + 1) + c];
    v = v + cc * P2;
    d1 = d1 + cc * a2;
    P0 = P1; P1 = P2; a0 = a1; a1 = a2;
  }
}
// x(t), x'(t) (3 components, real t)
template <int Q>
__device__ __forceinline__ void leg_r3(const double *C, double t, double x[3], double dx[3]) {
  double P0 = 1, P1 = t, a0 = 0, a1 = 1;
  for (int c = 0; c < 3; ++c) { x[c] = C[c] + C[3 + c] * t; dx[c] = C[3 + c]; }
#pragma unroll
  for (int j = 1; j + 1 < Q; ++j) {
    double P2 = ((2 * j + 1) * t * P1 - j * P0) * (1.0 / (j + 1));
    double a2 = a0 + (2 * j + 1) * P1;
    for (int c = 0; c < 3; ++c) {
      double cc = C[3 * (j + 1) + c];
      x[c] = fma(cc, P2, x[c]);
      dx[c] = fma(cc, a2, dx[c]);
    }
    P0 = P1; P1 = P2; a0 = a1; a1 = a2;
  }
}

// sum of a value over the 3 lanes {3e, 3e+1, 3e+2}
__device__ __forceinline__ double tri_sum(double v, int base) {
  double a = __shfl_sync(0xffffffffu, v, base), b = __shfl_sync(0xffffffffu, v, base + 1),
         c = __shfl_sync(0xffffffffu, v, base + 2);
  return a + b + c;
}

template <int P, int WPB>
__global__ void __launch_bounds__(WPB * 32)
    k_pair_zeta(int64_t npairs, const int64_t *__restrict__ perm, const int64_t *__restrict__ ptgt, int64_t kbase,
                const int32_t *__restrict__ pair_patch, const double *__restrict__ fit, const double *__restrict__ tx,
                const double *__restrict__ tnorm, const int64_t *__restrict__ self_node,
                const int8_t *__restrict__ side, Tables T, int n_omega, double rho0, double *__restrict__ Z,
                int32_t *__restrict__ pstat, unsigned long long *__restrict__ swapcnt) {
  using D = Dims<P>;
  using L = Layout<P>;
  constexpr int Q = D::Q, E = D::E, NP = D::NP, NQ = D::NQ, NV = D::NV, NS = D::NS, NZ = D::NZ;
  extern __shared__ double smem[];
  double *sU = smem;                  // [Q][Q]
  double *stgl = sU + Q * Q, *swgl = stgl + Q;
  double *sxo = swgl + Q, *swo = sxo + n_omega;
  double *ssqb = swo + n_omega;       // [(2P+1)][(2P+1)] sqrt binomials
  double *sfac = ssqb + (2 * P + 1) * (2 * P + 1);  // [2P+2] factorials
  constexpr int SQ = 2 * P + 1;
  int tab_doubles = Q * Q + 2 * Q + 2 * n_omega + SQ * SQ + (2 * P + 2);
  tab_doubles = (tab_doubles + 1) & ~1;
  WarpScratch<P> *wsall = reinterpret_cast<WarpScratch<P> *>(smem + tab_doubles);
  for (int i = threadIdx.x; i < Q * Q; i += blockDim.x) sU[i] = T.U[i];
  for (int i = threadIdx.x; i < Q; i += blockDim.x) { stgl[i] = T.tgl[i]; swgl[i] = T.wgl[i]; }
  for (int i = threadIdx.x; i < n_omega; i += blockDim.x) { sxo[i] = T.xo[i]; swo[i] = T.wo[i]; }
  for (int i = threadIdx.x; i < SQ * SQ; i += blockDim.x) ssqb[i] = T.sqb[(i / SQ) * 41 + (i % SQ)];
  if (threadIdx.x == 0) {
    double f = 1;
    sfac[0] = 1;
    for (int i = 1; i < 2 * P + 2; ++i) { f *= i; sfac[i] = f; }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpScratch<P> &ws = wsall[warp];
  const double inv4pi = 1.0 / (4.0 * kPi), s2 = 1.4142135623730950488;
  unsigned long long nswap = 0;

  for (int64_t s = (int64_t)blockIdx.x * WPB + warp; s < npairs; s += (int64_t)gridDim.x * WPB) {
    const int64_t k = perm[s];
    const int64_t t = ptgt[k - kbase];
    const int Pp = pair_patch[k];
    const double *blk = fit + (int64_t)Pp * L::STRIDE;
    // ---------------- target in the patch frame (reading A2)
    const double *hd = blk + L::HDR;
    double rp[3], nup[3] = {0, 0, 0};
    {
      double invh = 1.0 / hd[H_H];
      double d[3] = {tx[3 * t] - hd[H_O], tx[3 * t + 1] - hd[H_O + 1], tx[3 * t + 2] - hd[H_O + 2]};
      for (int r = 0; r < 3; ++r) rp[r] = (hd[H_RM + 3 * r] * d[0] + hd[H_RM + 3 * r + 1] * d[1] + hd[H_RM + 3 * r + 2] * d[2]) * invh;
      if (tnorm) {
        const double *nn = tnorm + 3 * t;
        for (int r = 0; r < 3; ++r) nup[r] = hd[H_RM + 3 * r] * nn[0] + hd[H_RM + 3 * r + 1] * nn[1] + hd[H_RM + 3 * r + 2] * nn[2];
      }
    }
    int self_local = -1;
    if (self_node) {
      int64_t sn = self_node[t];
      if (sn >= 0 && sn / D::N == Pp) self_local = (int)(sn % D::N);
    }
    const int sd = side ? (int)side[t] : 2;
    // gauge sign (reading A8)
    double sg;
    {
      double z = rp[2] - hd[H_VL + 2], zlo = hd[H_ZLO], zhi = hd[H_ZHI];
      if (self_local >= 0) sg = -1.0;
      else if (z > zhi + 0.1) sg = 1.0;
      else if (z < zlo - 0.1) sg = -1.0;
      else {
        const double *va = hd + H_VL, *vb = hd + H_VL + 3, *vc = hd + H_VL + 6;
        double det = (vb[0] - va[0]) * (vc[1] - va[1]) - (vc[0] - va[0]) * (vb[1] - va[1]);
        double l1 = ((rp[0] - va[0]) * (vc[1] - va[1]) - (vc[0] - va[0]) * (rp[1] - va[1])) / det;
        double l2 = ((vb[0] - va[0]) * (rp[1] - va[1]) - (rp[0] - va[0]) * (vb[1] - va[1])) / det;
        double l0 = 1 - l1 - l2;
        double mn = fmin(l0, fmin(l1, l2));
        if (mn >= -0.25 && sd != 2) sg = sd > 0 ? 1.0 : -1.0;
        else sg = (z - 0.5 * (zlo + zhi) > 0) ? 1.0 : -1.0;
      }
    }
    const double u[3] = {0.0, 0.0, sg};

    // ---------------- Step 4: harmonics at the target
    if (lane <= P) r_column<P>(rp[1], rp[2], rp[0], lane, ws.R);
    __syncwarp();
    for (int e = lane; e < NS; e += 32) {
      int l = 0;
      while (sidx(l + 1, 0) <= e) ++l;
      int m = e - sidx(l, 0);
      cd g[3];
      gradS(ws.R, l, m, g);
      cd ng = mk(0, 0);
      for (int a = 0; a < 3; ++a) { ws.GS[e][a] = g[a]; ng = ng + nup[a] * g[a]; }
      ws.NG[e] = ng;
      cd hn[3];
      hessS_v(ws.R, l, m, nup, hn);
      for (int a = 0; a < 3; ++a) ws.HN[e][a] = hn[a];
    }

    // ---------------- Step 5: t0 per edge (reading A12), lanes (e, c) = (lane/3, lane%3)
    {
      const int e = lane < 9 ? lane / 3 : 2, c = lane < 9 ? lane % 3 : 2, base = 3 * e;
      const double *C = blk + L::CM + e * Q * 3;
      const double rc = rp[c];
      auto horner_r = [&](double tt, double &v, double &d1, double &d2) { leg_r<Q>(C, c, tt, v, d1, d2); };
      double v, d1, d2;
      horner_r(-1.0, v, d1, d2);
      double A = v;
      horner_r(1.0, v, d1, d2);
      double ab = v - A, ar = rc - A;
      double tc = -1.0 + 2.0 * tri_sum(ar * ab, base) / tri_sum(ab * ab, base);
      bool go = true;
      for (int it = 0; it < 3; ++it) {
        horner_r(tc, v, d1, d2);
        double xr = v - rc;
        double g = tri_sum(xr * d1, base), gp = tri_sum(d1 * d1 + xr * d2, base);
        go = go && (gp > 0);
        if (go) tc -= g / gp;
      }
      horner_r(tc, v, d1, d2);
      double xr = v - rc;
      double f = tri_sum(xr * xr, base), dd = tri_sum(d1 * d1 + xr * d2, base), xp2 = tri_sum(d1 * d1, base);
      if (!(dd > 0)) dd = xp2;
      cd tz = mk(tc, sqrt(f / dd));
      bool conv = false;
      for (int it = 0; it < 20; ++it) {
        cd xv, xd;
        leg_c<Q>(C, c, tz, xv, xd);
        cd xrr = xv - mk(rc, 0);
        cd sq = xrr * xrr, pr = xrr * xd;
        cd F = mk(tri_sum(sq.x, base), tri_sum(sq.y, base));
        cd Fp = 2.0 * mk(tri_sum(pr.x, base), tri_sum(pr.y, base));
        if (!conv) {
          cd dt = cdiv(F, Fp);
          tz = tz - dt;
          if (cabs_(dt) < 1e-15 * (1.0 + cabs_(tz))) conv = true;
        }
        if (__all_sync(0xffffffffu, conv || lane >= 9)) break;
      }
      if (tz.y < 0) tz.y = -tz.y;
      conv = conv && isfinite(tz.x) && isfinite(tz.y);
      if (lane < 9 && c == 0) {
        ws.t0[e][0] = tz.x;
        ws.t0[e][1] = tz.y;
        ws.conv[e] = conv;
        double rho = bernstein_rho(tz.x, tz.y);
        ws.swap[e] = conv && rho < rho0;
        ws.direct[e] = rho >= kRhoDirect;
      }
    }
    __syncwarp();
    // model integrals (reading A11 / A11'): recurrences inside rho = 1.6, a 48-point rule outside
    if (lane < 3 && ws.swap[lane] && !ws.direct[lane])
      model_integrals<Q>(ws.t0[lane][0], fabs(ws.t0[lane][1]), ws.I[lane], ws.J[lane]);
    for (int e = 0; e < 3; ++e) {
      if (!(ws.swap[e] && ws.direct[e])) continue;
      const double a = ws.t0[e][0], b = fabs(ws.t0[e][1]);
      for (int j = lane; j < kNDirect; j += 32) {
        double xj = T.xd[j], Qv = (xj - a) * (xj - a) + b * b;
        double r1 = T.wd[j] / sqrt(Qv);
        ws.r13[0][j] = r1;
        ws.r13[1][j] = r1 / Qv;
      }
      __syncwarp();
      if (lane < Q) {
        double si = 0, sj = 0;
        for (int j = 0; j < kNDirect; ++j) {
          double pw = __ldg(T.xdp + j * Q + lane);
          si = fma(pw, ws.r13[0][j], si);
          sj = fma(pw, ws.r13[1][j], sj);
        }
        ws.I[e][lane] = si;
        ws.J[e][lane] = sj;
      }
      __syncwarp();
    }
    __syncwarp();

    // ---------------- weights and the scalar line integrals (Step 6)
    double om[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // Omega_0(plain) Omega[3] dOmega_0 dOmega[3]
    for (int kap = lane; kap < E; kap += 32) {
      const int e = kap / Q, kk = kap % Q;
      const double *y = blk + L::YL + 3 * kap, *tau = blk + L::TL + 3 * kap;
      double d[3] = {rp[0] - y[0], rp[1] - y[1], rp[2] - y[2]};
      double dn = sqrt(dot3(d, d));
      double w1, w3;
      if (ws.swap[e]) {
        double mu1 = 0, mu3 = 0;
        for (int c = 0; c < Q; ++c) {
          mu1 = fma(ws.I[e][c], sU[c * Q + kk], mu1);
          mu3 = fma(ws.J[e][c], sU[c * Q + kk], mu3);
        }
        double ta = stgl[kk] - ws.t0[e][0], tb = ws.t0[e][1];
        double r1 = sqrt(ta * ta + tb * tb) / dn;
        w1 = mu1 * r1;
        w3 = mu3 * r1 * r1 * r1;
      } else {
        w1 = swgl[kk] / dn;
        w3 = swgl[kk] / (dn * dn * dn);
        double dxu[3];
        cross3(d, u, dxu);
        om[0] += swgl[kk] * (-dot3(dxu, tau) / (dn * (dn + dot3(u, d))));
      }
      double nd = dot3(nup, d);
      double txd[3];
      cross3(tau, d, txd);
      for (int a = 0; a < 3; ++a) {
        ws.a[kap][a] = w1 * d[a];
        ws.b[kap][a] = w1 * nup[a] - w3 * nd * d[a];
        om[1 + a] -= w1 * tau[a];
        om[5 + a] += w3 * nd * tau[a];
      }
      om[4] += w3 * dot3(nup, txd);
    }
    for (int i = 0; i < 8; ++i) om[i] = warp_sum(om[i]);
    // Omega_0 on swap edges: sinh-split Gauss-Legendre on the interpolated edge (reading A9)
    for (int e = 0; e < 3; ++e) {
      if (!ws.swap[e]) continue;
      double a = fmin(1.0, fmax(-1.0, ws.t0[e][0])), b = fabs(ws.t0[e][1]);
      double sR = asinh((1 - a) / b), sL = asinh((-1 - a) / b);
      const double *C = blk + L::CM + e * Q * 3;
      double acc = 0;
      for (int j = lane; j < 2 * n_omega; j += 32) {
        int sdd = j / n_omega, jj = j % n_omega;
        double lo = sdd ? 0.0 : sL, hi = sdd ? sR : 0.0;
        if (!(hi > lo)) continue;
        double sv = lo + (hi - lo) * (sxo[jj] + 1) * 0.5, W = (hi - lo) * 0.5 * swo[jj];
        double tt = a + b * sinh(sv), dt = b * cosh(sv);
        double x[3], dx[3];
        leg_r3<Q>(C, tt, x, dx);
        double d[3] = {rp[0] - x[0], rp[1] - x[1], rp[2] - x[2]};
        double nd = sqrt(dot3(d, d)), dxu[3];
        cross3(d, u, dxu);
        acc += W * dt * (-dot3(dxu, dx) / (nd * (nd + dot3(u, d))));
      }
      om[0] += warp_sum(acc);
    }
    if (self_local >= 0) om[0] -= 2.0 * kPi;   // principal value (reading A7)
    __syncwarp();

    // ---------------- line-integral maps Q, dQ, V (Step 6)
    const double *GT = blk + L::GT, *ET = blk + L::ET;
    for (int task = lane; task < 2 * NQ + NV; task += 32) {
      if (task < 2 * NQ) {
        const int jk = task < NQ ? task : task - NQ;
        const double(*av)[3] = task < NQ ? ws.a : ws.b;
        double s0r = 0, s0i = 0, vr[3] = {0, 0, 0}, vi[3] = {0, 0, 0};
        for (int kap = 0; kap < E; ++kap) {
          const double *g = GT + (int64_t)kap * 6 * NQ + jk;
          double gr[3] = {__ldg(g), __ldg(g + 2 * NQ), __ldg(g + 4 * NQ)};
          double gi[3] = {__ldg(g + NQ), __ldg(g + 3 * NQ), __ldg(g + 5 * NQ)};
          double a0 = av[kap][0], a1 = av[kap][1], a2 = av[kap][2];
          s0r -= a0 * gr[0] + a1 * gr[1] + a2 * gr[2];
          s0i -= a0 * gi[0] + a1 * gi[1] + a2 * gi[2];
          vr[0] += a1 * gr[2] - a2 * gr[1];
          vr[1] += a2 * gr[0] - a0 * gr[2];
          vr[2] += a0 * gr[1] - a1 * gr[0];
          vi[0] += a1 * gi[2] - a2 * gi[1];
          vi[1] += a2 * gi[0] - a0 * gi[2];
          vi[2] += a0 * gi[1] - a1 * gi[0];
        }
        double *o = task < NQ ? ws.Qv[jk] : ws.dQ[jk];
        o[0] = s0r; o[1] = s0i;
        for (int a = 0; a < 3; ++a) { o[2 + 2 * a] = vr[a]; o[3 + 2 * a] = vi[a]; }
      } else {
        const int jk = task - 2 * NQ;
        double sr = 0, si = 0;
        for (int kap = 0; kap < E; ++kap) {
          const double *g = ET + (int64_t)kap * 6 * NV + jk;
          for (int a = 0; a < 3; ++a) {
            sr += ws.a[kap][a] * __ldg(g + 2 * a * NV);
            si += ws.a[kap][a] * __ldg(g + (2 * a + 1) * NV);
          }
        }
        ws.V[jk][0] = sr;
        ws.V[jk][1] = si;
      }
    }
    __syncwarp();

    // ---------------- Step 7: translation
    double *Zr = Z + s * NZ;
    for (int c = lane; c < NP; c += 32) {
      int l = 1;
      while (lmidx(l + 1, 1) <= c) ++l;
      int m = c - lmidx(l, 1) + 1;
      cq lam = qzero(), dlam = qzero();
      cd th = mk(0, 0);
      for (int j = 1; j <= l; ++j) {
        const int lj = l - j;
        const int kmin = max(-j, m - lj), kmax = min(j, m + lj);
        for (int kk = kmin; kk <= kmax; ++kk) {
          const double Tc = ssqb[(l + m) * SQ + (j + kk)] * ssqb[(l - m) * SQ + (j - kk)];
          const int mk_ = m - kk;
          cd Sv = rget(ws.R, lj, mk_);
          cd NGv;
          if (mk_ >= 0) NGv = ws.NG[sidx(lj, mk_)];
          else NGv = (((-mk_) & 1) ? -1.0 : 1.0) * conj(ws.NG[sidx(lj, -mk_)]);
          const int ak = kk < 0 ? -kk : kk;
          const double sgn = (kk < 0 && (ak & 1)) ? -1.0 : 1.0;
          const bool cj = kk < 0;
          {  // theta_1 (j >= 1): D_{j,l} T V^{(j,k)} S^{(l-j,m-k)}
            const double *vv = ws.V[vidx(j, ak)];
            cd Vv = mk(sgn * vv[0], sgn * (cj ? -vv[1] : vv[1]));
            double Dj = sfac[j - 1] * sfac[lj] / sfac[l];
            cfma(th, (Dj * Tc) * Vv, Sv);
          }
          if (j >= 2) {
            const double cT = sfac[j - 2] * sfac[lj] / sfac[l - 1] * Tc;
            const double *qv = ws.Qv[qidx(j, ak)], *dq = ws.dQ[qidx(j, ak)];
            cd cS = cT * Sv, cN = cT * NGv;
            for (int b = 0; b < 4; ++b) {
              cd qb = mk(sgn * qv[2 * b], sgn * (cj ? -qv[2 * b + 1] : qv[2 * b + 1]));
              cd dqb = mk(sgn * dq[2 * b], sgn * (cj ? -dq[2 * b + 1] : dq[2 * b + 1]));
              cd &L1 = b == 0 ? lam.s : lam.v[b - 1];
              cd &L2 = b == 0 ? dlam.s : dlam.v[b - 1];
              cfma(L1, qb, cS);
              cfma(L2, dqb, cS);
              cfma(L2, qb, cN);
            }
          }
        }
      }
      // I[gamma]: (Omega_0, Omega)(0, grad S^{(l,m)}(r')), omega first
      const int hs = sidx(l, m);
      const cd *g = ws.GS[hs], *hn = ws.HN[hs];
      const double O0 = om[0], Ov[3] = {om[1], om[2], om[3]}, dO0 = om[4], dOv[3] = {om[5], om[6], om[7]};
      cd gs = mk(0, 0), dgs = mk(0, 0), gv[3], dgv[3];
      for (int a = 0; a < 3; ++a) {
        gs = gs - Ov[a] * g[a];
        dgs = dgs - dOv[a] * g[a] - Ov[a] * hn[a];
        int b1 = (a + 1) % 3, b2 = (a + 2) % 3;
        gv[a] = O0 * g[a] + (Ov[b1] * g[b2] - Ov[b2] * g[b1]);
        dgv[a] = dO0 * g[a] + (dOv[b1] * g[b2] - dOv[b2] * g[b1]) + O0 * hn[a] + (Ov[b1] * hn[b2] - Ov[b2] * hn[b1]);
      }
      // W = -sqrt2 Im(I[lambda_1] + I[gamma]), dW likewise, Theta = sqrt2 Im I[theta_1] (G2)
      double W[4], dW[4];
      W[0] = -s2 * inv4pi * (lam.s.y + gs.y);
      dW[0] = -s2 * inv4pi * (dlam.s.y + dgs.y);
      for (int a = 0; a < 3; ++a) {
        W[1 + a] = -s2 * inv4pi * (lam.v[a].y + gv[a].y);
        dW[1 + a] = -s2 * inv4pi * (dlam.v[a].y + dgv[a].y);
      }
      cd Slm = ws.R[hs];
      double Th = s2 * inv4pi * (th.y + Slm.y * O0);
      // zeta vectors (Step 8, App. A.7; reading G3 for S')
      double nxW[3];
      cross3(nup, W + 1, nxW);
      Zr[c] = Th;
      Zr[NP + c] = W[0];
      Zr[NP + NP + c] = -W[1];
      Zr[NP + 2 * NP + c] = -W[2];
      Zr[NP + 3 * NP + c] = -W[3];
      Zr[5 * NP + c] = dW[0];
      Zr[5 * NP + NP + c] = -dW[1];
      Zr[5 * NP + 2 * NP + c] = -dW[2];
      Zr[5 * NP + 3 * NP + c] = -dW[3];
      Zr[9 * NP + c] = -dot3(nup, W + 1);
      for (int a = 0; a < 3; ++a) Zr[9 * NP + (1 + a) * NP + c] = -W[0] * nup[a] - nxW[a];
    }
    if (lane == 0 && pstat) pstat[k - kbase] = (ws.conv[0] && ws.conv[1] && ws.conv[2]) ? 0 : 1;
    nswap += ws.swap[0] + ws.swap[1] + ws.swap[2];
    __syncwarp();
  }
  if (swapcnt && lane == 0 && nswap) atomicAdd(swapcnt, nswap);
}

// ------------------------------------------------------------------------------------------------
// Step 8 contraction + smooth subtraction + CSR store.  One CTA per work item (patch, up to TILE
// pairs).  Thread (i, g): node i, pair group g; each thread carries RB = TILE / G pairs.
// ------------------------------------------------------------------------------------------------
template <int P>
struct ContractCfg {
  static constexpr int N = Dims<P>::N;
  static constexpr int G = (128 / N) > 0 ? (128 / N) : 1;
  static constexpr int RB = ((P >= 8 ? 8 : 16) + G - 1) / G;   // pairs per thread
  static constexpr int TILE = RB * G;                          // pairs per CTA tile
  static constexpr int THREADS = ((G * N + 31) / 32) * 32;
};

template <int P>
__global__ void __launch_bounds__(ContractCfg<P>::THREADS)
    k_contract(int64_t n_items, const int64_t *__restrict__ item_ptr, int64_t n_patches,
               const int64_t *__restrict__ seg_ptr, const int64_t *__restrict__ perm,
               const int64_t *__restrict__ ptgt, int64_t kbase, const int32_t *__restrict__ pair_patch,
               const double *__restrict__ fit, const double *__restrict__ Z, const double *__restrict__ nodes,
               const double *__restrict__ normals, const double *__restrict__ weights,
               const double *__restrict__ tx, const double *__restrict__ tnorm, const int64_t *__restrict__ self_node,
               uint32_t mask, int raw, int32_t *__restrict__ col_idx, double *vS, double *vD, double *vSp,
               double *vDp, int32_t *__restrict__ pstat) {
  using D = Dims<P>;
  using L = Layout<P>;
  using CC = ContractCfg<P>;
  constexpr int N = D::N, NP = D::NP, NZ = D::NZ, TILE = CC::TILE, G = CC::G, RB = CC::RB;
  __shared__ double sZ[TILE][NZ];
  __shared__ double sT[TILE][7];     // target x, nu'
  __shared__ int64_t sK[TILE];
  __shared__ int sSelf[TILE];
  const int64_t item = blockIdx.x;
  if (item >= n_items) return;
  // patch of this item: largest P with item_ptr[P] <= item
  int64_t lo = 0, hi = n_patches;
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (item_ptr[mid] <= item) lo = mid; else hi = mid;
  }
  const int64_t Pp = lo;
  const int64_t s0 = seg_ptr[Pp] + (item - item_ptr[Pp]) * TILE;
  const int cnt = (int)min((int64_t)TILE, seg_ptr[Pp + 1] - s0);
  const double *blk = fit + Pp * (int64_t)L::STRIDE;
  const double h = blk[L::HDR + H_H];
  // stage the tile
  for (int i = threadIdx.x; i < TILE * NZ; i += blockDim.x) {
    int r = i / NZ, c = i % NZ;
    sZ[r][c] = r < cnt ? Z[(s0 + r) * NZ + c] : 0.0;
  }
  for (int r = threadIdx.x; r < TILE; r += blockDim.x) {
    if (r < cnt) {
      int64_t k = perm[s0 + r], t = ptgt[k - kbase];
      sK[r] = k;
      for (int a = 0; a < 3; ++a) {
        sT[r][a] = tx[3 * t + a];
        sT[r][3 + a] = tnorm ? tnorm[3 * t + a] : 0.0;
      }
      int sl = -1;
      if (self_node) {
        int64_t sn = self_node[t];
        if (sn >= 0 && sn / N == Pp) sl = (int)(sn % N);
      }
      sSelf[r] = sl;
    }
  }
  __syncthreads();
  const int i = threadIdx.x % N, g = threadIdx.x / N;
  if (g >= G) return;
  const double *PD = blk + L::FIT, *PSp = PD + 4 * NP * N, *PSd = PD + 8 * NP * N, *PSg = PD + 9 * NP * N;
  double aS[RB], aD[RB], aSp[RB], aDp[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) aS[r] = aD[r] = aSp[r] = aDp[r] = 0;
  for (int c = 0; c < NP; ++c) {
    double psd = __ldg(PSd + c * N + i);
#pragma unroll
    for (int r = 0; r < RB; ++r) aS[r] = fma(sZ[g + r * G][c], psd, aS[r]);
  }
  for (int c = 0; c < 4 * NP; ++c) {
    double pd = __ldg(PD + c * N + i), psp = __ldg(PSp + c * N + i), psg = __ldg(PSg + c * N + i);
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const double *z = sZ[g + r * G];
      double zw = z[NP + c], zdw = z[5 * NP + c], zs = z[9 * NP + c];
      aD[r] = fma(zw, pd, aD[r]);
      aDp[r] = fma(zdw, pd, aDp[r]);
      aSp[r] = fma(zs, psp, aSp[r]);
      aS[r] = fma(zw, psg, aS[r]);
    }
  }
  // epilogue: global units, smooth subtraction (reading A14), store
  const double *xi = nodes + (Pp * N + i) * 3, *ni = normals + (Pp * N + i) * 3;
  const double wi = weights[Pp * N + i];
  const double x0 = xi[0], x1 = xi[1], x2 = xi[2], n0 = ni[0], n1 = ni[1], n2 = ni[2];
  const double inv4pi = 1.0 / (4.0 * kPi);
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    const int rr = g + r * G;
    if (rr >= cnt) continue;
    double S = aS[r] * h, Dv = aD[r], Sp = aSp[r], Dp = aDp[r] / h;
    if (!raw && sSelf[rr] != i) {
      double d0 = sT[rr][0] - x0, d1 = sT[rr][1] - x1, d2 = sT[rr][2] - x2;
      double r2 = d0 * d0 + d1 * d1 + d2 * d2, ir = rsqrt(r2);
      ir = ir * (1.5 - 0.5 * r2 * ir * ir);   // one Newton step -> full fp64 accuracy
      double ir3 = ir * ir * ir;
      double dn = d0 * n0 + d1 * n1 + d2 * n2;
      double dnp = d0 * sT[rr][3] + d1 * sT[rr][4] + d2 * sT[rr][5];
      double nn = n0 * sT[rr][3] + n1 * sT[rr][4] + n2 * sT[rr][5];
      S -= inv4pi * ir * wi;
      Dv -= inv4pi * dn * ir3 * wi;
      Sp += inv4pi * dnp * ir3 * wi;
      Dp -= inv4pi * (nn * ir3 - 3.0 * dn * dnp * ir3 * ir * ir) * wi;
    }
    const int64_t o = (sK[rr] - kbase) * N + i;
    if (col_idx) col_idx[o] = (int32_t)(Pp * N + i);
    bool bad = false;
    if (vS) { vS[o] = (mask & 1) ? S : 0.0; bad |= !isfinite(S); }
    if (vD) { vD[o] = (mask & 2) ? Dv : 0.0; bad |= !isfinite(Dv); }
    if (vSp) { vSp[o] = (mask & 4) ? Sp : 0.0; bad |= !isfinite(Sp); }
    if (vDp) { vDp[o] = (mask & 8) ? Dp : 0.0; bad |= !isfinite(Dp); }
    if (bad && pstat) atomicOr(pstat + (sK[rr] - kbase), 2);
  }
}

// ------------------------------------------------------------------------------------------------
// Chunk plumbing: pair -> target, patch-major permutation, work items, row pointers.
// ------------------------------------------------------------------------------------------------
__global__ void k_pair_targets(int64_t row_begin, int64_t row_end, const int64_t *__restrict__ pair_ptr, int64_t kbase,
                               int64_t *__restrict__ ptgt, int64_t *__restrict__ row_ptr, int n) {
  int64_t t = row_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > row_end) return;
  if (row_ptr) row_ptr[t - row_begin] = (pair_ptr[t] - kbase) * n;
  if (t == row_end) return;
  for (int64_t k = pair_ptr[t]; k < pair_ptr[t + 1]; ++k) ptgt[k - kbase] = t;
}

__global__ void k_row_ptr(int64_t row_begin, int64_t row_end, const int64_t *__restrict__ pair_ptr, int64_t obase,
                          int64_t *__restrict__ row_ptr, int n) {
  int64_t t = row_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > row_end) return;
  row_ptr[t - row_begin] = (pair_ptr[t] - obase) * n;
}

__global__ void k_patch_hist(int64_t npairs, int64_t kbase, const int32_t *__restrict__ pair_patch,
                             int64_t *__restrict__ cnt) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= npairs) return;
  atomicAdd((unsigned long long *)(cnt + pair_patch[kbase + k]), 1ull);
}

__global__ void k_patch_scatter(int64_t npairs, int64_t kbase, const int32_t *__restrict__ pair_patch,
                                int64_t *__restrict__ cursor, int64_t *__restrict__ perm) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= npairs) return;
  unsigned long long pos = atomicAdd((unsigned long long *)(cursor + pair_patch[kbase + k]), 1ull);
  perm[pos] = kbase + k;
}

__global__ void k_items(int64_t n_patches, const int64_t *__restrict__ seg_ptr, int tile, int64_t *__restrict__ items) {
  int64_t P = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (P >= n_patches) return;
  int64_t c = seg_ptr[P + 1] - seg_ptr[P];
  items[P] = (c + tile - 1) / tile;
}

__global__ void k_copy_i64(int64_t n, const int64_t *__restrict__ a, int64_t *__restrict__ b) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}

// CSR SpMV: warp per row.
__global__ void k_apply(int64_t n_rows, const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                        const double *__restrict__ val, const double *__restrict__ x, double *__restrict__ y) {
  int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (r >= n_rows) return;
  double s = 0;
  for (int64_t k = row_ptr[r] + lane; k < row_ptr[r + 1]; k += 32) s += val[k] * __ldg(x + col[k]);
  s = warp_sum(s);
  if (lane == 0) y[r] += s;
}

}  // namespace rrq
