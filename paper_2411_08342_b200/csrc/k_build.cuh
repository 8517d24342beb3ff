// The per-pair hot path, Steps 4-8 + smooth-rule subtraction (A14), as
// kernels over a sub-chunk of pairs in patch-major order (s = position in the permutation):
//
// Producer stream (one sub-chunk ahead of the consumer):
// k_pair_setup (thread per pair): target frame, gauge, tile slots.
// k_newton (lane per edge, warp work queue): the near-singular parameter t0 of every (pair, edge) and the
//   regime flags (Step 5).
// k_edge_lines (CTA rounds; LP lanes per pair): model integrals and SSQ weights of the swap edges, the GEMM
//   rows a = omega1 d and b = omega1 nu' - omega3 (nu'.d) d (tile-chunked for k_qmap), the scalar line
//   integrals Omega, Omega_0 and derivatives (Steps 5-6).
// k_target_gamma (warp per 3 pairs): harmonics at the target (Step 4) -> translation operands S', NG', and the
//   I[gamma] part of W, dW and the S(r') Omega_0 part of Theta (Step 7).
// Consumer stream:
// k_qmap (CTA per tile of 16 pairs of one patch): the line-integral maps [Q | V](pair) = a M,
//   dQ(pair) = b M_Q as one FP64 tensor-core GEMM (mma.sync m8n8k4 f64 = DMMA) against the patch's
//   operand M (built in k_edge_tables).
// k_translate (warp per pair): translation (Step 7) -> W, dW, Theta -> contraction vectors zeta (written
//   tile-chunked for k_contract).
// k_contract (CTA per tile of 16 pairs of one patch): Step 8 in matrix mode as DMMA GEMMs
//   zeta^T [P_D | P_Sp | P_Sd | P_Sg], then smooth subtraction, scaling and the CSR store.
#pragma once
#include "rrq_device.cuh"

namespace rrq {

// Bernstein ellipse parameter (reading A5): rho(t) = a + sqrt(a^2 - 1) with a = (|t - 1| + |t + 1|) / 2 the
// semi-major axis of the confocal ellipse through t (= max |t +- sqrt(t^2 - 1)|), by rsqrt_nr.
__device__ __forceinline__ double sqrt_nn(double x) { return x > 0 ? x * rsqrt_nr(x) : 0.0; }
__device__ __forceinline__ double bernstein_rho(double re, double im) {
  const double y2 = im * im;
  const double a = 0.5 * (sqrt_nn((re - 1) * (re - 1) + y2) + sqrt_nn((re + 1) * (re + 1) + y2));
  return a + sqrt_nn(a * a - 1.0);
}

// Model integrals I_k, J_k (reading A11): upward recurrences, cancellation-free I_0, J_0.
template <int Q>
__device__ __noinline__ void model_integrals(double a, double b, double *I, double *J) {
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
  // the recurrence runs in registers (fully unrolled; /k as a multiplication by the constant 1/k)
  const double a2b2 = a * a + b * b, is1 = 1.0 / s1, ism = 1.0 / sm;
  const double be = s1 - sm, bo = s1 + sm, ge = is1 - ism, go = is1 + ism;   // k-1 even / odd
  double Im2 = I[0], Jm1 = J[0];
  double Im1 = (s1 - sm) + a * Im2;   // k = 1 (k-1 = 0 even)
  double J1 = a * Jm1 - (is1 - ism);
  I[1] = Im1;
  J[1] = J1;
  Jm1 = J1;
#pragma unroll
  for (int k = 2; k < Q; ++k) {
    const bool odd = ((k - 1) & 1) != 0;
    const double beta = odd ? bo : be, gam = odd ? go : ge;
    const double Ik = (beta + (2 * k - 1) * a * Im1 - (k - 1) * a2b2 * Im2) * (1.0 / k);
    const double Jk = a * Jm1 - gam + (k - 1) * Im2;
    I[k] = Ik;
    J[k] = Jk;
    Im2 = Im1;
    Im1 = Ik;
    Jm1 = Jk;
  }
}

// Phase profiling of k_edge_lines (SM cycles between the CTA barriers, accumulated by thread 0 of each
// CTA; read back with rrq_debug_phase_cycles); slots 8-15: k_patch_fit_q's phases (rrq_debug_fit_cycles).
__device__ unsigned long long g_phase_cycles[16];
#define RRQ_PHASE_MARK(ph)                                                         \
  if (threadIdx.x == 0) {                                                          \
    const long long now = clock64();                                               \
    atomicAdd(&g_phase_cycles[ph], (unsigned long long)(now - ph_t));             \
    ph_t = now;                                                                    \
  }

// Per-pair row of k_target_gamma's output for k_translate (doubles): the translation operands
// S'^{(l',m')} = w(l',m') S^{(l',m')}(r') and NG' = w(l',m') nu'.grad S^{(l',m')} for l' < p, all m' (expanded
// over m' < 0 by S^{(l,-m)} = (-1)^m conj S^{(l,m)}), stored per (l',m') at l'^2 + l' + m' as
// (S'.y, S'.x, NG'.y, NG'.x); the I[gamma] parts of W and dW ([4][NP], zeta sign convention NOT applied);
// the S(r') Omega_0 part of Theta ([NP]); nu' in the patch frame.
template <int P>
struct XRow {
  using D = Dims<P>;
  static constexpr int SX = 0, W = 4 * P * P, DW = W + 4 * D::NP, TH = DW + 4 * D::NP, NU = TH + D::NP,
                       G = W, GSZ = (9 * D::NP + 4 + 1) / 2 * 2, STRIDE = (G + GSZ + 15) / 16 * 16;   // rows 128-B aligned
};
// Per-pair row of k_qmap's output: per (j, k >= 0), 2 <= j <= p, at EG qidx(j,k): [Q (4 quaternion comps,
// re/im) | dQ (same)] scaled by v_lambda(j,k); then V [2 NV] scaled by v_theta(j,k) (TrCfg).
template <int P>
struct QRow {
  using D = Dims<P>;
  static constexpr int EG = 16;
  static constexpr int V = EG * D::NQ, STRIDE = (V + 2 * D::NV + 15) / 16 * 16;   // rows 128-B aligned
};

// k_translate's schedule (see k_translate).  Outputs (l, m), m = 1..l, are grouped in blocks of WD
// consecutive m (l, m0 .. m0 + WD - 1); a block's work is, for each j = 2..l, a sweep over k of the terms
// Q^{(j,k)} S'^{(l-j, m-k)} of all WD outputs at once (k from the smallest to the largest k any output of
// the block takes).  Along the sweep output m0 + i needs S'^{(l-j, m0+i-k)}, i.e. the entry output m0 took
// i steps earlier: a window of WD S' entries in registers, one new entry per step.
__host__ __device__ constexpr int tr_wd(int P) { return P <= 4 ? 4 : (P <= 6 ? 3 : (P <= 8 ? 3 : 5)); }
__host__ __device__ constexpr int tr_block_len(int l, int m0, int wd) {
  int n = 0;
  const int m1 = (m0 + wd - 1 < l) ? m0 + wd - 1 : l;
  for (int j = 2; j <= l; ++j) {
    const int lp = l - j;
    const int lo = (-j > m0 - lp) ? -j : m0 - lp, hi = (j < m1 + lp) ? j : m1 + lp;
    n += hi - lo + 1;
  }
  return n;
}
// lanes needed when every block is split into contiguous pieces of at most st steps
__host__ __device__ constexpr int tr_lanes(int P, int st) {
  int n = 0;
  for (int l = 2; l <= P; ++l)
    for (int m0 = 1; m0 <= l; m0 += tr_wd(P)) n += (tr_block_len(l, m0, tr_wd(P)) + st - 1) / st;
  return n;
}
__host__ __device__ constexpr int tr_steps(int P) {
  int st = 1;
  while (tr_lanes(P, st) > 32) ++st;
  return st;
}

template <int P>
struct TrCfg {
  using D = Dims<P>;
  static constexpr int WD = tr_wd(P), STEPS = tr_steps(P);
  // a lane's flush slot: WD x (theta, lambda[4], dlambda[4], pad) (16-B aligned per output), an odd number
  // of 16-B groups per slot (conflict-free stores)
  static constexpr int SLW = 10 * WD + (WD % 2 ? 0 : 2);
  static constexpr int SXW = 6;                                  // smem (S'.y, S'.x, NG'.y, NG'.x | pad): 48 B
  static constexpr int SXSZ = SXW * (P * P + 1);                 // + one zero entry (out-of-range S', padding)
  // staged Q block: NQ entries + a zero entry at stride EQ = 18 doubles (144 B: entries whose positions
  // differ mod 8 start in different 16-B bank groups), then V at SV + 2 vpos: j = 1 at 0, 1, the entry at
  // position pos at pos + 2 (the zero entry's V at NQ + 2)
  static constexpr int EQ = 18, ZQ = D::NQ, SV = EQ * (D::NQ + 1), QSZ = SV + 2 * (D::NQ + 3);
  // a staging buffer = [Q block | S' block]; after the sweep the current buffer holds the 32 flush slots
  static constexpr int BUF = QSZ + SXSZ > 32 * SLW ? QSZ + SXSZ : 32 * SLW;
  static_assert(QSZ % 2 == 0 && BUF % 2 == 0, "translate buffer");
  static constexpr int GSZ = XRow<P>::GSZ;
  // NBUF = 1: a warp stages its next pair after the current one's epilogue (the load latency is covered by
  // the other warps); the smaller footprint buys more warps per SM than double buffering (NBUF = 2)
  static constexpr int NBUF = 1, WMAX = P >= 10 ? 8 : 16;
  static constexpr int PER_WARP = (NBUF * BUF + GSZ + 1) / 2 * 2;
  // per-CTA table (host-built, rrq_api.cu make_trtab): u32 codes [STEPS][32], u32 prime codes [STEPS][32],
  // u32 cinfo [NP], u8 shared-memory positions of the Q entries [NQ] and of the S' entries [P*P] |
  // f64 vlam [NQ], vth [NV], wS [P*P], olam [NP], oth [NP]
  static constexpr int NWORD = 2 * STEPS * 32 + D::NP + (D::NQ + P * P + 3) / 4, TABW = (NWORD + 1) / 2;
  static constexpr int POSQ_BYTE = 4 * (2 * STEPS * 32 + D::NP), POSS_BYTE = POSQ_BYTE + D::NQ;
  static constexpr int VLAM = TABW, VTH = VLAM + D::NQ, WS = VTH + D::NV, OLAM = WS + P * P, OTH = OLAM + D::NP;
  static constexpr int TAB_D = (OTH + D::NP + 1) / 2 * 2;
  static constexpr int SMEM_MAX = 224 * 1024;
  static constexpr int WPB_FIT = (SMEM_MAX / 8 - TAB_D) / PER_WARP;
  static constexpr int WPB = WPB_FIT > WMAX ? WMAX : WPB_FIT;
  static constexpr size_t SMEM = (size_t)(TAB_D + WPB * PER_WARP) * sizeof(double);
  // code: Q position (7 bits) | new S' position << 7 (SEB bits: 7, or 8 once p^2 + 1 > 128) | FA | FB | PRIME;
  // prime code: S' positions of window entries 1 .. WD-1, SEB bits each.  cinfo: l | m << 4 | i << 8 |
  // first lane << 12 | lanes << 20.
  static constexpr int SEB = P * P < 128 ? 7 : 8;
  static constexpr uint32_t SEM = (1u << SEB) - 1;
  static constexpr uint32_t FA = 1u << (7 + SEB), FB = FA << 1, PRIME = FA << 3;
  static_assert(WPB >= 2, "translate smem");
  static_assert(D::NQ < 127 && P * P < (1 << SEB) && WD <= 5 && SEB * (WD - 1) <= 32 && P < 16, "translate code fields");
};

// D = A B + C for one 8x8x4 fp64 tile (FP64 tensor core, SASS DMMA).  Fragments: a = A[lane/4][lane%4],
// b = B[lane%4][lane/4], c/d = C[lane/4][2 (lane%4) + {0,1}].
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Legendre-series edge interpolant (reading A4'): value and derivatives of one component at t from
// coefficients held in registers, by Bonnet's recurrence (j+1) P_{j+1} = (2j+1) t P_j - j P_{j-1} and
// P'_{j+1} = P'_{j-1} + (2j+1) P_j, P''_{j+1} = P''_{j-1} + (2j+1) P'_j (fully unrolled: constant
// coefficients, no divisions).
template <int Q>
__device__ __forceinline__ void leg_r(const double (&Cl)[Q], double t, double &v, double &d1, double &d2) {
  double P0 = 1, P1 = t, a0 = 0, a1 = 1, b0 = 0, b1 = 0;
  v = fma(Cl[1], t, Cl[0]);
  d1 = Cl[1];
  d2 = 0;
#pragma unroll
  for (int j = 1; j + 1 < Q; ++j) {
    const double P2 = ((2.0 * j + 1.0) / (j + 1.0)) * t * P1 - ((double)j / (j + 1.0)) * P0;
    const double a2 = fma(2.0 * j + 1.0, P1, a0), b2 = fma(2.0 * j + 1.0, a1, b0);
    v = fma(Cl[j + 1], P2, v);
    d1 = fma(Cl[j + 1], a2, d1);
    d2 = fma(Cl[j + 1], b2, d2);
    P0 = P1; P1 = P2; a0 = a1; a1 = a2; b0 = b1; b1 = b2;
  }
}
template <int Q>
__device__ __forceinline__ void leg_c(const double (&Cl)[Q], cd t, cd &v, cd &d1) {
  cd P0 = mk(1, 0), P1 = t, a0 = mk(0, 0), a1 = mk(1, 0);
  v = mk(fma(Cl[1], t.x, Cl[0]), Cl[1] * t.y);
  d1 = mk(Cl[1], 0);
#pragma unroll
  for (int j = 1; j + 1 < Q; ++j) {
    const double ca = (2.0 * j + 1.0) / (j + 1.0), cb = (double)j / (j + 1.0);
    const cd tp = t * P1;
    const cd P2 = mk(ca * tp.x - cb * P0.x, ca * tp.y - cb * P0.y);
    const cd a2 = mk(fma(2.0 * j + 1.0, P1.x, a0.x), fma(2.0 * j + 1.0, P1.y, a0.y));
    v = mk(fma(Cl[j + 1], P2.x, v.x), fma(Cl[j + 1], P2.y, v.y));
    d1 = mk(fma(Cl[j + 1], a2.x, d1.x), fma(Cl[j + 1], a2.y, d1.y));
    P0 = P1; P1 = P2; a0 = a1; a1 = a2;
  }
}
// x(t), x'(t) (3 components, real t) from coefficients C[j*3 + c] (read uniformly across the warp)
template <int Q>
__device__ __forceinline__ void leg_r3(const double *__restrict__ C, double t, double x[3], double dx[3]) {
  double P0 = 1, P1 = t, a0 = 0, a1 = 1;
  for (int c = 0; c < 3; ++c) { x[c] = fma(C[3 + c], t, C[c]); dx[c] = C[3 + c]; }
#pragma unroll
  for (int j = 1; j + 1 < Q; ++j) {
    const double P2 = ((2.0 * j + 1.0) / (j + 1.0)) * t * P1 - ((double)j / (j + 1.0)) * P0;
    const double a2 = fma(2.0 * j + 1.0, P1, a0);
    for (int c = 0; c < 3; ++c) {
      const double cc = C[3 * (j + 1) + c];
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

// k_qmap's tile configuration (see k_qmap); k_edge_lines writes the A rows in its tile-chunked layout.
template <int P>
struct QmapCfg {
  using D = Dims<P>;
  static constexpr int TP = 16, ROWS = 2 * TP, WARPS = 8;
  static constexpr int PG = TP / 8, NSPLIT = WARPS / PG;        // warp = (pair group of 8, column split)
  static constexpr int TQC = D::CQP / 8;                      // tiles per quaternion component
  static constexpr int NTQ = D::NCQ / 8, NTALL = D::NCP / 8, NTV = NTALL - NTQ;
  static constexpr int UQ = (TQC + NSPLIT - 1) / NSPLIT;       // a warp's tiles per component (at most)
  // Two column passes (the accumulators of all 440 columns of a 32-row tile do not fit the register budget
  // with room to prefetch B fragments): pass 0 = components scalar, x; pass 1 = components y, z + the V tiles.
  // Column split ns takes the Q tiles tl = ns + NSPLIT u < TQC of its pass's two components (2 DMMA each: a
  // and b rows) and, in pass 1, a contiguous range of V tiles (1 DMMA each) sized so that the SM
  // sub-partitions' loads match: warp w = ns PG + pg runs on sub-partition w % 4, so splits {0, 2} share one
  // pair of sub-partitions and {1, 3} the other.  Counts are compile-time per split (no predicated DMMA).
  __host__ __device__ static constexpr int nq(int ns) { return (TQC - ns + NSPLIT - 1) / NSPLIT; }
  static constexpr int VA0 = (NTV + 4 * (nq(1) + nq(3)) - 4 * (nq(0) + nq(2)) + 1) / 2;
  static constexpr int VA = VA0 < 0 ? 0 : (VA0 > NTV ? NTV : VA0), VB = NTV - VA;
  __host__ __device__ static constexpr int vcount(int ns) { return ns == 0 ? (VA + 1) / 2 : ns == 2 ? VA / 2 : ns == 1 ? (VB + 1) / 2 : VB / 2; }
  __host__ __device__ static constexpr int vstart(int ns) { return ns == 0 ? 0 : ns == 1 ? vcount(0) : ns == 2 ? vcount(0) + vcount(1) : vcount(0) + vcount(1) + vcount(2); }
  static constexpr int UV = vcount(0) > vcount(1) ? (vcount(0) > vcount(2) ? (vcount(0) > vcount(3) ? vcount(0) : vcount(3)) : (vcount(2) > vcount(3) ? vcount(2) : vcount(3)))
                                                  : (vcount(1) > vcount(2) ? (vcount(1) > vcount(3) ? vcount(1) : vcount(3)) : (vcount(2) > vcount(3) ? vcount(2) : vcount(3)));
  // k-rows per chunk: 16 where it divides an axis block (p = 8): with 2 stages it costs the shared memory of 4
  // stages of 8 rows and is 5 % faster (half as many barrier round trips, 4 k-steps to schedule per chunk)
#ifdef RRQ_QMAP_KC   // experiments: chunk rows (must divide 3 p~) and stage count from the command line
  static constexpr int KC = (D::E % RRQ_QMAP_KC == 0) ? RRQ_QMAP_KC : ((D::E % 8 == 0) ? 8 : 12), NCH = D::K / KC, CPA = D::E / KC;
#else
  static constexpr int KC = (D::E % 16 == 0) ? 16 : ((D::E % 8 == 0) ? 8 : 12), NCH = D::K / KC, CPA = D::E / KC;
#endif
#ifndef RRQ_QMAP_NST
#define RRQ_QMAP_NST 4
#endif
  // pipeline stages (chunks in flight); p >= 12: the stage is 37 KB (p = 12) / 73 KB (p = 14), 1 CTA per SM
#ifdef RRQ_QMAP_KC
  static constexpr int NST = P <= 10 ? RRQ_QMAP_NST : (P == 12 ? 4 : 2);
#else
  static constexpr int NST = KC == 16 ? 2 : (P <= 10 ? RRQ_QMAP_NST : (P == 12 ? 4 : 2));
#endif
  // A (the tile's 32 GEMM rows) is stored tile-chunked by k_edge_lines: chunk ch = [32 rows][KC] (ACH doubles,
  // rows 0..15 = a-rows of the tile's pairs, 16..31 = b-rows), so a stage = [A chunk | B chunk] is two bulk
  // copies and A needs no resident shared memory.  KC = 8: the halves of rows with (r >> 1) odd are swapped
  // (k ^ 4) so a quarter-warp's A fragments fall in distinct banks.  A stage holds the larger pass's B chunk.
  static constexpr int ACH = ROWS * KC, ABLK = NCH * ACH, STG = ACH + KC * D::NCSH1;
  static_assert(D::E % KC == 0, "a B chunk must lie within one axis block");
  static_assert(NSPLIT == 4 && PG == 2, "sub-partition balance assumes 4 column splits x 2 pair groups");
  static constexpr int MINB = P <= 8 ? 2 : 1;                 // CTAs per SM (register budget)
  static constexpr size_t SMEM = (size_t)NST * STG * sizeof(double);
  __host__ __device__ static constexpr int swz(int r) { return KC == 16 ? (r & 3) << 2 : KC == 8 ? ((r >> 1) & 1) << 2 : 0; }
  // offset of A element (row r, k) in a tile block
  __host__ __device__ static constexpr int aoff(int r, int k) { return (k / KC) * ACH + r * KC + ((k % KC) ^ swz(r)); }
};

// Per-pair setup (thread per pair; latency-bound index chasing done with full occupancy): the target in
// the patch frame (A2: origin, rotation, scale 1/h), nu' in the frame, the self node, the gauge sign (A8).
struct __align__(16) PairSetup {
  double rp[3], nup[3], u3;
  int32_t Pp, self_local;
  int64_t k, aslot;   // aslot = (k_qmap tile of the pair within the sub-chunk) << 5 | row in the tile
};
static_assert(sizeof(PairSetup) == 80, "PairSetup layout");
// What k_contract's epilogue needs of a pair (global target position and normal, pair index, self node),
// written by k_pair_setup in the sub-chunk's patch-major order so a tile's entries are one bulk copy.
struct __align__(16) ContractPair {
  double x[3], n[3];
  int64_t k;
  int32_t self_local, pad;
};
static_assert(sizeof(ContractPair) == 64, "ContractPair layout");

template <int P>
__global__ void k_pair_setup(int64_t sA, int64_t sB, const int64_t *__restrict__ perm, const int64_t *__restrict__ ptgt,
                             int64_t kbase, const int32_t *__restrict__ pair_patch, const double *__restrict__ fit,
                             const double *__restrict__ tx, const double *__restrict__ tnorm,
                             const int64_t *__restrict__ self_node, const int8_t *__restrict__ side,
                             const int64_t *__restrict__ seg_ptr, const int64_t *__restrict__ item_ptr, int64_t it0,
                             PairSetup *__restrict__ setup, ContractPair *__restrict__ cpair) {
  using D = Dims<P>;
  using L = Layout<P>;
  const int64_t s = sA + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= sB) return;
        const int64_t k = perm[s], t = ptgt[k - kbase];
        const int Pp = pair_patch[k];
        const double *hd = fit + (int64_t)Pp * L::STRIDE + L::HDR;
        double rp[3], nup[3] = {0, 0, 0};
        {
          const double invh = 1.0 / hd[H_H];
          const double d[3] = {tx[3 * t] - hd[H_O], tx[3 * t + 1] - hd[H_O + 1], tx[3 * t + 2] - hd[H_O + 2]};
          for (int r = 0; r < 3; ++r) rp[r] = (hd[H_RM + 3 * r] * d[0] + hd[H_RM + 3 * r + 1] * d[1] + hd[H_RM + 3 * r + 2] * d[2]) * invh;
          if (tnorm) {
            const double *nn = tnorm + 3 * t;
            for (int r = 0; r < 3; ++r) nup[r] = hd[H_RM + 3 * r] * nn[0] + hd[H_RM + 3 * r + 1] * nn[1] + hd[H_RM + 3 * r + 2] * nn[2];
          }
        }
        int self_local = -1;
        if (self_node) {
          const int64_t sn = self_node[t];
          if (sn >= 0 && sn / D::N == Pp) self_local = (int)(sn % D::N);
        }
        const int sd = side ? (int)side[t] : 2;
        double sg;
        {
          const double z = rp[2] - hd[H_VL + 2], zlo = hd[H_ZLO], zhi = hd[H_ZHI];
          if (self_local >= 0) sg = -1.0;
          else if (z > zhi + 0.1) sg = 1.0;
          else if (z < zlo - 0.1) sg = -1.0;
          else {
            const double *va = hd + H_VL, *vb = hd + H_VL + 3, *vc = hd + H_VL + 6;
            const double det = (vb[0] - va[0]) * (vc[1] - va[1]) - (vc[0] - va[0]) * (vb[1] - va[1]);
            const double l1 = ((rp[0] - va[0]) * (vc[1] - va[1]) - (vc[0] - va[0]) * (rp[1] - va[1])) / det;
            const double l2 = ((vb[0] - va[0]) * (rp[1] - va[1]) - (rp[0] - va[0]) * (vb[1] - va[1])) / det;
            const double l0 = 1 - l1 - l2;
            const double mn = fmin(l0, fmin(l1, l2));
            if (mn >= -0.25 && sd != 2) sg = sd > 0 ? 1.0 : -1.0;
            else sg = (z - 0.5 * (zlo + zhi) > 0) ? 1.0 : -1.0;
          }
        }
        // whole records with 16-B stores
        double2 *q = reinterpret_cast<double2 *>(setup + (s - sA));
        q[0] = make_double2(rp[0], rp[1]);
        q[1] = make_double2(rp[2], nup[0]);
        q[2] = make_double2(nup[1], nup[2]);
        q[3] = make_double2(sg, __longlong_as_double((long long)(uint32_t)Pp | ((long long)self_local << 32)));
        const int64_t pos = s - seg_ptr[Pp], tile = item_ptr[Pp] + pos / QmapCfg<P>::TP - it0;
        q[4] = make_double2(__longlong_as_double(k), __longlong_as_double(tile << 5 | (pos % QmapCfg<P>::TP)));
        const double x0 = tx[3 * t], x1 = tx[3 * t + 1], x2 = tx[3 * t + 2];
        const double n0 = tnorm ? tnorm[3 * t] : 0.0, n1 = tnorm ? tnorm[3 * t + 1] : 0.0, n2 = tnorm ? tnorm[3 * t + 2] : 0.0;
        double2 *cp = reinterpret_cast<double2 *>(cpair + (s - sA));
        cp[0] = make_double2(x0, x1);
        cp[1] = make_double2(x2, n0);
        cp[2] = make_double2(n1, n2);
        cp[3] = make_double2(__longlong_as_double(k), __longlong_as_double((long long)(uint32_t)self_local));
}

// ------------------------------------------------------------------------------------------------
// k_newton: the near-singular parameter t0 of every (pair, edge) (Step 5; readings A12, A12',
// A12''), one lane per edge.  Work index w = e np + i (edge-major over the sub-chunk's patch-major pairs), so
// the lanes of a warp share the edge number and - but for patch boundaries - the patch: the Legendre
// coefficients of the edge interpolant (A4') are read through warp-uniform cached loads instead of living
// in registers, the three components of x(t) share one Legendre recurrence, and the sums over components
// are local to a lane (no shuffles).
// The complex Newton iteration count varies from 2 to 20 between edges, so a warp is a small work queue:
// it draws batches of 32 consecutive edges (one atomic per batch), computes their starting guesses
// together (3 real Newton steps + the quadratic model: uniform work) into shared-memory slots, and a lane
// whose edge has converged takes the next slot while the other lanes keep iterating.
// Output per edge: t0 (re, |im|) and a flag byte (bit 0 converged, bit 1 swap regime A5, bit 2 direct rule
// A11').
// ------------------------------------------------------------------------------------------------
constexpr int kNewtonThreads = 128, kNewtonSlot = 7;
// Bonnet recurrence constants: a[j] = (2j+1)/(j+1), b[j] = j/(j+1), d[j] = 2j+1
struct LegTab { double a[32], b[32], d[32]; };
constexpr LegTab make_leg_tab() {
  LegTab t{};
  for (int j = 0; j < 32; ++j) { t.a[j] = (2.0 * j + 1.0) / (j + 1.0); t.b[j] = (double)j / (j + 1.0); t.d[j] = 2.0 * j + 1.0; }
  return t;
}
__constant__ LegTab kLeg = make_leg_tab();

// Starting guess of one edge: chord projection, 3 real Newton steps on (x - r').x', quadratic-model complex
// guess (A12).  C2 = the edge's 3 Q Legendre coefficients [j][c] as 16-B pairs.
template <int Q>
__device__ __forceinline__ cd newton_guess(const double2 *__restrict__ C2, const double (&rc)[3]) {
  // chord projection: x(1) = sum_j C_j, x(-1) = sum_j (-1)^j C_j
  double abab = 0, arab = 0;
  {
    double v[3] = {0, 0, 0}, A[3] = {0, 0, 0};
#pragma unroll 1
    for (int j = 0; j < Q; j += 2) {   // coefficients of P_j, P_{j+1}: 3 aligned 16-B loads
      const double2 u0 = __ldg(C2 + 3 * (j >> 1)), u1 = __ldg(C2 + 3 * (j >> 1) + 1), u2 = __ldg(C2 + 3 * (j >> 1) + 2);
      v[0] += u0.x; A[0] += u0.x; v[1] += u0.y; A[1] += u0.y; v[2] += u1.x; A[2] += u1.x;
      v[0] += u1.y; A[0] -= u1.y; v[1] += u2.x; A[1] -= u2.x; v[2] += u2.y; A[2] -= u2.y;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double ab = v[c] - A[c], ar = rc[c] - A[c];
      abab += ab * ab;
      arab += ar * ab;
    }
  }
  double tc = -1.0 + 2.0 * arab / (abab > 0 ? abab : 1.0);
  // x(t) - r', x'(t), x''(t) at real t (Bonnet's recurrence and its derivatives, one recurrence for the 3
  // components).  The j loop is rolled two steps at a time (recurrence constants from kLeg) so that the
  // compiler does not hoist all 3 Q coefficient loads into registers.
  double xr[3], d1[3], d2[3];
  auto eval_r = [&](double t) {
    double P0 = 1, P1 = t, a0 = 0, a1 = 1, b0 = 0, b1 = 0;
    {
      const double2 u0 = __ldg(C2), u1 = __ldg(C2 + 1), u2 = __ldg(C2 + 2);
      const double c0[3] = {u0.x, u0.y, u1.x}, c1[3] = {u1.y, u2.x, u2.y};
#pragma unroll
      for (int c = 0; c < 3; ++c) { xr[c] = fma(c1[c], t, c0[c]) - rc[c]; d1[c] = c1[c]; d2[c] = 0; }
    }
#pragma unroll 1
    for (int j = 1; j + 1 < Q; j += 2) {   // coefficients of P_{j+1}, P_{j+2}: flat index 3 (j + 1), even
      const double2 *cp = C2 + 3 * ((j + 1) >> 1);
      const double2 u0 = __ldg(cp), u1 = __ldg(cp + 1), u2 = __ldg(cp + 2);
      const double cj[2][3] = {{u0.x, u0.y, u1.x}, {u1.y, u2.x, u2.y}};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double P2 = kLeg.a[j + h] * t * P1 - kLeg.b[j + h] * P0;
        const double a2 = fma(kLeg.d[j + h], P1, a0), b2 = fma(kLeg.d[j + h], a1, b0);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          xr[c] = fma(cj[h][c], P2, xr[c]);
          d1[c] = fma(cj[h][c], a2, d1[c]);
          d2[c] = fma(cj[h][c], b2, d2[c]);
        }
        P0 = P1; P1 = P2; a0 = a1; a1 = a2; b0 = b1; b1 = b2;
      }
    }
  };
  bool go = true;
#pragma unroll 1
  for (int it = 0; it < 3; ++it) {
    eval_r(tc);
    const double g = xr[0] * d1[0] + xr[1] * d1[1] + xr[2] * d1[2];
    const double gp = (d1[0] * d1[0] + xr[0] * d2[0]) + (d1[1] * d1[1] + xr[1] * d2[1]) + (d1[2] * d1[2] + xr[2] * d2[2]);
    go = go && (gp > 0);
    if (go) tc -= g * rcp_nr(gp);
  }
  eval_r(tc);
  const double f = xr[0] * xr[0] + xr[1] * xr[1] + xr[2] * xr[2], xp2 = d1[0] * d1[0] + d1[1] * d1[1] + d1[2] * d1[2];
  double dd = (d1[0] * d1[0] + xr[0] * d2[0]) + (d1[1] * d1[1] + xr[1] * d2[1]) + (d1[2] * d1[2] + xr[2] * d2[2]);
  if (!(dd > 0)) dd = xp2;
  return mk(tc, sqrt_nn(f * rcp_nr(dd > 0 ? dd : 1.0)));
}

// One complex Newton step t <- t - F / F', F(t) = (x(t) - r').(x(t) - r'); returns the step dt.
template <int Q>
__device__ __forceinline__ cd newton_step(const double2 *__restrict__ C2, const double (&rc)[3], cd tz) {
  cd P0 = mk(1, 0), P1 = tz, a0 = mk(0, 0), a1 = mk(1, 0), xv[3], xd[3];
  {
    const double2 u0 = __ldg(C2), u1 = __ldg(C2 + 1), u2 = __ldg(C2 + 2);
    const double c0[3] = {u0.x, u0.y, u1.x}, c1[3] = {u1.y, u2.x, u2.y};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      xv[c] = mk(fma(c1[c], tz.x, c0[c]) - rc[c], c1[c] * tz.y);
      xd[c] = mk(c1[c], 0);
    }
  }
#pragma unroll 1
  for (int j = 1; j + 1 < Q; j += 2) {
    const double2 *cp = C2 + 3 * ((j + 1) >> 1);
    const double2 u0 = __ldg(cp), u1 = __ldg(cp + 1), u2 = __ldg(cp + 2);
    const double cj[2][3] = {{u0.x, u0.y, u1.x}, {u1.y, u2.x, u2.y}};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const double ca = kLeg.a[j + h], cb = kLeg.b[j + h], dj = kLeg.d[j + h];
      const cd tp = tz * P1;
      const cd P2 = mk(ca * tp.x - cb * P0.x, ca * tp.y - cb * P0.y);
      const cd a2 = mk(fma(dj, P1.x, a0.x), fma(dj, P1.y, a0.y));
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        xv[c] = mk(fma(cj[h][c], P2.x, xv[c].x), fma(cj[h][c], P2.y, xv[c].y));
        xd[c] = mk(fma(cj[h][c], a2.x, xd[c].x), fma(cj[h][c], a2.y, xd[c].y));
      }
      P0 = P1; P1 = P2; a0 = a1; a1 = a2;
    }
  }
  cd F = mk(0, 0), Fp = mk(0, 0);
#pragma unroll
  for (int c = 0; c < 3; ++c) { F = F + xv[c] * xv[c]; Fp = Fp + xv[c] * xd[c]; }
  return cdiv(F, 2.0 * Fp);
}

template <int P>
__global__ void __launch_bounds__(kNewtonThreads, 4)
    k_newton(int64_t np_, const PairSetup *__restrict__ setup, const double *__restrict__ fit, double rho0,
             double2 *__restrict__ T0, uint8_t *__restrict__ EF, unsigned long long *__restrict__ counter) {
  using D = Dims<P>;
  using L = Layout<P>;
  constexpr int Q = D::Q;
  __shared__ double slots[kNewtonThreads / 32][32][kNewtonSlot];   // tz, r'[3], w, patch (odd stride)
  const int lane = threadIdx.x & 31;
  double (*sl)[kNewtonSlot] = slots[threadIdx.x >> 5];
  const long long total = 3 * np_;
  auto coef = [&](long long w, int Pp) {
    const int e = w >= 2 * np_ ? 2 : (w >= np_ ? 1 : 0);
    return reinterpret_cast<const double2 *>(fit + (int64_t)Pp * L::STRIDE + L::CM + e * Q * 3);
  };
  // lane state: the edge being iterated
  bool have = false;
  long long w = 0;
  cd tz = mk(0, 0);
  double rc[3] = {0, 0, 0}, dt2_prev = 0;
  const double2 *C2 = nullptr;
  int it = 0;
  int avail = 0, head = 0;   // warp-uniform: unclaimed slots of the current batch
  bool more = true;
  for (;;) {
    unsigned need = __ballot_sync(0xffffffffu, !have);
    while (need && (avail > 0 || more)) {
      if (avail == 0) {   // draw the next batch and compute its starting guesses (all lanes together)
        long long b = 0;
        if (lane == 0) b = (long long)atomicAdd(counter, 32ull);
        b = __shfl_sync(0xffffffffu, b, 0);
        if (b >= total) { more = false; break; }
        avail = (int)(total - b < 32 ? total - b : 32);
        head = 0;
        __syncwarp();
        if (lane < avail) {
          const long long wn = b + lane;
          const int e = wn >= 2 * np_ ? 2 : (wn >= np_ ? 1 : 0);
          const PairSetup &q = setup[wn - e * np_];
          const double r3[3] = {q.rp[0], q.rp[1], q.rp[2]};
          const int Pp = q.Pp;
          const cd g = newton_guess<Q>(coef(wn, Pp), r3);
          double *o = sl[lane];
          o[0] = g.x; o[1] = g.y; o[2] = r3[0]; o[3] = r3[1]; o[4] = r3[2];
          o[5] = __longlong_as_double(wn); o[6] = __longlong_as_double((long long)Pp);
        }
        __syncwarp();
      }
      const int rank = __popc(need & ((1u << lane) - 1u));
      if (!have && rank < avail) {
        const double *o = sl[head + rank];
        tz = mk(o[0], o[1]);
        rc[0] = o[2]; rc[1] = o[3]; rc[2] = o[4];
        w = __double_as_longlong(o[5]);
        C2 = coef(w, (int)__double_as_longlong(o[6]));
        have = true;
        it = 0;
        dt2_prev = 0;
      }
      const int nt = min(__popc(need), avail);
      head += nt;
      avail -= nt;
      need = __ballot_sync(0xffffffffu, !have);
    }
    if (!__any_sync(0xffffffffu, have)) break;
    if (have) {
      const cd dt = newton_step<Q>(C2, rc, tz);
      tz = tz - dt;
      bool conv = false;
      // |dt| < 1e-15 (1 + |t|) and |dt| < 1e-3 |t| compared as squares (no hypot)
      const double dt2 = dt.x * dt.x + dt.y * dt.y, tz2 = tz.x * tz.x + tz.y * tz.y;
      const double tza = tz2 > 0 ? tz2 * rsqrt_nr(tz2) : 0.0;
      const double tol2 = 1e-30 * (1.0 + tza) * (1.0 + tza);
      if (dt2 < tol2) conv = true;
      // A12'': quadratic regime and the predicted next step |dt|^3 / |dt_prev|^2 below the tolerance
      else if (dt2_prev > 0 && dt2 < 1e-2 * dt2_prev && dt2 * dt2 * dt2 < tol2 * dt2_prev * dt2_prev) conv = true;
      // A12': root certainly outside the swap ellipse
      else if (it >= 1 && dt2 < 1e-6 * tz2 && bernstein_rho(tz.x, tz.y) > 2.0 * rho0) conv = true;
      dt2_prev = dt2;
      ++it;
      if (conv || it == 20) {
        if (tz.y < 0) tz.y = -tz.y;
        conv = conv && isfinite(tz.x) && isfinite(tz.y);
        const double rho = bernstein_rho(tz.x, tz.y);
        T0[w] = make_double2(tz.x, tz.y);
        EF[w] = (uint8_t)((conv ? 1 : 0) | ((conv && rho < rho0) ? 2 : 0) | ((rho >= kRhoDirect) ? 4 : 0));
        have = false;
      }
    }
  }
}

// ------------------------------------------------------------------------------------------------
// k_edge_lines: the edge work of a pair after k_newton (Steps 5-6):
// model integrals and SSQ weights of the swap-regime edges, the GEMM rows a = omega1 d and
// b = omega1 nu' - omega3 (nu'.d) d (tile-chunked for k_qmap), the scalar line integrals Omega, Omega_0 and
// their nu'-derivatives (OM, 8 doubles per pair), Omega_0 on swap edges by the sinh rule (A9).
// CTA rounds of WPB * PPW pairs in three barrier-separated steps: (1) every warp loads its pairs' setup and
// t0 / flags and lists the swap edges CTA-wide; (2) the model integrals (a thread per edge inside rho = 1.6,
// a warp per edge with the 48-point rule outside) and the sinh rule (a warp per edge, round-robin over the
// list); (3) the weights: LP lanes per pair sweep its 3 p~ edge nodes (p = 8: a half-warp
// per pair, one edge per sweep).
// ------------------------------------------------------------------------------------------------
template <int P>
struct EdgeCfg {
  using D = Dims<P>;
  static constexpr int WPB = 8;
  static constexpr int LP = (D::E % 32 == 0 || P > 8) ? 32 : 16;   // lanes per pair in the weights step
  static constexpr int HW = 32 / LP;                               // pairs side by side in a warp
  static constexpr int PPW = 3 * HW;                               // pairs per warp per round (48-pair CTA rounds at p <= 8)
  static constexpr int MINB = P <= 8 ? 3 : 2;
};
template <int P>
struct EdgePair {
  using D = Dims<P>;
  double I[3][D::Q], J[3][D::Q];
  double t0[3][2];
  double rp[3], nup[3], u3, o0e[3];
  int64_t k, aslot;               // PairSetup::k, aslot
  int Pp, self_local, active, pad;
  int swap[3], conv[3], direct[3], pad2;
};

// Sums of 8 values over the LP lanes of a group (LP = 16: 8 shuffles; LP = 32: warp_sum8): on return lane L
// holds the sum of value index ((L >> 2) & 7) (LP = 32) or ((L >> 1) & 7) (LP = 16) of its group.
template <int LP>
__device__ __forceinline__ double group_sum8(const double (&v)[8], int lane) {
  if constexpr (LP == 32) {
    return warp_sum8(v, lane);
  } else {
    const bool b3 = (lane >> 3) & 1, b2 = (lane >> 2) & 1, b1 = (lane >> 1) & 1;
    double w[4], x[2];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double keep = b3 ? v[4 + j] : v[j], send = b3 ? v[j] : v[4 + j];
      w[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const double keep = b2 ? w[2 + j] : w[j], send = b2 ? w[j] : w[2 + j];
      x[j] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    double y = (b1 ? x[1] : x[0]) + __shfl_xor_sync(0xffffffffu, b1 ? x[0] : x[1], 2);
    y += __shfl_xor_sync(0xffffffffu, y, 1);
    return y;
  }
}

template <int P>
__global__ void __launch_bounds__(EdgeCfg<P>::WPB * 32, EdgeCfg<P>::MINB)
    k_edge_lines(int64_t sA, int64_t sB, const double *__restrict__ fit, Tables T, int n_omega,
                 double *__restrict__ Arow, double *__restrict__ OM, int32_t *__restrict__ pstat, int64_t obase,
                 unsigned long long *__restrict__ swapcnt, const PairSetup *__restrict__ setup, int want_dp,
                 const double2 *__restrict__ T0, const uint8_t *__restrict__ EF) {
  using D = Dims<P>;
  using L = Layout<P>;
  using EC = EdgeCfg<P>;
  using QC = QmapCfg<P>;
  constexpr int Q = D::Q, E = D::E, WPB = EC::WPB, PPW = EC::PPW, LP = EC::LP, HW = EC::HW;
  extern __shared__ double smem[];
  double *sU = smem;                  // [Q][Q]
  double *stgl = sU + Q * Q, *swgl = stgl + Q;
  double *sxo = swgl + Q, *swo = sxo + n_omega;
  double *sxdp = swo + n_omega;       // [kNDirect][Q] powers of the direct-rule nodes (reading A11')
  double *sr13 = sxdp + kNDirect * Q; // [WPB][2][kNDirect] direct-rule scratch
  int tab_doubles = Q * Q + 2 * Q + 2 * n_omega + kNDirect * Q + WPB * 2 * kNDirect;
  tab_doubles = (tab_doubles + 1) & ~1;
  EdgePair<P> *pst = reinterpret_cast<EdgePair<P> *>(smem + tab_doubles);
  __shared__ int nsw;                          // swap edges of the round (CTA-wide list)
  __shared__ int swl[WPB * PPW * 3];
  for (int i = threadIdx.x; i < Q * Q; i += blockDim.x) sU[i] = T.U[i];
  for (int i = threadIdx.x; i < Q; i += blockDim.x) { stgl[i] = T.tgl[i]; swgl[i] = T.wgl[i]; }
  for (int i = threadIdx.x; i < n_omega; i += blockDim.x) { sxo[i] = T.xo[i]; swo[i] = T.wo[i]; }
  for (int i = threadIdx.x; i < kNDirect * Q; i += blockDim.x) sxdp[i] = T.xdp[i];
  if (threadIdx.x == 0) nsw = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double *r13 = sr13 + warp * 2 * kNDirect;
  EdgePair<P> *mine = pst + warp * PPW;
  unsigned long long nswap = 0;
  const int64_t np_ = sB - sA;
  long long ph_t = clock64();
  for (int64_t base = sA + (int64_t)blockIdx.x * WPB * PPW; base < sB; base += (int64_t)gridDim.x * WPB * PPW) {
    // ---------------- step 1: the warp's pairs (k_pair_setup, k_newton) and the swap-edge list
    if (lane < PPW) {
      EdgePair<P> &ps = mine[lane];
      const int64_t s = base + warp * PPW + lane;
      const bool active = s < sB;
      ps.active = active;
      if (active) {
        const PairSetup &q = setup[s - sA];
        ps.k = q.k; ps.Pp = q.Pp; ps.self_local = q.self_local; ps.u3 = q.u3; ps.aslot = q.aslot;
        for (int a = 0; a < 3; ++a) { ps.rp[a] = q.rp[a]; ps.nup[a] = q.nup[a]; }
      }
    }
    if (lane >= 8 && lane < 8 + 3 * PPW) {
      const int pp = (lane - 8) / 3, e = (lane - 8) % 3;
      EdgePair<P> &ps = mine[pp];
      const int64_t s = base + warp * PPW + pp;
      if (s < sB) {
        const int64_t w = e * np_ + (s - sA);
        const double2 tz = T0[w];
        const int fl = EF[w];
        ps.t0[e][0] = tz.x;
        ps.t0[e][1] = tz.y;
        ps.conv[e] = fl & 1;
        ps.swap[e] = (fl >> 1) & 1;
        ps.direct[e] = (fl >> 2) & 1;
        if (fl & 2) swl[atomicAdd(&nsw, 1)] = (warp * PPW + pp) * 3 + e;
      }
    }
    __syncthreads();
    RRQ_PHASE_MARK(0);
    // ---------------- step 2: model integrals (reading A11 / A11') and Omega_0 on the swap edges by the
    // sinh-split Gauss-Legendre rule (reading A9)
    // warp 0: the recurrences (a lane per edge; one long scalar dependency chain each); warps 1 ..: the per-edge
    // warp work, so no warp has both on its critical path to the barrier
    const int nsw_ = nsw;
    if (warp == 0)
      for (int q = lane; q < nsw_; q += 32) {
        EdgePair<P> &ps = pst[swl[q] / 3];
        const int e = swl[q] % 3;
        if (!ps.direct[e]) model_integrals<Q>(ps.t0[e][0], fabs(ps.t0[e][1]), ps.I[e], ps.J[e]);
      }
    for (int q = warp - 1; q >= 0 && q < nsw_; q += WPB - 1) {
      const int code = swl[q], e = code % 3;
      EdgePair<P> &ps = pst[code / 3];
      const double *blk = fit + (int64_t)ps.Pp * L::STRIDE;
      if (ps.direct[e]) {   // 48-point rule for rho(t0) >= 1.6
        const double a = ps.t0[e][0], b = fabs(ps.t0[e][1]);
        for (int j = lane; j < kNDirect; j += 32) {
          const double xj = T.xd[j], Qv = (xj - a) * (xj - a) + b * b, rs = rsqrt(Qv);
          const double r1 = T.wd[j] * rs;
          r13[j] = r1;
          r13[kNDirect + j] = r1 * rs * rs;
        }
        __syncwarp();
        if (lane < Q) {   // two interleaved partial sums (shorter dependency chains)
          double si0 = 0, sj0 = 0, si1 = 0, sj1 = 0;
#pragma unroll 4
          for (int j = 0; j < kNDirect; j += 2) {
            const double pw0 = sxdp[j * Q + lane], pw1 = sxdp[(j + 1) * Q + lane];
            si0 = fma(pw0, r13[j], si0);
            sj0 = fma(pw0, r13[kNDirect + j], sj0);
            si1 = fma(pw1, r13[j + 1], si1);
            sj1 = fma(pw1, r13[kNDirect + j + 1], sj1);
          }
          ps.I[e][lane] = si0 + si1;
          ps.J[e][lane] = sj0 + sj1;
        }
        __syncwarp();
      }
      const double rp[3] = {ps.rp[0], ps.rp[1], ps.rp[2]};
      const double u[3] = {0.0, 0.0, ps.u3};
      const double a = fmin(1.0, fmax(-1.0, ps.t0[e][0])), b = fabs(ps.t0[e][1]);
      const double sR = asinh((1 - a) / b), sL = asinh((-1 - a) / b);
      const double *C = blk + L::CM + e * Q * 3;
      double acc = 0;
      for (int j = lane; j < 2 * n_omega; j += 32) {
        const int sdd = j / n_omega, jj = j % n_omega;
        const double lo = sdd ? 0.0 : sL, hi = sdd ? sR : 0.0;
        if (!(hi > lo)) continue;
        const double sv = lo + (hi - lo) * (sxo[jj] + 1) * 0.5, W = (hi - lo) * 0.5 * swo[jj];
        const double ex = exp(sv), iex = rcp_nr(ex);
        const double tt = a + b * 0.5 * (ex - iex), dt = b * 0.5 * (ex + iex);
        double x[3], dx[3];
        leg_r3<Q>(C, tt, x, dx);
        const double d[3] = {rp[0] - x[0], rp[1] - x[1], rp[2] - x[2]};
        const double nd2 = dot3(d, d), nd = nd2 * rsqrt_nr(nd2);
        double dxu[3];
        cross3(d, u, dxu);
        acc += W * dt * (-dot3(dxu, dx) * rcp_nr(nd * (nd + dot3(u, d))));
      }
      acc = warp_sum(acc);
      if (lane == 0) ps.o0e[e] = acc;
    }
    __syncthreads();
    RRQ_PHASE_MARK(1);
    // ---------------- step 3: weights and the scalar line integrals (Step 6)
    if (threadIdx.x == 0) nsw = 0;   // read last in step 2; written next after the round's barrier
    const int sub = lane % LP, grp = lane / LP;
#pragma unroll 1
    for (int r = 0; r < PPW / HW; ++r) {
      const int pp = r * HW + grp;
      EdgePair<P> &ps = mine[pp];
      const bool act = ps.active;
      const double *blk = fit + (int64_t)(act ? ps.Pp : 0) * L::STRIDE;
      const int64_t aslot = act ? ps.aslot : 0;
      double *Ar = Arow + (aslot >> 5) * QC::ABLK;   // k_qmap's tile block (tile-chunked rows)
      const int arow_ = (int)(aslot & 31);
      const double rp[3] = {ps.rp[0], ps.rp[1], ps.rp[2]}, nup[3] = {ps.nup[0], ps.nup[1], ps.nup[2]};
      const double u[3] = {0.0, 0.0, ps.u3};
      double om[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // Omega_0(plain) Omega[3] dOmega_0 dOmega[3]
      if (act) {
        for (int kap = sub; kap < E; kap += LP) {
          const int e = kap / Q, kk = kap % Q;
          const double *y = blk + L::YL + 3 * kap, *tau = blk + L::TL + 3 * kap;
          const double d[3] = {rp[0] - y[0], rp[1] - y[1], rp[2] - y[2]};
          const double d2 = dot3(d, d), idn = rsqrt_nr(d2), dn = d2 * idn;   // |d| > 0: targets are off the edges
          double w1, w3;
          if (ps.swap[e]) {
            double mu1 = 0, mu3 = 0;
#pragma unroll 4
            for (int c = 0; c < Q; ++c) {
              mu1 = fma(ps.I[e][c], sU[c * Q + kk], mu1);
              mu3 = fma(ps.J[e][c], sU[c * Q + kk], mu3);
            }
            const double ta = stgl[kk] - ps.t0[e][0], tb = ps.t0[e][1];
            const double tt2 = ta * ta + tb * tb, r1 = tt2 * rsqrt_nr(tt2) * idn;
            w1 = mu1 * r1;
            w3 = mu3 * r1 * r1 * r1;
          } else {
            w1 = swgl[kk] * idn;
            w3 = w1 * idn * idn;
            double dxu[3];
            cross3(d, u, dxu);
            om[0] += swgl[kk] * (-dot3(dxu, tau) * rcp_nr(dn * (dn + dot3(u, d))));
          }
          const double nd = dot3(nup, d);
          double txd[3];
          cross3(tau, d, txd);
          for (int a = 0; a < 3; ++a) {
            Ar[QC::aoff(arow_, a * E + kap)] = w1 * d[a];                                 // row a (k = axis E + kappa)
            if (want_dp) Ar[QC::aoff(QC::TP + arow_, a * E + kap)] = w1 * nup[a] - w3 * nd * d[a];   // row b (D')
            om[1 + a] -= w1 * tau[a];
            om[5 + a] += w3 * nd * tau[a];
          }
          om[4] += w3 * dot3(nup, txd);
        }
      }
      double red = group_sum8<LP>(om, lane);
      const int vi = LP == 32 ? (lane >> 2) & 7 : (lane >> 1) & 7;
      const bool writer = LP == 32 ? (lane & 3) == 0 : (lane & 1) == 0;
      if (act && writer) {
        if (vi == 0) {   // Omega_0: the swap edges' sinh-rule parts and the principal-value shift (reading A7)
          for (int e = 0; e < 3; ++e)
            if (ps.swap[e]) red += ps.o0e[e];
          if (ps.self_local >= 0) red -= 2.0 * kPi;
        }
        OM[(base + warp * PPW + pp - sA) * 8 + vi] = red;
      }
    }
    if (lane < PPW) {
      EdgePair<P> &ps = mine[lane];
      if (ps.active) {
        if (pstat) pstat[ps.k - obase] = (ps.conv[0] && ps.conv[1] && ps.conv[2]) ? 0 : 1;
        nswap += ps.swap[0] + ps.swap[1] + ps.swap[2];
      }
    }
    __syncthreads();
    RRQ_PHASE_MARK(2);
  }
  if (swapcnt && nswap) atomicAdd(swapcnt, nswap);
}

// ------------------------------------------------------------------------------------------------
// k_target_gamma: the target-side harmonics of a pair (Step 4) and the I[gamma] parts (Step 7):
// S, grad S, nu'.grad S, Hess S nu' at r' -> the translation operands S', NG' (XRow), and with the scalar
// line integrals OM of k_edge_lines: I[gamma] = (Omega_0, Omega)(0, grad S(r')), its
// nu'-derivative, W_gamma = -sqrt2 Im I[gamma], and the S(r') Omega_0 part of Theta (G2).
// k_translate adds the lambda_1 / theta_1 parts.  Warp per 3 pairs, no CTA barrier: lane = (pair, column m)
// holds R_l^m of its column in registers, neighbour columns by shuffles.
// ------------------------------------------------------------------------------------------------
template <int P>
struct TgtPair {
  using D = Dims<P>;
  cd R[D::NS];                 // R_l^m at (y', z', x'): S^{(l,m)}(r') for m >= 0
  double rp[3], nup[3], om[8];
  int64_t aslot;
  int active, pad;
};
template <int P>
struct TgtCfg {
  using D = Dims<P>;
  static constexpr int WPB = P >= 14 ? 4 : 8;
  // pairs per warp per round: as many as fit with one lane per (pair, column m), m = 0..p (the register-column
  // path); p = 10: 3 pairs through the shared-memory table path (2 pairs of 11 columns measured 40 % slower)
  static constexpr int PPW = P == 10 ? 3 : (32 / (P + 1) > 6 ? 6 : 32 / (P + 1));
  static constexpr size_t PER_WARP = sizeof(cd) * PPW * D::NS * 3 + PPW * sizeof(TgtPair<P>);
  static constexpr size_t SMEM = (size_t)(hc_size(P) + P * P) * sizeof(double) + WPB * PER_WARP;
  static constexpr int MINB = P <= 8 ? 2 : 1;
};

template <int P>
__global__ void __launch_bounds__(TgtCfg<P>::WPB * 32, TgtCfg<P>::MINB)
    k_target_gamma(int64_t sA, int64_t sB, Tables T, double *__restrict__ Xrow, const double *__restrict__ OM,
                   const double *__restrict__ trtab, const PairSetup *__restrict__ setup, int want_dp) {
  using D = Dims<P>;
  using XR = XRow<P>;
  constexpr int NP = D::NP, NS = D::NS, WPB = TgtCfg<P>::WPB, kPPW = TgtCfg<P>::PPW, NPO = (8 * kPPW + 31) / 32;
  extern __shared__ double smem[];
  double *shc = smem;   // [hc_size(P)]
  double *wS = smem + hc_size(P);   // [P * P] w(l', m') of the translation operands (TrCfg)
  for (int i = threadIdx.x; i < hc_size(P); i += blockDim.x) shc[i] = T.hc[i];
  for (int i = threadIdx.x; i < P * P; i += blockDim.x) wS[i] = trtab[TrCfg<P>::WS + i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char *wbase = reinterpret_cast<unsigned char *>(smem + hc_size(P) + P * P) + (size_t)warp * TgtCfg<P>::PER_WARP;
  cd (*GS)[NS][3] = reinterpret_cast<cd (*)[NS][3]>(wbase);
  TgtPair<P> *mine = reinterpret_cast<TgtPair<P> *>(wbase + sizeof(cd) * kPPW * NS * 3);
  const double inv4pi = 1.0 / (4.0 * kPi), s2 = 1.4142135623730950488;
  // the round's inputs (lanes < PPW: a pair's setup record; all lanes: the 8 PPW scalar line integrals) are
  // loaded one round ahead into registers, so their latency is covered by the previous round's work
  const int64_t stride = (int64_t)gridDim.x * WPB * kPPW;
  double pv[6] = {0, 0, 0, 0, 0, 0}, po[NPO];
  int64_t pa = 0;
  auto prefetch = [&](int64_t b) {
    if (lane < kPPW && b + lane < sB) {
      const PairSetup &q = setup[b + lane - sA];
      pa = q.aslot;
      for (int a = 0; a < 3; ++a) { pv[a] = q.rp[a]; pv[3 + a] = q.nup[a]; }
    }
#pragma unroll
    for (int j = 0; j < NPO; ++j) {
      const int i = lane + 32 * j;
      po[j] = (i < 8 * kPPW && b + (i >> 3) < sB) ? OM[(b + (i >> 3) - sA) * 8 + (i & 7)] : 0.0;
    }
  };
  int64_t base = sA + ((int64_t)blockIdx.x * WPB + warp) * kPPW;
  if (base < sB) prefetch(base);
  for (; base < sB; base += stride) {
    if (lane < kPPW) {
      TgtPair<P> &ps = mine[lane];
      const bool active = base + lane < sB;
      ps.active = active;
      if (active) {
        ps.aslot = pa;
        for (int a = 0; a < 3; ++a) { ps.rp[a] = pv[a]; ps.nup[a] = pv[3 + a]; }
      }
    }
#pragma unroll
    for (int j = 0; j < NPO; ++j) {
      const int i = lane + 32 * j;
      if (i < 8 * kPPW) mine[i >> 3].om[i & 7] = po[j];
    }
    if (base + stride < sB) prefetch(base + stride);
    __syncwarp();
    if constexpr (kPPW * (P + 1) <= 32) {
      // lane = (pair, column m): R_l^m of its column in registers (the r_column recurrence), the
      // neighbour columns m +- 1 by shuffles for grad S^{(l,m)} (grad_fast's rules), then straight away the
      // translation operands S', NG' of (l, +-m) (XRow) and the R / grad tables the gamma step reads
      const int pp = lane / (P + 1) < kPPW ? lane / (P + 1) : kPPW - 1, m = lane % (P + 1);
      const bool in = lane < kPPW * (P + 1);
      TgtPair<P> &ps = mine[pp];
      const bool act = in && ps.active;
      const double X = ps.rp[1], Y = ps.rp[2], Z = ps.rp[0], r2 = X * X + Y * Y + Z * Z;
      cd rmm = mk(1.0, 0.0);
      for (int k = 1; k <= m; ++k) rmm = shc[HC_DG + k] * (mk(X, Y) * rmm);
      cd Rc[P + 1];
#pragma unroll
      for (int l = 0; l <= P; ++l) {
        cd v = mk(0.0, 0.0);
        if (l == m) v = rmm;
        else if (l == m + 1) v = shc[HC_SB + m] * Z * rmm;
        else if (l > m + 1)
          v = (shc[HC_RA + sidx(l - 1, m)] * Z) * Rc[l - 1] - (shc[HC_RB + sidx(l - 1, m)] * r2) * Rc[l - 2];
        Rc[l] = act ? v : mk(0.0, 0.0);
        if (act && l >= m) ps.R[sidx(l, m)] = Rc[l];
      }
      const double nup[3] = {ps.nup[0], ps.nup[1], ps.nup[2]};
      double2 *xo = reinterpret_cast<double2 *>(Xrow + (base + pp - sA) * XR::STRIDE + XR::SX);
      const bool last = m == P;
#pragma unroll
      for (int l = 0; l <= P; ++l) {
        cd g[3] = {mk(0.0, 0.0), mk(0.0, 0.0), mk(0.0, 0.0)};
        if (l >= 1) {
          const cd r0 = Rc[l - 1];
          cd rp = mk(__shfl_down_sync(0xffffffffu, r0.x, 1), __shfl_down_sync(0xffffffffu, r0.y, 1));
          cd rm = mk(__shfl_up_sync(0xffffffffu, r0.x, 1), __shfl_up_sync(0xffffffffu, r0.y, 1));
          if (last) rp = mk(0.0, 0.0);               // R^{m+1} with m + 1 > l - 1
          if (m == 0) rm = mk(-rp.x, rp.y);          // R_{l-1}^{-1} = -conj R_{l-1}^{1}
          const double *dc = shc + HC_DC + 3 * (l * l + l + m);
          g[0] = dc[0] * r0;
          g[1] = 0.5 * (dc[2] * rm - dc[1] * rp);
          const cd t = 0.5 * (dc[1] * rp + dc[2] * rm);
          g[2] = mk(-t.y, t.x);
        }
        if (!act || l < m) continue;
        cd *gs = GS[pp][sidx(l, m)];
        gs[0] = g[0]; gs[1] = g[1]; gs[2] = g[2];
        if (l < P) {   // translation operands, l' < p
          const cd ng = nup[0] * g[0] + nup[1] * g[1] + nup[2] * g[2], r = Rc[l];
          const double w = wS[l * l + l + m];
          double *o = reinterpret_cast<double *>(xo + 2 * (l * l + l + m));
          st_global_256(o, w * r.y, w * r.x, w * ng.y, w * ng.x);   // a whole 32-B entry per store
          if (m > 0) {   // S^{(l,-m)} = (-1)^m conj S^{(l,m)}, same for nu'.grad S
            const double sg = (m & 1) ? -w : w;
            st_global_256(o - 8 * m, -sg * r.y, sg * r.x, -sg * ng.y, sg * ng.x);
          }
        }
      }
    } else {
      // solid harmonics of the warp's pairs: lanes (pair, column m)
      for (int i = lane; i < kPPW * (P + 1); i += 32) {
        TgtPair<P> &ps = mine[i / (P + 1)];
        if (ps.active) r_column<P>(ps.rp[1], ps.rp[2], ps.rp[0], i % (P + 1), ps.R, shc);
      }
      __syncwarp();
      // gradient tables (kept for the gamma step), then the translation operands S', NG' (XRow): flat over pairs
      for (int i = lane; i < kPPW * NS; i += 32) {
        const int pp = i / NS, e = i % NS;
        if (!mine[pp].active) continue;
        const int l = tri_inv(e);   // sidx(l, 0) <= e < sidx(l + 1, 0)
        grad_fast(mine[pp].R, l, e - sidx(l, 0), shc, GS[pp][e]);
      }
      __syncwarp();
      constexpr int NSX = sidx(P, 0);   // l' < p
      for (int i = lane; i < kPPW * NSX; i += 32) {
        const int pp = i / NSX, e = i % NSX;
        TgtPair<P> &ps = mine[pp];
        if (!ps.active) continue;
        const int l = tri_inv(e);   // sidx(l, 0) <= e < sidx(l + 1, 0)
        const int m = e - sidx(l, 0);
        const cd *g = GS[pp][e];
        const cd ng = ps.nup[0] * g[0] + ps.nup[1] * g[1] + ps.nup[2] * g[2], r = ps.R[e];
        const double w = wS[l * l + l + m];
        double *o = Xrow + (base + pp - sA) * XR::STRIDE + XR::SX + 4 * (l * l + l + m);
        st_global_256(o, w * r.y, w * r.x, w * ng.y, w * ng.x);   // a whole 32-B entry per store
        if (m > 0) {   // S^{(l,-m)} = (-1)^m conj S^{(l,m)}, same for nu'.grad S
          const double sg = (m & 1) ? -w : w;
          st_global_256(o - 8 * m, -sg * r.y, sg * r.x, -sg * ng.y, sg * ng.x);
        }
      }
    }
    if (lane < 3 * kPPW && mine[lane / 3].active)
      Xrow[(base + lane / 3 - sA) * XR::STRIDE + XR::NU + lane % 3] = mine[lane / 3].nup[lane % 3];
    if (lane < kPPW && mine[lane].active)   // k_contract tile slot (k_translate writes zeta there)
      Xrow[(base + lane - sA) * XR::STRIDE + XR::NU + 3] = __longlong_as_double(mine[lane].aslot);
    __syncwarp();
    // ---------------- I[gamma]: (Omega_0, Omega)(0, grad S(r')), omega first; its nu'-derivative with
    // Hess S nu'; W_gamma = -sqrt2 Im I[gamma]; the S(r') Omega_0 part of Theta
    for (int i = lane; i < kPPW * NP; i += 32) {
      const int pp = i / NP, c = i % NP;
      TgtPair<P> &ps = mine[pp];
      if (!ps.active) continue;
      double *X = Xrow + (base + pp - sA) * XR::STRIDE;
      const double nup[3] = {ps.nup[0], ps.nup[1], ps.nup[2]};
      const double O0 = ps.om[0], Ov[3] = {ps.om[1], ps.om[2], ps.om[3]}, dO0 = ps.om[4],
                   dOv[3] = {ps.om[5], ps.om[6], ps.om[7]};
      const int l = tri_inv(c) + 1;   // lmidx(l, 1) <= c < lmidx(l + 1, 1)
      const int m = c - lmidx(l, 1) + 1, hs = sidx(l, m);
      const cd *g = GS[pp][hs];
      cd hn[3] = {mk(0.0, 0.0), mk(0.0, 0.0), mk(0.0, 0.0)};
      if (want_dp) hess_fast(GS[pp], l, m, nup, shc, hn);
      double gs = 0, dgs = 0, gv[3], dgv[3];
      for (int a = 0; a < 3; ++a) {
        gs -= Ov[a] * g[a].y;
        dgs -= dOv[a] * g[a].y + Ov[a] * hn[a].y;
        const int b1 = (a + 1) % 3, b2 = (a + 2) % 3;
        gv[a] = O0 * g[a].y + (Ov[b1] * g[b2].y - Ov[b2] * g[b1].y);
        dgv[a] = dO0 * g[a].y + (dOv[b1] * g[b2].y - dOv[b2] * g[b1].y) + O0 * hn[a].y +
                 (Ov[b1] * hn[b2].y - Ov[b2] * hn[b1].y);
      }
      const double f = -s2 * inv4pi;
      X[XR::W + c] = f * gs;
      if (want_dp) X[XR::DW + c] = f * dgs;
      for (int a = 0; a < 3; ++a) {
        X[XR::W + (1 + a) * NP + c] = f * gv[a];
        if (want_dp) X[XR::DW + (1 + a) * NP + c] = f * dgv[a];
      }
      X[XR::TH + c] = s2 * inv4pi * ps.R[hs].y * O0;
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------------------------
// k_qmap: line-integral maps (Step 6) as a DMMA GEMM per tile of TP pairs
// of one patch: rows [a(pairs) ; b(pairs)] x M (k_edge_tables).  K runs axis-major (k = axis E + kappa) and
// the Q columns component-major, so the structurally zero blocks of M (axis c-1 of vector component c, the
// cross product) are skipped whole.  Warp = (pair group of 8, column split); the a- and b-row tiles share
// every Q-column B fragment (2 DMMA per load), the V columns need the a rows only.  A staged in shared
// memory by cp.async (row stride == 4 mod 16 doubles), M streamed in KC-row chunks (double buffered,
// row stride == 8 mod 16).  Two CTAs per SM so one's staging / stores overlap the other's DMMA loop.
// The epilogue scales by v_lambda / v_theta (TrCfg) and stores the QRow layout for k_translate.
// ------------------------------------------------------------------------------------------------

// One KC-row chunk of column pass H of the k_qmap GEMM for a warp of column split NS; ZC = the quaternion
// component whose M block is zero in this chunk's axis, -1 if none of the pass's (compile time, so the
// skipped tiles cost nothing).
// Tiles: local component cl (component 2H + cl), u-th of the warp: column tile cl TQC + NS + NSPLIT u of the
// pass's block; V (pass 1): 2 TQC + vstart(NS) + u.  The B fragments of a k-step are loaded before its DMMAs.
template <int P, int ZC, int NS, bool DP, int H>
__device__ __forceinline__ void qmap_chunk(const double *arow, const double *brow, int sw, const double *bb,
                                           double (&accA)[2][QmapCfg<P>::UQ][2], double (&accB)[2][QmapCfg<P>::UQ][2],
                                           double (&accV)[QmapCfg<P>::UV][2]) {
  using C = QmapCfg<P>;
  constexpr int NCSH = H ? Dims<P>::NCSH1 : Dims<P>::NCSH0, NQT = C::nq(NS), NVT = H ? C::vcount(NS) : 0,
                V0 = C::vstart(NS);
#pragma unroll
  for (int kk = 0; kk < C::KC; kk += 4) {
    const double a = arow[kk ^ sw], b = DP ? brow[kk ^ sw] : 0.0;
    const double *bk = bb + kk * NCSH;
    double bq[2][C::UQ], bv[C::UV > 0 ? C::UV : 1];
#pragma unroll
    for (int cl = 0; cl < 2; ++cl)
#pragma unroll
      for (int u = 0; u < NQT; ++u) bq[cl][u] = (2 * H + cl == ZC) ? 0.0 : bk[(cl * C::TQC + NS + u * C::NSPLIT) * 8];
#pragma unroll
    for (int u = 0; u < NVT; ++u) bv[u] = bk[(2 * C::TQC + V0 + u) * 8];
#pragma unroll
    for (int cl = 0; cl < 2; ++cl) {
      if (2 * H + cl == ZC) continue;
#pragma unroll
      for (int u = 0; u < NQT; ++u) {
        dmma(accA[cl][u][0], accA[cl][u][1], a, bq[cl][u]);
        if constexpr (DP) dmma(accB[cl][u][0], accB[cl][u][1], b, bq[cl][u]);   // dQ rows only when D' is built
      }
    }
#pragma unroll
    for (int u = 0; u < NVT; ++u) dmma(accV[u][0], accV[u][1], a, bv[u]);
  }
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// 1-D bulk copies (TMA engine) completing on an mbarrier.
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// DP = false (kernel mask without D'): the b rows (dQ) are neither copied, multiplied nor stored.
template <int P, bool DP>
__global__ void __launch_bounds__(QmapCfg<P>::WARPS * 32, QmapCfg<P>::MINB)
    k_qmap(int64_t item0, int64_t item1, const int64_t *__restrict__ item_ptr, const int32_t *__restrict__ item_patch,
           const int64_t *__restrict__ seg_ptr, int64_t sA, const double *__restrict__ fit,
           const double *__restrict__ Arow, double *__restrict__ Qrow, const double *__restrict__ trtab) {
  using D = Dims<P>;
  using L = Layout<P>;
  using C = QmapCfg<P>;
  using QR = QRow<P>;
  constexpr int TP = C::TP, KC = C::KC, NCH = C::NCH;
  extern __shared__ __align__(16) double sst[];   // [NST][A chunk | B chunk]
  const int64_t item = item0 + blockIdx.x;
  if (item >= item1) return;
  const int64_t Pp = item_patch[item];
  const int64_t s0 = seg_ptr[Pp] + (item - item_ptr[Pp]) * TP;
  const int cnt = (int)min((int64_t)TP, seg_ptr[Pp + 1] - s0);
  const double *M0 = fit + Pp * (int64_t)L::STRIDE + L::MQ, *M1 = fit + Pp * (int64_t)L::STRIDE + L::MQ1;
  const double *Ablk = Arow + (item - item0) * (int64_t)C::ABLK;   // rows of absent pairs: never read back
  // pipeline over 2 NCH virtual chunks (pass h = vc / NCH, K chunk vc % NCH): bar[b] = "stage b landed"
  // (bulk-copy transactions), emp[b] = "all warps done with stage b" (one arrival per warp); no CTA-wide
  // barrier inside the K loop, and the pass-1 chunks stream in during the pass-0 epilogue
  __shared__ uint64_t bar[C::NST], emp[C::NST];
  // a chunk's a rows (0..TP-1) come first: without D' only that half is copied
  constexpr unsigned ACHB = (unsigned)(C::ACH * sizeof(double)) / (DP ? 1 : 2);
  constexpr unsigned CHB0 = (unsigned)(KC * D::NCSH0 * sizeof(double)), CHB1 = (unsigned)(KC * D::NCSH1 * sizeof(double));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NST; ++i) {
      mbar_init(&bar[i], 1);
      mbar_init(&emp[i], C::WARPS);
    }
    mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](int vc) {   // thread 0
    const int b = vc % C::NST, h = vc / NCH, ch = vc % NCH;
    double *st = sst + b * C::STG;
    mbar_expect_tx(&bar[b], ACHB + (h ? CHB1 : CHB0));
    bulk_g2s(st, Ablk + (int64_t)ch * C::ACH, ACHB, &bar[b]);
    if (h) bulk_g2s(st + C::ACH, M1 + (int64_t)ch * KC * D::NCSH1, CHB1, &bar[b]);
    else bulk_g2s(st + C::ACH, M0 + (int64_t)ch * KC * D::NCSH0, CHB0, &bar[b]);
  };
  if (threadIdx.x == 0)   // chunks 0 .. NST-2 in flight from the start
    for (int vc = 0; vc < C::NST - 1; ++vc) issue(vc);
  const int ns = warp / C::PG, pg = warp % C::PG;
  double accA[2][C::UQ][2], accB[2][C::UQ][2], accV[C::UV][2];
  const int ar = pg * 8 + (lane >> 2), sw = C::swz(ar);
  const int aofs = ar * KC + (lane & 3);
  const int pr = pg * 8 + (lane >> 2);
  double *out = Qrow + (s0 + pr - sA) * QR::STRIDE;
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int u = 0; u < C::UQ; ++u) accA[c][u][0] = accA[c][u][1] = accB[c][u][0] = accB[c][u][1] = 0.0;
#pragma unroll
    for (int u = 0; u < C::UV; ++u) accV[u][0] = accV[u][1] = 0.0;
    const int bofs = C::ACH + (lane & 3) * (h ? D::NCSH1 : D::NCSH0) + (lane >> 2);
    for (int ch = 0; ch < NCH; ++ch) {
      const int vc = h * NCH + ch;
      const int nx = vc + C::NST - 1;   // chunk to issue now, into the stage chunk vc-1 used
      if (threadIdx.x == 0 && nx < 2 * NCH) {
        if (vc >= 1) mbar_wait(&emp[nx % C::NST], ((vc - 1) / C::NST) & 1);
        fence_proxy_async();
        issue(nx);
      }
      mbar_wait(&bar[vc % C::NST], (vc / C::NST) & 1);
      const double *stg = sst + (vc % C::NST) * C::STG;
      const double *arow = stg + aofs, *brow = arow + TP * KC, *bb = stg + bofs;
      const int zc = 1 + ch / C::CPA;   // axis of this chunk: component axis + 1 has a zero block
#define RRQ_QCHUNK(Z, N, HH) qmap_chunk<P, Z, N, DP, HH>(arow, brow, sw, bb, accA, accB, accV)
      // ZC = -1: no zero block among the pass's two components in this chunk's axis
#define RRQ_QNS(N) (h == 0 ? (zc == 1 ? RRQ_QCHUNK(1, N, 0) : RRQ_QCHUNK(-1, N, 0)) \
                           : (zc == 2 ? RRQ_QCHUNK(2, N, 1) : zc == 3 ? RRQ_QCHUNK(3, N, 1) : RRQ_QCHUNK(-1, N, 1)))
      switch (ns) {
        case 0: RRQ_QNS(0); break;
        case 1: RRQ_QNS(1); break;
        case 2: RRQ_QNS(2); break;
        default: RRQ_QNS(3); break;
      }
#undef RRQ_QNS
#undef RRQ_QCHUNK
      __syncwarp();
      if (lane == 0) mbar_arrive(&emp[vc % C::NST]);
    }
    // store: C[row = lane/4][col = 2 (lane%4) + {0,1}]; a lane owns the pass's two components of Q (and dQ)
    // of entry e: two 32-B sectors (rows are 128-B aligned).  M's columns carry v_lambda / v_theta.
    if (pr < cnt) {
#pragma unroll
      for (int u = 0; u < C::UQ; ++u) {
        const int tl = ns + u * C::NSPLIT;
        if (tl >= C::TQC) continue;   // == u < nq(ns)
        const int e = tl * 4 + (lane & 3);   // entry qidx(j,k)
        if (e >= D::NQ) continue;
        // the pass's two components of Q (and of dQ) of the entry are 32 contiguous bytes each: one STG.256
        double *o = out + QR::EG * e + 4 * h;
        st_global_256(o, accA[0][u][0], accA[0][u][1], accA[1][u][0], accA[1][u][1]);
        if constexpr (DP) st_global_256(o + 8, accB[0][u][0], accB[0][u][1], accB[1][u][0], accB[1][u][1]);
      }
      if (h == 1) {
        const int v0 = ns == 0 ? C::vstart(0) : ns == 1 ? C::vstart(1) : ns == 2 ? C::vstart(2) : C::vstart(3);
        const int nv = ns == 0 ? C::vcount(0) : ns == 1 ? C::vcount(1) : ns == 2 ? C::vcount(2) : C::vcount(3);
#pragma unroll
        for (int u = 0; u < C::UV; ++u) {
          if (u >= nv) continue;
          const int col = (v0 + u) * 8 + 2 * (lane & 3);
          if (col < 2 * D::NV) *reinterpret_cast<double2 *>(out + QR::V + col) = make_double2(accV[u][0], accV[u][1]);
        }
      }
    }
  }
}

// k_contract's tile configuration (see k_contract); k_translate writes zeta in its tile-chunked layout.
template <int P>
struct ContractCfg {
  using D = Dims<P>;
  static constexpr int TP = 16, MT = TP / 8, NT = (D::N + 7) / 8;
  // warps per CTA (even: a warp's tiles share one M-tile) chosen so the MT x NT output tiles divide evenly:
  // p = 6: 10 tiles on 10 warps, p = 8: 16 on 8, p = 10: 26 on 14 (2 each), p = 12: 36 on 12, p = 14: 50 on 10
  static constexpr int WARPS = P == 4 ? 4 : P == 6 ? 10 : P == 8 ? 8 : P == 10 ? 14 : P == 12 ? 12 : 10;
  static constexpr int TILES = MT * NT, TPW = (TILES + WARPS - 1) / WARPS;
  static constexpr int NB = Layout<P>::NF;   // B row stride (== the fit operators' row stride)
  // k-rows per chunk: 16 where it divides 4 NP (a Z chunk row is then one 128-B line), else 12 or 8; where none
  // divides (p = 10: 4 NP = 220) 16 with a zero-padded last chunk: its Z entries beyond 4 NP are never written
  // (the Z buffer is zeroed when allocated) and multiply the rows that follow the operator in the fit block
  static constexpr int K4 = 4 * D::NP;
  static constexpr int KC = (K4 % 16 == 0) ? 16 : (K4 % 12 == 0) ? 12 : ((K4 % 8 == 0) ? 8 : 16);
  static constexpr int NCH = (K4 + KC - 1) / KC;
  static constexpr bool KPAD = K4 % KC != 0;
  // Z is stored tile-chunked by k_translate (a tile's block of ZBLK doubles): the Theta part [TP][ZTS]
  // (ZTS == 4 mod 16: conflict-free A fragments), then per K chunk ch the W | dW | S slices [3][TP][KC]
  // (k = component NP + c of zeta(W), zeta(dW), zeta_S).  A pipeline stage = [B chunk | Z chunk], two
  // bulk copies; the small footprint lets 3 CTAs share an SM.  Rows are XOR-swizzled in 4-column groups
  // (KC = 16: by r mod 4; KC = 8: by bit 1 of r) so a half-warp's A fragments hit distinct banks.
  static constexpr int ZTS = D::NP + ((4 - D::NP % 16) + 16) % 16, ZT = TP * ZTS, ZCH = 3 * TP * KC;
  static constexpr int64_t ZBLK = (int64_t)ZT + (int64_t)NCH * ZCH;
  static constexpr size_t SMEM_B = 3 * (size_t)KC * NB;                                       // PD | PSp | PSg
  static constexpr size_t STG = SMEM_B + ZCH;
  static constexpr size_t SNODE = (7 * D::N + 1) / 2 * 2;   // the patch's nodes [N][3], normals [N][3], weights [N]
  static constexpr size_t SMEM = (ZT + 2 * STG + SNODE) * sizeof(double) + TP * 64;   // + ContractPair[TP]
  static constexpr int MINB = (P <= 8 && SMEM * 3 <= 225 * 1024) ? 3 : (P <= 10 ? 2 : 1);   // p = 10: registers (TPW = 4)
  // p <= 10: the P_Sd fragments of Theta . P_Sd are loaded into registers before the Z tile lands; p >= 12:
  // TPW x NK would not fit the register file, so they are read as they are used
  static constexpr bool BQREG = P <= 10;
  __host__ __device__ static constexpr int swz(int r) { return KC == 16 ? (r & 3) << 2 : KC == 8 ? ((r >> 1) & 1) << 2 : 0; }
  // position of zeta entry (block b = 0 Theta, 1..4 zeta(W), 5..8 zeta(dW), 9..12 zeta_S; c = (l,m)) of tile row r
  __host__ __device__ static constexpr int64_t zoff(int b, int r, int c) {
    return b == 0 ? (int64_t)r * ZTS + c
                  : (int64_t)ZT + (int64_t)((((b - 1) & 3) * D::NP + c) / KC) * ZCH + (int64_t)((b - 1) >> 2) * TP * KC +
                        r * KC + (((((b - 1) & 3) * D::NP + c) % KC) ^ swz(r));
  }
};

// ------------------------------------------------------------------------------------------------
// k_translate: Step 7 (P:L1263-1268 eq cdlp1dintegral): for each (l,m),
// lambda_1, its nu'-derivative and theta_1 from Q^{(j,k)}, dQ^{(j,k)}, V^{(j,k)} and S(r'), plus the
// gamma parts from k_target_gamma -> W, dW, Theta -> zeta = (Theta, zeta(W), zeta(dW), zeta_S).
//
// The translation is a 2-D convolution  out(l,m) = sum_{j,k} c(l,m,j,k) A^{(j,k)} S^{(l-j,m-k)}  whose
// coefficient factors as u(l,m) v(j,k) w(l-j,m-k) (T = F(l,m)/(F(j,k) F(l',m')), F(a,b) = sqrt((a+b)!(a-b)!),
// and the factorial ratios of C_j, D_j split the same way).  k_qmap stores A = v A and k_target_gamma stores
// S' = w S (expanded over m' < 0), so the inner loop is pure FMAs on the Im parts (only Im(lambda),
// Im(theta) enter W, dW, Theta): Im(A S) = A.x S.y + A.y S.x, with A^{(j,-k)} = (-1)^k conj A^{(j,k)} folded
// into sign flips of (A.x, A.y).
// One warp per pair; shared memory bandwidth is the bound, so every operand is loaded once per use by
// as many outputs as possible: a lane works on one block of WD outputs (l, m0 .. m0+WD-1) (TrCfg) and
// sweeps k for each j, loading per step one Q / dQ / V entry (used by all WD outputs) and ONE new S'
// entry (the S' window of the WD outputs slides by one entry per step, in registers).  A block's steps
// are split into contiguous pieces over several lanes so that every lane runs the same STEPS steps
// (host-built codes, make_trtab in rrq_api.cu); a piece starts by loading the whole window (PRIME), a new
// j starts from an all-zero window (RESET; PRIME where the sweep is clipped at k = -j).  Each lane
// writes its WD partial outputs to its slot once, after the sweep; the epilogue (lanes over c) sums the
// slots of a c's block, adds the j = 1 theta terms and the gamma parts and writes zeta.  Rows are
// prefetched with cp.async one pair ahead.
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ double flip_if(double x, uint32_t bit) {
  return __longlong_as_double(__double_as_longlong(x) ^ ((unsigned long long)bit << 63));
}

// DP = false (kernel mask without D'): no dQ staging, no dlambda accumulation, no zeta(dW); mask: Theta is
// written only with S, zeta_S only with S'.
template <int P, bool DP>
__global__ void __launch_bounds__(TrCfg<P>::WPB * 32, 1)
    k_translate(int64_t sA, int64_t sB, const double *__restrict__ Xrow, const double *__restrict__ Qrow,
                const double *__restrict__ trtab, double *__restrict__ Zrow, uint32_t mask) {
  using D = Dims<P>;
  using C = TrCfg<P>;
  using XR = XRow<P>;
  using QR = QRow<P>;
  constexpr int NP = D::NP, WPB = C::WPB, EQ = C::EQ, SXW = C::SXW, WD = C::WD;
  extern __shared__ __align__(16) double sm[];
  for (int i = threadIdx.x; i < C::TAB_D; i += blockDim.x) sm[i] = trtab[i];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double *wb = sm + C::TAB_D + (size_t)warp * C::PER_WARP;
  double *GB = wb + C::NBUF * C::BUF;   // buffer b: wb + b BUF = [Q block | S' block]
  auto zero_entries = [&](int b) {  // the zero Q entry (+ its V) and the zero S' entry (never staged)
    double *qd = wb + b * C::BUF;
    if (lane < 16) qd[EQ * C::ZQ + lane] = 0.0;
    else if (lane < 18) qd[C::SV + 2 * (C::ZQ + 2) + lane - 16] = 0.0;
    else if (lane < 22) qd[C::QSZ + SXW * P * P + lane - 18] = 0.0;
  };
  for (int b = 0; b < C::NBUF; ++b) zero_entries(b);
  __syncthreads();
  const uint32_t *code = reinterpret_cast<const uint32_t *>(sm);
  const uint32_t *pcode = code + C::STEPS * 32;
  const uint32_t *cinfo = pcode + C::STEPS * 32;
  const uint8_t *posq = reinterpret_cast<const uint8_t *>(cinfo + NP), *poss = posq + D::NQ;
  const double *olam = sm + C::OLAM, *oth = sm + C::OTH;
  const int64_t stride = (int64_t)gridDim.x * WPB;

  // Q row (entry e -> position posq[e] at stride EQ; V of (j >= 2, k) next to it) and the S'/NG' block
  // (entry e -> position poss[e] at stride SXW): positions chosen by the host to spread the main loop's
  // shared-memory banks.  Destinations of this lane's 16-B chunks, fixed for every pair (registers).
  // 16-B chunks per Q entry staged: Q | dQ (8), or Q only (4) without D'
  constexpr int CPE = DP ? 8 : 4, LCPE = DP ? 3 : 2;
  constexpr int NCQ_ = CPE * D::NQ, NLQ = (NCQ_ + 31) / 32, NLV = (D::NV + 31) / 32, NLS = (2 * P * P + 31) / 32;
  int dq[NLQ], dv[NLV], ds[NLS];
#pragma unroll
  for (int u = 0; u < NLQ; ++u) {
    const int i = lane + 32 * u;
    dq[u] = i < NCQ_ ? EQ * posq[i >> LCPE] + 2 * (i & (CPE - 1)) : 0;
  }
#pragma unroll
  for (int u = 0; u < NLV; ++u) {
    const int i = lane + 32 * u;
    dv[u] = i < D::NV ? C::SV + 2 * (i < 2 ? i : posq[i - 2] + 2) : 0;
  }
#pragma unroll
  for (int u = 0; u < NLS; ++u) {
    const int i = lane + 32 * u;
    ds[u] = i < 2 * P * P ? C::QSZ + SXW * poss[i >> 1] + 2 * (i & 1) : 0;
  }
  auto issue_qs = [&](int64_t s, int b) {
    const double *qg = Qrow + (s - sA) * QR::STRIDE, *xg = Xrow + (s - sA) * XR::STRIDE + XR::SX;
    double *qd = wb + b * C::BUF;
#pragma unroll
    for (int u = 0; u < NLQ; ++u) {
      const int i = lane + 32 * u;
      if (i < NCQ_) cp_async16(qd + dq[u], qg + 2 * (DP ? i : ((i >> 2) << 3 | (i & 3))));
    }
#pragma unroll
    for (int u = 0; u < NLV; ++u)
      if (lane + 32 * u < D::NV) cp_async16(qd + dv[u], qg + QR::V + 2 * (lane + 32 * u));
#pragma unroll
    for (int u = 0; u < NLS; ++u)
      if (lane + 32 * u < 2 * P * P) cp_async16(qd + ds[u], xg + 2 * (lane + 32 * u));
  };
  auto issue_g = [&](int64_t s) {
    const double *xg = Xrow + (s - sA) * XR::STRIDE + XR::G;
    for (int i = lane; i < C::GSZ / 2; i += 32) cp_async16(GB + 2 * i, xg + 2 * i);
  };

  const double inv4pi = 1.0 / (4.0 * kPi), s2 = 1.4142135623730950488;
  int64_t s = sA + (int64_t)blockIdx.x * WPB + warp;
  if (s < sB) {
    issue_qs(s, 0);
    issue_g(s);
  }
  cp_async_commit();
  for (int it = 0; s < sB; s += stride, ++it) {
    const int cb = C::NBUF == 2 ? (it & 1) : 0;
    if constexpr (C::NBUF == 2) {
      if (s + stride < sB) issue_qs(s + stride, cb ^ 1);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    double *qbw = wb + cb * C::BUF;
    const double *qb = qbw, *sx = qbw + C::QSZ;
    // main loop: a ring of WD S' entries (S'.y, S'.x, NG'.y, NG'.x); the entry loaded at step t sits in
    // ring slot t mod WD, and output m0 + i at step t uses the one loaded at step t - i (static indices in
    // the unrolled loop: no register moves)
    double th[WD], lam[WD][4], dl[WD][4];
    double2 ws[WD], wg[WD];
#pragma unroll
    for (int i = 0; i < WD; ++i) {
      th[i] = 0;
      ws[i] = wg[i] = make_double2(0.0, 0.0);
#pragma unroll
      for (int b = 0; b < 4; ++b) lam[i][b] = dl[i][b] = 0;
    }
#pragma unroll
    for (int t = 0; t < C::STEPS; ++t) {
      const uint32_t cw = code[t * 32 + lane];
      const int qe = cw & 127, se = (cw >> 7) & C::SEM;
      ws[t % WD] = *reinterpret_cast<const double2 *>(sx + SXW * se);
      wg[t % WD] = *reinterpret_cast<const double2 *>(sx + SXW * se + 2);
      if (t == 0 || (cw & C::PRIME)) {   // every piece and every sweep starts with a PRIME
        const uint32_t pw = pcode[t * 32 + lane];
#pragma unroll
        for (int i = 1; i < WD; ++i) {
          const int pe = (pw >> (C::SEB * (i - 1))) & C::SEM;
          ws[(t - i + WD * C::STEPS) % WD] = *reinterpret_cast<const double2 *>(sx + SXW * pe);
          wg[(t - i + WD * C::STEPS) % WD] = *reinterpret_cast<const double2 *>(sx + SXW * pe + 2);
        }
      }
      const double *e = qb + EQ * qe;
      double2 q[4], dq[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        q[b] = *reinterpret_cast<const double2 *>(e + 2 * b);
        dq[b] = DP ? *reinterpret_cast<const double2 *>(e + 8 + 2 * b) : make_double2(0.0, 0.0);
      }
      double2 v = *reinterpret_cast<const double2 *>(qb + C::SV + 2 * (qe + 2));
      // k < 0: A^{(j,-k)} = (-1)^k conj A^{(j,k)}, so Im(A S) = A.x S.y + A.y S.x takes -A.x (odd k, FA) or
      // -A.y (even k, FB): flipped in place on this step's Q operands (used by all WD outputs)
      const uint32_t fa = (cw & C::FA) ? 1u : 0u, fb = (cw & C::FB) ? 1u : 0u;
      v.x = flip_if(v.x, fa);
      v.y = flip_if(v.y, fb);
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        q[b].x = flip_if(q[b].x, fa);
        q[b].y = flip_if(q[b].y, fb);
        dq[b].x = flip_if(dq[b].x, fa);
        dq[b].y = flip_if(dq[b].y, fb);
      }
#pragma unroll
      for (int i = 0; i < WD; ++i) {
        const int r = (t - i + WD * C::STEPS) % WD;
        const double A = ws[r].x, B = ws[r].y, An = wg[r].x, Bn = wg[r].y;
        th[i] = fma(v.x, A, fma(v.y, B, th[i]));
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          lam[i][b] = fma(q[b].x, A, fma(q[b].y, B, lam[i][b]));
          if constexpr (DP) dl[i][b] = fma(dq[b].x, A, fma(dq[b].y, B, fma(q[b].x, An, fma(q[b].y, Bn, dl[i][b]))));
        }
      }
    }
    // j = 1 theta terms of this lane's outputs c = lane, lane + 32, ... (no lambda part: C_1 = 0; |m - k| > l - 1
    // reads the zero S' entry), taken before the slots overwrite the buffer
    constexpr int NH = (NP + 31) / 32;   // outputs per lane
    double T1[NH];
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      T1[h] = 0;
      const int c = lane + 32 * h;
      if (c >= NP) continue;
      const uint32_t ci = cinfo[c];
      const int l = ci & 15, m = (ci >> 4) & 15;
#pragma unroll
      for (int k = -1; k <= 1; ++k) {
        const int lp = l - 1, mp = m - k;
        const int se = (mp >= -lp && mp <= lp) ? poss[lp * lp + lp + mp] : P * P;
        const double *vv = qb + C::SV + 2 * vidx(1, k < 0 ? -k : k);
        const double A = k < 0 ? -sx[SXW * se] : sx[SXW * se], B = sx[SXW * se + 1];
        T1[h] = fma(vv[0], A, fma(vv[1], B, T1[h]));
      }
    }
    __syncwarp();
    {   // this lane's slot (in the current buffer): WD x (theta, lambda[4], dlambda[4], pad)
      double2 *d = reinterpret_cast<double2 *>(qbw + C::SLW * lane);
#pragma unroll
      for (int i = 0; i < WD; ++i) {
        d[5 * i] = make_double2(th[i], lam[i][0]);
        d[5 * i + 1] = make_double2(lam[i][1], lam[i][2]);
        d[5 * i + 2] = make_double2(lam[i][3], dl[i][0]);
        d[5 * i + 3] = make_double2(dl[i][1], dl[i][2]);
        d[5 * i + 4] = make_double2(dl[i][3], 0.0);
      }
    }
    __syncwarp();
    // epilogue: lanes over c = (l, m); gamma parts from GB (W [4][NP], dW [4][NP], Theta [NP], nu')
    const double nup[3] = {GB[9 * NP], GB[9 * NP + 1], GB[9 * NP + 2]};
    using CC = ContractCfg<P>;   // Z in k_contract's tile-chunked layout; the tile slot rides in the G block
    const int64_t aslot = __double_as_longlong(GB[9 * NP + 3]);
    double *Zt = Zrow + (aslot >> 5) * CC::ZBLK;
    const int zr = (int)(aslot & 31);
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      const int c = lane + 32 * h;
      if (c >= NP) continue;
      const uint32_t ci = cinfo[c];
      const int ib = (ci >> 8) & 15, fl = (ci >> 12) & 255, nl = (ci >> 20) & 63;
      double T = T1[h], L[4] = {0, 0, 0, 0}, DL[4] = {0, 0, 0, 0};
      for (int q = 0; q < nl; ++q) {
        const double2 *d = reinterpret_cast<const double2 *>(qbw + C::SLW * (fl + q) + 10 * ib);
        const double2 d0 = d[0], d1 = d[1], d2 = d[2], d3 = d[3], d4 = d[4];
        T += d0.x;
        L[0] += d0.y; L[1] += d1.x; L[2] += d1.y; L[3] += d2.x;
        DL[0] += d2.y; DL[1] += d3.x; DL[2] += d3.y; DL[3] += d4.x;
      }
      const double fo = -s2 * inv4pi * olam[c];
      double W[4], dW[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        W[a] = fo * L[a] + GB[a * NP + c];
        dW[a] = fo * DL[a] + GB[4 * NP + a * NP + c];
      }
      const double Th = s2 * inv4pi * oth[c] * T + GB[8 * NP + c];
      // zeta vectors (Step 8, App. A.7; reading G3 for S')
      double nxW[3];
      cross3(nup, W + 1, nxW);
      if (mask & 1) Zt[CC::zoff(0, zr, c)] = Th;
      Zt[CC::zoff(1, zr, c)] = W[0];
      Zt[CC::zoff(2, zr, c)] = -W[1];
      Zt[CC::zoff(3, zr, c)] = -W[2];
      Zt[CC::zoff(4, zr, c)] = -W[3];
      if constexpr (DP) {
        Zt[CC::zoff(5, zr, c)] = dW[0];
        Zt[CC::zoff(6, zr, c)] = -dW[1];
        Zt[CC::zoff(7, zr, c)] = -dW[2];
        Zt[CC::zoff(8, zr, c)] = -dW[3];
      }
      if (mask & 4) {
        Zt[CC::zoff(9, zr, c)] = -dot3(nup, W + 1);
        for (int a = 0; a < 3; ++a) Zt[CC::zoff(10 + a, zr, c)] = -W[0] * nup[a] - nxW[a];
      }
    }
    __syncwarp();
    zero_entries(cb);   // the slots overwrote them
    __syncwarp();
    if (s + stride < sB) {
      if constexpr (C::NBUF == 1) issue_qs(s + stride, 0);
      issue_g(s + stride);
    }
    cp_async_commit();
  }
  cp_async_wait<0>();
}

// ------------------------------------------------------------------------------------------------
// k_contract: Step 8 in matrix mode (App. A.7) as DMMA GEMMs per tile of TP pairs of one
// patch: D = zeta(W) P_D, D' = zeta(dW) P_D, S' = zeta_S P_Sp, S = Theta P_Sd + zeta(W) P_Sg, then global
// units (A2), the smooth-rule subtraction (A14) and the CSR store.  Warp w owns the (M-tile, N-tile)
// pairs w, w + WARPS, ...; 4 accumulator tiles (S, D, S', D') each.  The Theta part of the tile's zeta
// and, per K chunk, the fit-operator rows with the matching zeta chunk are staged by bulk copies
// (ContractCfg: tile-chunked zeta written by k_translate), two stages, 3 CTAs per SM at p <= 8.
// ------------------------------------------------------------------------------------------------

// MK: the kernel mask at compile time (15 = all four, 3 = S|D: the DMMAs of the other kernels are compiled out --
// a predicated-off DMMA still occupies the tensor pipe), 0 = taken from `mask` at run time.
template <int P, int MK>
__global__ void __launch_bounds__(ContractCfg<P>::WARPS * 32, ContractCfg<P>::MINB)
    k_contract(int64_t item0, int64_t item1, const int64_t *__restrict__ item_ptr, const int32_t *__restrict__ item_patch,
               const int64_t *__restrict__ seg_ptr, int64_t sA, const ContractPair *__restrict__ cpair,
               const double *__restrict__ fit, const double *__restrict__ Zrow, const double *__restrict__ nodes,
               const double *__restrict__ normals, const double *__restrict__ weights, uint32_t mask, int raw, int64_t obase, int32_t *__restrict__ col_idx, double *vS, double *vD,
               double *vSp, double *vDp, int32_t *__restrict__ pstat) {
  using D = Dims<P>;
  using L = Layout<P>;
  using CC = ContractCfg<P>;
  constexpr int N = D::N, NP = D::NP, TP = CC::TP, ZTS = CC::ZTS, NB = CC::NB, KC = CC::KC;
  extern __shared__ __align__(16) double sz[];
  double *sB = sz + CC::ZT;                        // [2][B chunk: 3][KC][NB | Z chunk: 3][TP][KC]
  double *sN = sB + 2 * CC::STG;                   // nodes [N][3] | normals [N][3] | weights [N] of the patch
  ContractPair *sC = reinterpret_cast<ContractPair *>(sN + CC::SNODE);   // [TP] the tile's pairs
  const int64_t item = item0 + blockIdx.x;
  if (item >= item1) return;
  const int64_t Pp = item_patch[item];
  const int64_t s0 = seg_ptr[Pp] + (item - item_ptr[Pp]) * TP;
  const int cnt = (int)min((int64_t)TP, seg_ptr[Pp + 1] - s0);
  const double *blk = fit + Pp * (int64_t)L::STRIDE;
  const double *PD = blk + L::FIT, *PSp = PD + 4 * NP * NB, *PSd = PD + 8 * NP * NB, *PSg = PD + 9 * NP * NB;
  const double *Zblk = Zrow + (item - item0) * CC::ZBLK;   // rows of absent pairs: never read back
  // stage ch & 1: rows [ch KC, (ch+1) KC) of P_D, P_Sp, P_Sg and the tile's Z chunk ch; the Theta part,
  // the patch's nodes and the tile's pair records ride on chunk 0's barrier.  1-D bulk copies (TMA) on
  // mbarriers, issued by thread 0 (and 32 for the prologue extras).
  __shared__ uint64_t bar[2], emp[2];
  constexpr unsigned ROWB = (unsigned)(NB * sizeof(double)), ZCB = (unsigned)(CC::ZCH * sizeof(double));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&emp[0], CC::WARPS);
    mbar_init(&emp[1], CC::WARPS);
    mbar_fence_init();
  }
  __syncthreads();
  // the fit operators are stored with the padded row stride NB, so a chunk of each is one contiguous copy
  // kernel mask: an operand is staged / multiplied only if a selected kernel needs it (P_D: D, D'; P_Sp: S';
  // P_Sg, P_Sd: S); a masked-off kernel's zeta blocks were not written by k_translate
  const uint32_t km = MK ? (uint32_t)MK : mask;
  const bool wS = km & 1, wD = km & 2, wSp = km & 4, wDp = km & 8;
  const unsigned nops = (unsigned)((wD || wDp) + wSp + wS);
  auto issue = [&](int ch, unsigned extra) {
    uint64_t *br = &bar[ch & 1];
    if (threadIdx.x == 0) {
      mbar_expect_tx(br, nops * KC * ROWB + ZCB + extra);
      double *dst = sB + (ch & 1) * CC::STG;
      if (wD || wDp) bulk_g2s(dst, PD + (int64_t)ch * KC * NB, KC * ROWB, br);
      if (wSp) bulk_g2s(dst + KC * NB, PSp + (int64_t)ch * KC * NB, KC * ROWB, br);
      if (wS) bulk_g2s(dst + 2 * KC * NB, PSg + (int64_t)ch * KC * NB, KC * ROWB, br);
      bulk_g2s(dst + CC::SMEM_B, Zblk + CC::ZT + (int64_t)ch * CC::ZCH, ZCB, br);
    }
  };
  {
    const unsigned zb = wS ? (unsigned)(CC::ZT * sizeof(double)) : 0u, nb3 = (unsigned)(3 * N * sizeof(double)),
                   nb1 = (unsigned)(N * sizeof(double)), cb = (unsigned)(cnt * sizeof(ContractPair));
    issue(0, zb + 2 * nb3 + nb1 + cb);
    if (threadIdx.x == 32) {
      if (wS) bulk_g2s(sz, Zblk, zb, &bar[0]);
      bulk_g2s(sN, nodes + Pp * N * 3, nb3, &bar[0]);
      bulk_g2s(sN + 3 * N, normals + Pp * N * 3, nb3, &bar[0]);
      bulk_g2s(sN + 6 * N, weights + Pp * N, nb1, &bar[0]);
      bulk_g2s(sC, cpair + (s0 - sA), cb, &bar[0]);
    }
  }
  // P_Sd fragments for Theta . P_Sd straight from global, issued before waiting for the Z tile
  constexpr int NK = (NP + 3) / 4;
  double bq[CC::BQREG ? CC::TPW : 1][CC::BQREG ? NK : 1];
  auto psd = [&](int tw, int q) {
    const int tile = warp + tw * CC::WARPS, bn = (tile / CC::MT) * 8 + (lane >> 2), kk = 4 * q + (lane & 3);
    return (wS && tile < CC::TILES && bn < N && kk < NP) ? __ldg(PSd + kk * NB + bn) : 0.0;
  };
  if constexpr (CC::BQREG) {
#pragma unroll
    for (int tw = 0; tw < CC::TPW; ++tw)
#pragma unroll
      for (int q = 0; q < NK; ++q) bq[tw][q] = psd(tw, q);
  }
  const double h = blk[L::HDR + H_H];
  const double inv4pi = 1.0 / (4.0 * kPi);
  double acc[CC::TPW][8];
#pragma unroll
  for (int tw = 0; tw < CC::TPW; ++tw)
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[tw][q] = 0.0;
  mbar_wait(&bar[0], 0);   // Z tile (and chunk 0)
#pragma unroll
  for (int tw = 0; tw < CC::TPW; ++tw) {
    const int tile = warp + tw * CC::WARPS;
    if (tile >= CC::TILES || !wS) continue;
    const double *zr = sz + ((tile % CC::MT) * 8 + (lane >> 2)) * ZTS + (lane & 3);
#pragma unroll
    for (int q = 0; q < NK; ++q) {
      const int kk = 4 * q + (lane & 3);
      double bv;
      if constexpr (CC::BQREG) bv = bq[tw][q];
      else bv = psd(tw, q);
      dmma(acc[tw][0], acc[tw][1], kk < NP ? zr[4 * q] : 0.0, bv);
    }
  }
  // the 4 NP blocks, B double-buffered through shared memory; emp[b] = "every warp is done with buffer b"
  // (no CTA-wide barrier in the K loop).  A warp's tiles share the M-tile (tile = warp + WARPS tw).
  static_assert(CC::WARPS % CC::MT == 0, "a warp's tiles share one M-tile");
  const int mtw = warp % CC::MT;
  const int zrow = mtw * 8 + (lane >> 2), zsw = CC::swz(zrow);
  const int zofs = zrow * KC + (lane & 3);
  for (int ch = 0; ch < CC::NCH; ++ch) {
    if (ch + 1 < CC::NCH && threadIdx.x == 0) {   // refill buffer (ch+1)&1 once every warp has left chunk ch-1
      if (ch >= 1) mbar_wait(&emp[(ch + 1) & 1], ((ch - 1) >> 1) & 1);
      fence_proxy_async();
      issue(ch + 1, 0);
    }
    mbar_wait(&bar[ch & 1], (ch >> 1) & 1);
    const double *bb = sB + (ch & 1) * CC::STG;
    const double *zr = bb + CC::SMEM_B + zofs;
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
      const double zw = zr[kk ^ zsw], zdw = zr[TP * KC + (kk ^ zsw)], zs = zr[2 * TP * KC + (kk ^ zsw)];
#pragma unroll
      for (int tw = 0; tw < CC::TPW; ++tw) {
        const int tile = warp + tw * CC::WARPS;
        if (tile >= CC::TILES) continue;
        const int bn = (tile / CC::MT) * 8 + (lane >> 2);
        const bool bok = bn < N;
        const int br = (kk + (lane & 3)) * NB + bn;
        const double bd = bok ? bb[br] : 0.0, bsp = bok ? bb[KC * NB + br] : 0.0, bsg = bok ? bb[2 * KC * NB + br] : 0.0;
        if (wD) dmma(acc[tw][2], acc[tw][3], zw, bd);
        if (wDp) dmma(acc[tw][6], acc[tw][7], zdw, bd);
        if (wSp) dmma(acc[tw][4], acc[tw][5], zs, bsp);
        if (wS) dmma(acc[tw][0], acc[tw][1], zw, bsg);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&emp[ch & 1]);
  }
  // unrolled (the accumulators stay in registers; a rolled loop indexes them through local memory)
#pragma unroll
  for (int tw = 0; tw < CC::TPW; ++tw) {
    const int tile = warp + tw * CC::WARPS;
    if (tile >= CC::TILES) continue;
    const int mt = tile % CC::MT, nt = tile / CC::MT;
    const double aS0 = acc[tw][0], aS1 = acc[tw][1], aD0 = acc[tw][2], aD1 = acc[tw][3], aSp0 = acc[tw][4],
                 aSp1 = acc[tw][5], aDp0 = acc[tw][6], aDp1 = acc[tw][7];
  // epilogue: C[row = lane/4][col = 2 (lane%4) + {0,1}]
    const int row = mt * 8 + (lane >> 2);
    if (row >= cnt) continue;
    const double accS[2] = {aS0, aS1}, accD[2] = {aD0, aD1}, accSp[2] = {aSp0, aSp1}, accDp[2] = {aDp0, aDp1};
    double oS[2], oD[2], oSp[2], oDp[2];
    bool bad = false;
    const int i0 = nt * 8 + 2 * (lane & 3);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int i = i0 + q;
      double S = accS[q] * h, Dv = accD[q], Sp = accSp[q], Dp = accDp[q] / h;
      if (!raw && i < N && sC[row].self_local != i) {
        const double *xi = sN + 3 * i, *ni = sN + 3 * N + 3 * i;
        const double wi = sN[6 * N + i];
        const double *tr = sC[row].x, *tn = sC[row].n;
        const double d0 = tr[0] - xi[0], d1 = tr[1] - xi[1], d2 = tr[2] - xi[2];
        const double r2 = d0 * d0 + d1 * d1 + d2 * d2;
        const double ir = rsqrt_nr(r2);
        const double ir3 = ir * ir * ir;
        const double dn = d0 * ni[0] + d1 * ni[1] + d2 * ni[2];
        const double dnp = d0 * tn[0] + d1 * tn[1] + d2 * tn[2];
        const double nn = ni[0] * tn[0] + ni[1] * tn[1] + ni[2] * tn[2];
        S -= inv4pi * ir * wi;
        Dv -= inv4pi * dn * ir3 * wi;
        Sp += inv4pi * dnp * ir3 * wi;
        Dp -= inv4pi * (nn * ir3 - 3.0 * dn * dnp * ir3 * ir * ir) * wi;
      }
      oS[q] = wS ? S : 0.0;
      oD[q] = wD ? Dv : 0.0;
      oSp[q] = wSp ? Sp : 0.0;
      oDp[q] = wDp ? Dp : 0.0;
      if (i < N) bad |= !isfinite(oS[q]) || !isfinite(oD[q]) || !isfinite(oSp[q]) || !isfinite(oDp[q]);
    }
    const int64_t o = (sC[row].k - obase) * N + i0;
    if (i0 + 1 < N) {   // the usual case: both columns, 16-B stores
      if (col_idx) *reinterpret_cast<int2 *>(col_idx + o) = make_int2((int32_t)(Pp * N + i0), (int32_t)(Pp * N + i0 + 1));
      if (vS) *reinterpret_cast<double2 *>(vS + o) = make_double2(oS[0], oS[1]);
      if (vD) *reinterpret_cast<double2 *>(vD + o) = make_double2(oD[0], oD[1]);
      if (vSp) *reinterpret_cast<double2 *>(vSp + o) = make_double2(oSp[0], oSp[1]);
      if (vDp) *reinterpret_cast<double2 *>(vDp + o) = make_double2(oDp[0], oDp[1]);
    } else if (i0 < N) {
      if (col_idx) col_idx[o] = (int32_t)(Pp * N + i0);
      if (vS) vS[o] = oS[0];
      if (vD) vD[o] = oD[0];
      if (vSp) vSp[o] = oSp[0];
      if (vDp) vDp[o] = oDp[0];
    }
    if (bad && pstat) atomicOr(pstat + (sC[row].k - obase), 2);
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

// item -> patch map for the tile kernels (items of patch P are [items[P], items[P+1])).
__global__ void k_item_patch(int64_t n_patches, const int64_t *__restrict__ items, int32_t *__restrict__ item_patch) {
  int64_t P = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (P >= n_patches) return;
  for (int64_t i = items[P]; i < items[P + 1]; ++i) item_patch[i] = (int32_t)P;
}

// The pair range [pair_ptr[row_begin], pair_ptr[row_end]) of a build call, written to mapped host memory.
__global__ void k_pair_range(const int64_t *__restrict__ pair_ptr, int64_t row_begin, int64_t row_end, int64_t *out) {
  if (threadIdx.x == 0) {
    out[0] = pair_ptr[row_begin];
    out[1] = pair_ptr[row_end];
  }
}

__global__ void k_copy_i64(int64_t n, const int64_t *__restrict__ a, int64_t *__restrict__ b) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}

// CSR SpMV: warp per row.
// Test hook (rrq_debug_zeta): zeta rows of the last sub-chunk, in pair order, out of the tile-chunked layout.
template <int P>
__global__ void k_debug_zeta(int64_t np_, const PairSetup *__restrict__ setup, const double *__restrict__ Z,
                             double *__restrict__ out) {
  using CC = ContractCfg<P>;
  constexpr int NP = Dims<P>::NP;
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= np_ * 13 * NP) return;
  const int64_t i = w / (13 * NP);
  const int bc = (int)(w % (13 * NP)), b = bc / NP, c = bc % NP;
  const int64_t a = setup[i].aslot;
  out[w] = Z[(a >> 5) * CC::ZBLK + CC::zoff(b, (int)(a & 31), c)];
}

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
