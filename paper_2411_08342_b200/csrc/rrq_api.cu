// C ABI of librrq.so (include/rrq.h): argument validation, scratch management, launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rrq.h"
#include "k_build.cuh"
#include "k_near.cuh"
#include "k_patch.cuh"
#include "k_smooth.cuh"

namespace rrq_host {
void gauss_legendre(int n, double *x, double *w);
void vandermonde_inverse(int n, const double *t, double *U);
}  // namespace rrq_host

using namespace rrq;

struct rrq_ctx_s {
  rrq_params prm;
  std::string err;
  int64_t launches = 0;
  int num_sms = 148;
  int device = 0;                // the device current at rrq_create; every call must run with it current
  // constant tables (device) + host copies
  double *d_tab = nullptr;
  double *d_trtab = nullptr;   // k_translate schedule + scale tables (TrCfg<p>)
  Tables T;
  std::vector<double> h_t, h_w, h_U;
  // scratch
  struct Buf {
    void *p = nullptr;
    size_t n = 0;
  };
  int64_t last_np = 0, last_nz = 0, last_sA = 0;
  int last_set = 0;
  // The producer kernels' outputs are double-buffered (set = sub-chunk parity) so that the producer stream (k_pair_setup,
  // k_newton, k_edge_lines, k_target_gamma of sub-chunk i+1) runs concurrently with the consumer stream (k_qmap, k_translate, k_contract of
  // sub-chunk i): the edge kernel is FP64-latency bound and the GEMM kernels leave the FP64 pipe ~40 % idle.
  Buf Arow[2], Xrow[2], psetup[2], cpair[2], et0[2], om[2], Qrow, ipatch;
  cudaStream_t st2 = nullptr;                      // producer stream (created on first use)
  cudaEvent_t ev_edge[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr}, ev_fork = nullptr, ev_join = nullptr;
  bool overlap = true;                             // RRQ_NO_OVERLAP=1 runs everything on the caller's stream
  double scratch_bytes = 24e9;                     // sub-chunk scratch budget (RRQ_SCRATCH_BYTES: test hook)
  Buf balls, cell_cnt, cell_items, patch_cell, tcnt, ptgt, perm, seg, cursor, items, Z, fitwork, one, swapcnt;
  // Small device->host reads inside rrq_build_correction (the pair range, the per-patch segment and item offsets)
  // go through mapped pinned memory written by a kernel, not cudaMemcpyAsync: a D2H memcpy queues behind
  // whatever the caller's own D2H copies hold on the copy engine (an e2e loop copying the previous chunk's
  // weights out), which would stall this call's host-side planning for the length of that copy.
  int64_t *hmap = nullptr;
  size_t hmap_n = 0;
  // device-time accounting (rrq_set_timing)
  bool timing = false;
  double t_ms[RRQ_NSTAGES] = {};
  int64_t t_n[RRQ_NSTAGES] = {};
  int64_t stats[2] = {0, 0};
  struct Pend {
    int stage;
    cudaEvent_t a, b;
  };
  std::vector<Pend> pend;
  std::vector<cudaEvent_t> pool;
};

static cudaEvent_t ev_get(rrq_ctx c) {
  if (c->pool.empty()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  cudaEvent_t e = c->pool.back();
  c->pool.pop_back();
  return e;
}
// Bracket a launch with events on its stream (only when timing is enabled).
struct TScope {
  rrq_ctx c;
  int stage;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  TScope(rrq_ctx c_, int s_, cudaStream_t st_) : c(c_), stage(s_), st(st_) {
    if (c->timing) {
      a = ev_get(c);
      cudaEventRecord(a, st);
    }
  }
  ~TScope() {
    if (c->timing) {
      cudaEvent_t b = ev_get(c);
      cudaEventRecord(b, st);
      c->pend.push_back({stage, a, b});
    }
  }
};
static void t_flush(rrq_ctx c) {
  for (auto &p : c->pend) {
    cudaEventSynchronize(p.b);
    float ms = 0;
    cudaEventElapsedTime(&ms, p.a, p.b);
    c->t_ms[p.stage] += ms;
    c->t_n[p.stage] += 1;
    c->pool.push_back(p.a);
    c->pool.push_back(p.b);
  }
  c->pend.clear();
}

static thread_local std::string g_create_err;

static rrq_status fail(rrq_ctx c, rrq_status s, const std::string &m) {
  if (c) c->err = m; else g_create_err = m;
  return s;
}

static rrq_status cuda_check(rrq_ctx c, const char *where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, RRQ_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
  return RRQ_OK;
}

static bool ensure(rrq_ctx c, rrq_ctx_s::Buf &b, size_t bytes) {
  if (bytes == 0) bytes = 8;
  if (b.n >= bytes) return true;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.n = 0;
  if (cudaMalloc(&b.p, bytes) != cudaSuccess) {
    cudaGetLastError();
    c->err = "scratch allocation of " + std::to_string(bytes) + " bytes failed";
    return false;
  }
  b.n = bytes;
  return true;
}

static bool ensure_hmap(rrq_ctx c, size_t n) {
  if (c->hmap_n >= n) return true;
  if (c->hmap) cudaFreeHost(c->hmap);
  c->hmap = nullptr;
  c->hmap_n = 0;
  if (cudaHostAlloc((void **)&c->hmap, n * sizeof(int64_t), cudaHostAllocMapped) != cudaSuccess) {
    cudaGetLastError();
    c->err = "mapped host allocation of " + std::to_string(n * sizeof(int64_t)) + " bytes failed";
    return false;
  }
  c->hmap_n = n;
  return true;
}

template <typename T>
static T *bp(rrq_ctx_s::Buf &b) { return reinterpret_cast<T *>(b.p); }

static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// Exported functions get C linkage from their declarations in include/rrq.h.

// k_translate's host-built table (TrCfg<P>).  Blocks of WD outputs (l, m0 .. m0 + WD - 1), l-major; a block's
// steps are its j = 2..l sweeps over k (from the smallest to the largest k any output of the block takes),
// each step = the Q entry (j, |k|) (k < 0: the sign of Q.x flipped for odd k (FA), of Q.y for even k (FB)) and the
// new window entry S'^{(l-j, m0-k)} (the zero entry ZE outside |m'| <= l').  A block is split into
// ceil(len / STEPS) contiguous pieces of near-equal length, one lane each (lanes in block order); a piece's
// first step and every sweep's first step carry PRIME: window entries 1 .. WD-1 (S'^{(l-j, m0+i-k)}, mostly
// the zero entry) are loaded.  Padding steps read the zero Q entry ZQ.  cinfo[c] = l | m << 4 | i << 8 |
// first lane << 12 | lanes << 20 (i = m - m0).
// Scale factors: v_lambda(j,k) = (j-2)!/F(j,k), v_theta(j,k) = (j-1)!/F(j,k), w(l',m') = l'!/F(l',m'),
// u_lambda(l,m) = F(l,m)/(l-1)!, u_theta(l,m) = F(l,m)/l!, F(a,b) = sqrt((a+b)! (a-b)!).
// The shared-memory positions of the Q entries (pq) and of the S' entries (ps) are chosen by annealing so
// that at each step the 8 lanes of a quarter-warp read entries in distinct 16-B bank groups.
template <int P>
static std::vector<double> make_trtab() {
  using C = TrCfg<P>;
  using D = Dims<P>;
  constexpr int ZE = P * P, WD = C::WD, ST = C::STEPS, ZQ = C::ZQ;
  struct Step { int qe, se, k, flags, pe[4]; };
  auto sidx2 = [](int lp, int mp) { return (mp < -lp || mp > lp) ? ZE : lp * lp + lp + mp; };
  struct Blk { int l, m0; std::vector<Step> st; };
  std::vector<Blk> blks;
  for (int l = 2; l <= P; ++l)
    for (int m0 = 1; m0 <= l; m0 += WD) {
      Blk B{l, m0, {}};
      const int m1 = std::min(m0 + WD - 1, l);
      for (int j = 2; j <= l; ++j) {
        const int lp = l - j, lo = std::max(-j, m0 - lp), hi = std::min(j, m1 + lp);
        for (int k = lo; k <= hi; ++k) {
          Step t{qidx(j, std::abs(k)), sidx2(lp, m0 - k), k, 0, {ZE, ZE, ZE, ZE}};
          for (int i = 1; i < WD; ++i) t.pe[i - 1] = (m0 + i <= l) ? sidx2(lp, m0 + i - k) : ZE;
          if (k < 0) t.flags |= (std::abs(k) & 1) ? C::FA : C::FB;
          if (k == lo && j > 2) t.flags |= C::PRIME;   // a new sweep: window entries 1 .. WD-1 reloaded
          B.st.push_back(t);
        }
      }
      if ((int)B.st.size() != tr_block_len(l, m0, WD)) { std::fprintf(stderr, "rrq: translate block length\n"); std::abort(); }
      blks.push_back(B);
    }
  // pieces of each block (near-equal contiguous parts of at most ST steps, one lane each, padded to ST); the
  // blocks are laid over the 32 lanes in the order `order` (a block's pieces on consecutive lanes), which the
  // bank search below may permute
  std::vector<std::vector<std::vector<Step>>> pieces(blks.size());
  int total_lanes = 0;
  for (size_t b = 0; b < blks.size(); ++b) {
    const int len = (int)blks[b].st.size(), n = (len + ST - 1) / ST;
    for (int q = 0; q < n; ++q) {
      const int f = (int)((int64_t)q * len / n), e = (int)((int64_t)(q + 1) * len / n);
      std::vector<Step> pc;
      for (int i = f; i < e; ++i) {
        Step t = blks[b].st[i];
        if (i == f) t.flags = (t.flags & (C::FA | C::FB)) | C::PRIME;
        pc.push_back(t);
      }
      if ((int)pc.size() > ST) { std::fprintf(stderr, "rrq: translate piece too long\n"); std::abort(); }
      while ((int)pc.size() < ST) pc.push_back(Step{ZQ, ZE, 0, 0, {ZE, ZE, ZE, ZE}});
      pieces[b].push_back(pc);
    }
    total_lanes += n;
  }
  if (total_lanes > 32) { std::fprintf(stderr, "rrq: translate schedule needs more than 32 lanes\n"); std::abort(); }
  std::vector<int> order(blks.size());
  for (size_t b = 0; b < blks.size(); ++b) order[b] = (int)b;
  std::vector<std::vector<Step>> lanes(32);
  std::vector<int> bfirst(blks.size()), bcnt(blks.size());
  auto assign = [&]() {
    int L = 0;
    for (int b : order) {
      bfirst[b] = L;
      bcnt[b] = (int)pieces[b].size();
      for (auto &pc : pieces[b]) lanes[L++] = pc;
    }
    for (; L < 32; ++L) {
      lanes[L].assign(ST, Step{ZQ, ZE, 0, 0, {ZE, ZE, ZE, ZE}});
      lanes[L][0].flags = (int)C::PRIME;
    }
  };
  assign();
  // Bank model (quarter-warp: 8 lanes per wavefront of 16-B accesses, tools/lds_banks.cu): a Q entry at
  // position x starts in 16-B group x mod 8 (stride 144 B) and its 8 chunks and V follow; an S' entry at
  // position y starts in group 3y mod 8 (stride 48 B).  Cost of a quarter = 9 x (max distinct Q entries in
  // one group) + 2 x (same for the new S' entries) (+ the PRIME loads, which all lanes issue at step 0).
  std::vector<int> pq(D::NQ + 1), ps(ZE + 1);
  for (int e = 0; e <= D::NQ; ++e) pq[e] = e;
  for (int e = 0; e <= ZE; ++e) ps[e] = e;
  auto mult = [](const int *ent, const int *grp, int n) {
    uint64_t m[8][4] = {};   // entries < 256 (p = 14: p^2 + 1 = 197)
    for (int i = 0; i < n; ++i) m[grp[i]][ent[i] >> 6] |= 1ull << (ent[i] & 63);
    int best = 1;
    for (int g = 0; g < 8; ++g)
      best = std::max(best, __builtin_popcountll(m[g][0]) + __builtin_popcountll(m[g][1]) + __builtin_popcountll(m[g][2]) +
                                __builtin_popcountll(m[g][3]));
    return best;
  };
  auto cost = [&]() {
    int tot = 0;
    for (int t = 0; t < ST; ++t)
      for (int q = 0; q < 4; ++q) {
        int eq[8], gq[8], es[8], gs[8];
        for (int i = 0; i < 8; ++i) {
          const Step &s = lanes[8 * q + i][t];
          eq[i] = s.qe; gq[i] = pq[s.qe] & 7;
          es[i] = s.se; gs[i] = (3 * ps[s.se]) & 7;
        }
        tot += 9 * mult(eq, gq, 8) + 2 * mult(es, gs, 8);
        if (t == 0)
          for (int w = 0; w < WD - 1; ++w) {
            for (int i = 0; i < 8; ++i) { es[i] = lanes[8 * q + i][0].pe[w]; gs[i] = (3 * ps[es[i]]) & 7; }
            tot += 2 * mult(es, gs, 8);
          }
      }
    return tot;
  };
  int cur = cost(), best = cur;
  std::vector<int> best_pq = pq, best_ps = ps;
  uint64_t rng = 0x9E3779B97F4A7C15ull;
  auto rnd = [&]() { rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17; return rng; };
  double T = 3.0;
  // search length: ~100k moves at p = 8 (0.8 s, once per process and order: make_trtab_p caches), fewer for the
  // long schedules of the high orders
  static const int n_anneal = std::getenv("RRQ_TRTAB_ITERS") ? std::atoi(std::getenv("RRQ_TRTAB_ITERS")) : (900000 / ST > 200000 ? 200000 : 900000 / ST);
  std::vector<int> best_order = order;
  for (int it = 0; it < n_anneal; ++it) {
    const int kind = (int)(rnd() % 3);   // 0: Q positions, 1: S' positions, 2: block order over the lanes
    int a, b2;
    if (kind == 2) {
      a = (int)(rnd() % order.size()); b2 = (int)(rnd() % order.size());
      if (a == b2) continue;
      std::swap(order[a], order[b2]);
      assign();
    } else {
      std::vector<int> &v = kind == 0 ? pq : ps;
      const int n = kind == 0 ? D::NQ : ZE;   // the zero entries keep the last positions
      a = (int)(rnd() % n); b2 = (int)(rnd() % n);
      if (a == b2) continue;
      std::swap(v[a], v[b2]);
    }
    const int c = cost();
    const double u = (double)(rnd() >> 11) * (1.0 / 9007199254740992.0);
    if (c <= cur || u < std::exp((cur - c) / T)) cur = c;
    else if (kind == 2) { std::swap(order[a], order[b2]); assign(); }
    else std::swap(kind == 0 ? pq[a] : ps[a], kind == 0 ? pq[b2] : ps[b2]);
    if (cur < best) { best = cur; best_pq = pq; best_ps = ps; best_order = order; }
    T = std::max(0.05, T * 0.9997);
  }
  order = best_order;
  assign();
  pq = best_pq; ps = best_ps;
  if (std::getenv("RRQ_DEBUG_TRTAB"))   // modelled shared-memory wavefronts of the main loop against the conflict-free count
    std::fprintf(stderr, "rrq: translate schedule p = %d: %d steps, bank cost %d (conflict-free %d)\n", P, ST, best,
                 ST * 4 * 11 + 4 * 2 * (WD - 1));
  std::vector<uint32_t> w(C::NWORD, 0u);
  for (int l2 = 0; l2 < 32; ++l2)
    for (int t = 0; t < ST; ++t) {
      const Step &s = lanes[l2][t];
      w[t * 32 + l2] = (uint32_t)pq[s.qe] | (uint32_t)ps[s.se] << 7 | (uint32_t)s.flags;
      uint32_t pw = 0;
      for (int i = 0; i < WD - 1; ++i) pw |= (uint32_t)ps[s.pe[i]] << (C::SEB * i);
      w[ST * 32 + t * 32 + l2] = pw;
    }
  uint32_t *ci = w.data() + 2 * ST * 32;
  for (size_t b = 0; b < blks.size(); ++b)
    for (int i = 0; i < WD && blks[b].m0 + i <= blks[b].l; ++i) {
      const int l = blks[b].l, m = blks[b].m0 + i;
      ci[lmidx(l, m)] = (uint32_t)l | (uint32_t)m << 4 | (uint32_t)i << 8 | (uint32_t)bfirst[b] << 12 |
                        (uint32_t)bcnt[b] << 20;
    }
  ci[lmidx(1, 1)] = 1u | 1u << 4;   // (1,1): j = 1 terms only (no slots)
  {   // shared-memory positions of the Q entries and S' entries
    uint8_t *pb = reinterpret_cast<uint8_t *>(ci + D::NP);
    for (int e = 0; e < D::NQ; ++e) pb[e] = (uint8_t)pq[e];
    for (int e = 0; e < ZE; ++e) pb[D::NQ + e] = (uint8_t)ps[e];
  }
  auto fact = [](int n) { long double f = 1; for (int i = 2; i <= n; ++i) f *= i; return f; };
  auto F = [&](int a, int b) { const int ab = std::abs(b); return std::sqrt(fact(a + ab) * fact(a - ab)); };
  std::vector<double> out(C::TAB_D, 0.0);
  std::memcpy(out.data(), w.data(), w.size() * sizeof(uint32_t));
  double *vlam = out.data() + C::VLAM, *vth = out.data() + C::VTH, *wS = out.data() + C::WS;
  double *olam = out.data() + C::OLAM, *oth = out.data() + C::OTH;
  for (int j = 2; j <= P; ++j)
    for (int k = 0; k <= j; ++k) vlam[qidx(j, k)] = (double)(fact(j - 2) / F(j, k));
  for (int j = 1; j <= P; ++j)
    for (int k = 0; k <= j; ++k) vth[vidx(j, k)] = (double)(fact(j - 1) / F(j, k));
  for (int lp = 0; lp < P; ++lp)
    for (int mp = -lp; mp <= lp; ++mp) wS[lp * lp + lp + mp] = (double)(fact(lp) / F(lp, mp));
  for (int l = 1; l <= P; ++l)
    for (int m = 1; m <= l; ++m) {
      olam[lmidx(l, m)] = (double)(F(l, m) / fact(l - 1));
      oth[lmidx(l, m)] = (double)(F(l, m) / fact(l));
    }
  return out;
}

static std::vector<double> make_trtab_p_uncached(int p);
// the schedule search is deterministic: one table per order and process
static const std::vector<double> &make_trtab_p(int p) {
  static std::mutex mu;
  static std::map<int, std::vector<double>> cache;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(p);
  if (it == cache.end()) it = cache.emplace(p, make_trtab_p_uncached(p)).first;
  return it->second;
}
static std::vector<double> make_trtab_p_uncached(int p) {
  switch (p) {
    case 4: return make_trtab<4>();
    case 6: return make_trtab<6>();
    case 8: return make_trtab<8>();
    case 10: return make_trtab<10>();
    case 12: return make_trtab<12>();
    default: return make_trtab<14>();
  }
}

// Host-side check of k_translate's packed schedule (no CUDA call): decode the table exactly as the kernel's main
// loop and epilogue do (TrCfg field widths, window ring, prime codes, slot sums) and compare the terms every
// output (l, m) receives with the definition of the direct translation (G4):
//   W^{(l,m)} <- sum_{j=2..l} sum_{|k|<=j, |m-k|<=l-j} Q^{(j,k)} S'^{(l-j, m-k)},  k < 0 by conjugate symmetry
// (sign flags FA for odd k, FB for even k).  Returns 0 if every output gets exactly its terms once.
template <int P>
static int check_trtab() {
  using C = TrCfg<P>;
  using D = Dims<P>;
  constexpr int WD = C::WD, ST = C::STEPS, ZE = P * P, ZQ = C::ZQ;
  const std::vector<double> &tab = make_trtab_p(P);
  const uint32_t *code = reinterpret_cast<const uint32_t *>(tab.data());
  const uint32_t *pcode = code + ST * 32, *cinfo = pcode + ST * 32;
  const uint8_t *posq = reinterpret_cast<const uint8_t *>(cinfo + D::NP), *poss = posq + D::NQ;
  // position -> entry (the zero entries keep the last positions)
  std::vector<int> qent(D::NQ + 1, -1), sent(ZE + 1, -1);
  for (int e = 0; e < D::NQ; ++e) { if (posq[e] > D::NQ || qent[posq[e]] >= 0) return 1; qent[posq[e]] = e; }
  for (int e = 0; e < ZE; ++e) { if (poss[e] > ZE || sent[poss[e]] >= 0) return 2; sent[poss[e]] = e; }
  if (qent[ZQ] >= 0 || sent[ZE] >= 0) return 3;   // the zero entries' positions must be free
  qent[ZQ] = ZQ; sent[ZE] = ZE;
  // a term: Q entry, sign flags, S' entry;  acc[lane][i] = terms accumulated for output i of the lane's block
  struct Term { int q, fl, s; bool operator<(const Term &o) const { return q != o.q ? q < o.q : fl != o.fl ? fl < o.fl : s < o.s; } bool operator==(const Term &o) const { return q == o.q && fl == o.fl && s == o.s; } };
  std::vector<std::vector<Term>> acc(32 * WD);
  for (int lane = 0; lane < 32; ++lane) {
    int ring[8];
    for (int i = 0; i < WD; ++i) ring[i] = ZE;
    for (int t = 0; t < ST; ++t) {
      const uint32_t cw = code[t * 32 + lane];
      const int qe = cw & 127, se = (cw >> 7) & C::SEM;
      if (qe > D::NQ || se > ZE) return 4;
      ring[t % WD] = sent[se];
      if (t == 0 || (cw & C::PRIME)) {
        const uint32_t pw = pcode[t * 32 + lane];
        for (int i = 1; i < WD; ++i) {
          const int pe = (pw >> (C::SEB * (i - 1))) & C::SEM;
          if (pe > ZE) return 5;
          ring[(t - i + WD * ST) % WD] = sent[pe];
        }
      }
      const int fl = ((cw & C::FA) ? 1 : 0) | ((cw & C::FB) ? 2 : 0);
      for (int i = 0; i < WD; ++i) {
        const int s = ring[(t - i + WD * ST) % WD];
        if (qent[qe] == ZQ || s == ZE) continue;   // a zero operand: no contribution
        acc[lane * WD + i].push_back(Term{qent[qe], fl, s});
      }
    }
  }
  for (int l = 1; l <= P; ++l)
    for (int m = 1; m <= l; ++m) {
      const uint32_t ci = cinfo[lmidx(l, m)];
      if ((int)(ci & 15) != l || (int)((ci >> 4) & 15) != m) return 6;
      const int ib = (ci >> 8) & 15, fl0 = (ci >> 12) & 255, nl = (ci >> 20) & 63;
      std::vector<Term> got, want;
      for (int q = 0; q < nl; ++q) {
        if (fl0 + q >= 32 || ib >= WD) return 7;
        const auto &v = acc[(fl0 + q) * WD + ib];
        got.insert(got.end(), v.begin(), v.end());
      }
      for (int j = 2; j <= l; ++j)
        for (int k = -j; k <= j; ++k) {
          const int lp = l - j, mp = m - k;
          if (mp < -lp || mp > lp) continue;
          want.push_back(Term{qidx(j, k < 0 ? -k : k), k < 0 ? ((-k) & 1 ? 1 : 2) : 0, lp * lp + lp + mp});
        }
      std::sort(got.begin(), got.end());
      std::sort(want.begin(), want.end());
      if (!(got == want)) return 100 + lmidx(l, m);
    }
  return 0;
}

int rrq_selftest_translate_schedule(int p) {
  switch (p) {
    case 4: return check_trtab<4>();
    case 6: return check_trtab<6>();
    case 8: return check_trtab<8>();
    case 10: return check_trtab<10>();
    case 12: return check_trtab<12>();
    case 14: return check_trtab<14>();
  }
  return -1;
}

static cudaError_t set_kernel_attributes(int p, int n_omega);

// Every entry point runs with the device the context was created on (its tables, scratch and the kernels'
// shared-memory attributes belong to that device).
static rrq_status check_device(rrq_ctx c) {
  int d = -1;
  if (cudaGetDevice(&d) != cudaSuccess || d != c->device)
    return fail(c, RRQ_ERR_INVALID_ARG, "the current CUDA device is not the one this rrq_ctx was created on");
  return RRQ_OK;
}

rrq_status rrq_create(const rrq_params *params, rrq_ctx *out) {
  if (!out) return fail(nullptr, RRQ_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (!params) return fail(nullptr, RRQ_ERR_INVALID_ARG, "params is NULL");
  const rrq_params &p = *params;
  if (p.p != 4 && p.p != 6 && p.p != 8 && p.p != 10 && p.p != 12 && p.p != 14)
    return fail(nullptr, RRQ_ERR_NOT_IMPLEMENTED, "p must be one of 4, 6, 8, 10, 12, 14");
  if (p.n_nodes != p.p * p.p) return fail(nullptr, RRQ_ERR_INVALID_ARG, "n_nodes must be p*p (collapsed GL, A1)");
  if (p.p_edge != 2 * p.p) return fail(nullptr, RRQ_ERR_NOT_IMPLEMENTED, "p_edge must be 2p (reading A4)");
  if (p.n_omega < 1 || p.n_omega > 128) return fail(nullptr, RRQ_ERR_INVALID_ARG, "n_omega must be in [1,128]");
  if (!(p.rho_swap > 1.0)) return fail(nullptr, RRQ_ERR_INVALID_ARG, "rho_swap must be > 1");
  if (!(p.eta >= 0.0)) return fail(nullptr, RRQ_ERR_INVALID_ARG, "eta must be >= 0");
  rrq_ctx c = new rrq_ctx_s();
  c->prm = p;
  int dev = 0;
  cudaGetDevice(&dev);
  c->device = dev;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, dev);
  {
    const char *e = std::getenv("RRQ_NO_OVERLAP");
    c->overlap = !(e && std::atoi(e) != 0);
    const char *sb = std::getenv("RRQ_SCRATCH_BYTES");
    if (sb && std::atof(sb) > 0) c->scratch_bytes = std::atof(sb);
  }
  int q = p.p_edge, no = p.n_omega;
  c->h_t.resize(q);
  c->h_w.resize(q);
  c->h_U.resize(q * q);
  rrq_host::gauss_legendre(q, c->h_t.data(), c->h_w.data());
  rrq_host::vandermonde_inverse(q, c->h_t.data(), c->h_U.data());
  std::vector<double> xo(no), wo(no), sqb(41 * 41, 0.0);
  rrq_host::gauss_legendre(no, xo.data(), wo.data());
  for (int n = 0; n <= 40; ++n) {
    double b = 1;
    for (int k = 0; k <= n; ++k) {
      sqb[n * 41 + k] = std::sqrt(b);
      b = b * (n - k) / (k + 1);
    }
  }
  std::vector<double> xd(kNDirect), wd(kNDirect), xdp(kNDirect * q);
  rrq_host::gauss_legendre(kNDirect, xd.data(), wd.data());
  for (int j = 0; j < kNDirect; ++j) {
    double pw = 1;
    for (int k = 0; k < q; ++k) { xdp[j * q + k] = pw; pw *= xd[j]; }
  }
  std::vector<double> hcv(HC_SIZE, 0.0);
  for (int l = 0; l <= HC_LMAX; ++l)
    for (int m = -l; m <= l; ++m) {
      double lm = l - m, lp = l + m;
      double *dc = hcv.data() + HC_DC + 3 * (l * l + l + m);
      dc[0] = lm * lp > 0 ? std::sqrt(lm * lp) : 0.0;
      dc[1] = lm * (lm - 1) > 0 ? std::sqrt(lm * (lm - 1)) : 0.0;
      dc[2] = lp * (lp - 1) > 0 ? std::sqrt(lp * (lp - 1)) : 0.0;
    }
  for (int m = 0; m <= HC_LMAX; ++m) {
    hcv[HC_DG + m] = m > 0 ? std::sqrt((2.0 * m - 1.0) / (2.0 * m)) : 1.0;
    hcv[HC_SB + m] = std::sqrt(2.0 * m + 1.0);
  }
  for (int l = 0; l <= HC_LMAX; ++l)
    for (int m = 0; m <= l; ++m) {
      double den = std::sqrt((double)(l + 1 + m) * (l + 1 - m));
      hcv[HC_RA + sidx(l, m)] = (2.0 * l + 1.0) / den;
      hcv[HC_RB + sidx(l, m)] = std::sqrt((double)(l + m) * (l - m)) / den;
    }
  size_t tot = 2 * q + q * q + 2 * no + 41 * 41 + 2 * kNDirect + kNDirect * q + HC_SIZE;
  if (cudaMalloc(&c->d_tab, tot * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    delete c;
    return fail(nullptr, RRQ_ERR_CUDA, "cudaMalloc of constant tables failed (no CUDA device?)");
  }
  std::vector<double> h(tot);
  double *t = h.data();
  std::copy(c->h_t.begin(), c->h_t.end(), t);
  std::copy(c->h_w.begin(), c->h_w.end(), t + q);
  std::copy(c->h_U.begin(), c->h_U.end(), t + 2 * q);
  std::copy(xo.begin(), xo.end(), t + 2 * q + q * q);
  std::copy(wo.begin(), wo.end(), t + 2 * q + q * q + no);
  std::copy(sqb.begin(), sqb.end(), t + 2 * q + q * q + 2 * no);
  double *td = t + 2 * q + q * q + 2 * no + 41 * 41;
  std::copy(xd.begin(), xd.end(), td);
  std::copy(wd.begin(), wd.end(), td + kNDirect);
  std::copy(xdp.begin(), xdp.end(), td + 2 * kNDirect);
  std::copy(hcv.begin(), hcv.end(), td + 2 * kNDirect + kNDirect * q);
  cudaMemcpy(c->d_tab, h.data(), tot * sizeof(double), cudaMemcpyHostToDevice);
  c->T.tgl = c->d_tab;
  c->T.wgl = c->d_tab + q;
  c->T.U = c->d_tab + 2 * q;
  c->T.xo = c->d_tab + 2 * q + q * q;
  c->T.wo = c->T.xo + no;
  c->T.sqb = c->T.wo + no;
  c->T.xd = c->T.sqb + 41 * 41;
  c->T.wd = c->T.xd + kNDirect;
  c->T.xdp = c->T.wd + kNDirect;
  c->T.hc = c->T.xdp + kNDirect * q;
  {
    const std::vector<double> &tt = make_trtab_p(p.p);
    if (cudaMalloc(&c->d_trtab, tt.size() * sizeof(double)) == cudaSuccess)
      cudaMemcpy(c->d_trtab, tt.data(), tt.size() * sizeof(double), cudaMemcpyHostToDevice);
  }
  // dynamic shared-memory opt-ins of this p's kernels, on this context's device (per device, per context:
  // no process-global state, so contexts on several devices or host threads do not race)
  if (set_kernel_attributes(p.p, p.n_omega) != cudaSuccess) {
    g_create_err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(cudaGetLastError());
    rrq_destroy(c);
    return RRQ_ERR_CUDA;
  }
  if (cuda_check(c, "rrq_create") != RRQ_OK) {
    g_create_err = c->err;
    rrq_destroy(c);
    return RRQ_ERR_CUDA;
  }
  *out = c;
  return RRQ_OK;
}

void rrq_destroy(rrq_ctx c) {
  if (!c) return;
  t_flush(c);
  for (auto e : c->pool) cudaEventDestroy(e);
  if (c->swapcnt.p) cudaFree(c->swapcnt.p);
  if (c->hmap) cudaFreeHost(c->hmap);
  cudaFree(c->d_tab);
  if (c->d_trtab) cudaFree(c->d_trtab);
  if (c->st2) cudaStreamDestroy(c->st2);
  for (cudaEvent_t e : {c->ev_edge[0], c->ev_edge[1], c->ev_free[0], c->ev_free[1], c->ev_fork, c->ev_join})
    if (e) cudaEventDestroy(e);
  for (auto *b : {&c->Arow[0], &c->Arow[1], &c->Xrow[0], &c->Xrow[1], &c->psetup[0], &c->psetup[1], &c->et0[0], &c->et0[1], &c->om[0], &c->om[1], &c->cpair[0],
                  &c->cpair[1], &c->Qrow, &c->ipatch, &c->balls, &c->cell_cnt, &c->cell_items, &c->patch_cell, &c->tcnt, &c->ptgt, &c->perm, &c->seg,
                  &c->cursor, &c->items, &c->Z, &c->fitwork, &c->one})
    if (b->p) cudaFree(b->p);
  delete c;
}

const char *rrq_last_error(rrq_ctx c) { return c ? c->err.c_str() : g_create_err.c_str(); }

int64_t rrq_launch_count(rrq_ctx c) { return c ? c->launches : 0; }

rrq_status rrq_debug_zeta(rrq_ctx c, int64_t max_pairs, int64_t *perm, double *Z, int64_t *n_out) {
  if (!c || !n_out) return RRQ_ERR_INVALID_ARG;
  cudaDeviceSynchronize();
  int64_t n = std::min(max_pairs, c->last_np);
  if (perm && n > 0) cudaMemcpy(perm, bp<int64_t>(c->perm) + c->last_sA, n * sizeof(int64_t), cudaMemcpyDeviceToHost);
  if (Z && n > 0) {   // gather the rows out of k_contract's tile-chunked layout
    double *tmp = nullptr;
    if (cudaMalloc(&tmp, (size_t)n * c->last_nz * sizeof(double)) != cudaSuccess) return fail(c, RRQ_ERR_CUDA, "debug buffer");
    const PairSetup *su = bp<PairSetup>(c->psetup[c->last_set]);
    const double *zb = bp<double>(c->Z);
    const unsigned g = nblk(n * c->last_nz, 256);
    switch (c->prm.p) {
      case 4: k_debug_zeta<4><<<g, 256>>>(n, su, zb, tmp); break;
      case 6: k_debug_zeta<6><<<g, 256>>>(n, su, zb, tmp); break;
      case 8: k_debug_zeta<8><<<g, 256>>>(n, su, zb, tmp); break;
      case 10: k_debug_zeta<10><<<g, 256>>>(n, su, zb, tmp); break;
      case 12: k_debug_zeta<12><<<g, 256>>>(n, su, zb, tmp); break;
      default: k_debug_zeta<14><<<g, 256>>>(n, su, zb, tmp); break;
    }
    cudaMemcpy(Z, tmp, (size_t)n * c->last_nz * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(tmp);
  }
  *n_out = n;
  return cuda_check(c, "rrq_debug_zeta");
}

rrq_status rrq_debug_phase_cycles(rrq_ctx c, uint64_t out[8], int reset) {
  if (!c) return RRQ_ERR_INVALID_ARG;
  cudaDeviceSynchronize();
  if (out) cudaMemcpyFromSymbol(out, g_phase_cycles, 8 * sizeof(uint64_t));
  if (reset) {
    uint64_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  }
  return cuda_check(c, "rrq_debug_phase_cycles");
}

rrq_status rrq_debug_fit_cycles(rrq_ctx c, uint64_t out[8], int reset) {
  if (!c) return RRQ_ERR_INVALID_ARG;
  cudaDeviceSynchronize();
  if (out) cudaMemcpyFromSymbol(out, g_phase_cycles, 8 * sizeof(uint64_t), 8 * sizeof(uint64_t));
  if (reset) {
    uint64_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z), 8 * sizeof(uint64_t));
  }
  return cuda_check(c, "rrq_debug_fit_cycles");
}

rrq_status rrq_set_timing(rrq_ctx c, int enable) {
  if (!c) return RRQ_ERR_INVALID_ARG;
  c->timing = enable != 0;
  return RRQ_OK;
}

rrq_status rrq_set_overlap(rrq_ctx c, int enable) {
  if (!c) return RRQ_ERR_INVALID_ARG;
  c->overlap = enable != 0;
  return RRQ_OK;
}

rrq_status rrq_reset_timing(rrq_ctx c) {
  if (!c) return RRQ_ERR_INVALID_ARG;
  t_flush(c);
  for (int i = 0; i < RRQ_NSTAGES; ++i) { c->t_ms[i] = 0; c->t_n[i] = 0; }
  c->stats[0] = c->stats[1] = 0;
  return RRQ_OK;
}

rrq_status rrq_get_timing(rrq_ctx c, double ms[RRQ_NSTAGES], int64_t launches[RRQ_NSTAGES], int64_t stats[2]) {
  if (!c) return RRQ_ERR_INVALID_ARG;
  t_flush(c);
  for (int i = 0; i < RRQ_NSTAGES; ++i) {
    if (ms) ms[i] = c->t_ms[i];
    if (launches) launches[i] = c->t_n[i];
  }
  if (stats) { stats[0] = c->stats[0]; stats[1] = c->stats[1]; }
  return RRQ_OK;
}

rrq_status rrq_get_tables(rrq_ctx c, double *t, double *w, double *U) {
  if (!c) return RRQ_ERR_INVALID_ARG;
  if (t) std::copy(c->h_t.begin(), c->h_t.end(), t);
  if (w) std::copy(c->h_w.begin(), c->h_w.end(), w);
  if (U) std::copy(c->h_U.begin(), c->h_U.end(), U);
  return RRQ_OK;
}

static rrq_status check_surface(rrq_ctx c, const rrq_surface *s) {
  if (!s) return fail(c, RRQ_ERR_INVALID_ARG, "surface is NULL");
  if (s->n_patches <= 0) return fail(c, RRQ_ERR_INVALID_ARG, "n_patches must be > 0");
  if (s->n_patches > (int64_t)INT32_MAX / c->prm.n_nodes) return fail(c, RRQ_ERR_CAPACITY, "too many nodes for int32 col_idx");
  if (!s->nodes || !s->normals || !s->weights || !s->verts || !s->edge_x || !s->edge_dx)
    return fail(c, RRQ_ERR_INVALID_ARG, "surface arrays must be non-NULL device pointers");
  return RRQ_OK;
}

static rrq_status check_targets(rrq_ctx c, const rrq_targets *t) {
  if (!t) return fail(c, RRQ_ERR_INVALID_ARG, "targets is NULL");
  if (t->n_targets < 0) return fail(c, RRQ_ERR_INVALID_ARG, "n_targets < 0");
  if (t->n_targets > 0 && !t->x) return fail(c, RRQ_ERR_INVALID_ARG, "targets x is NULL");
  return RRQ_OK;
}

static rrq_status compute_balls(rrq_ctx c, const rrq_surface *s, cudaStream_t st) {
  if (!ensure(c, c->balls, s->n_patches * 5 * sizeof(double))) return RRQ_ERR_CUDA;
  k_patch_balls<<<nblk(s->n_patches, 128), 128, 0, st>>>(s->n_patches, c->prm.n_nodes, c->prm.p_edge, s->nodes,
                                                       s->weights, s->verts, s->edge_x, bp<double>(c->balls));
  c->launches++;
  return cuda_check(c, "k_patch_balls");
}

rrq_status rrq_near_list(rrq_ctx c, const rrq_surface *s, const rrq_targets *tg, int64_t *pair_ptr,
                         int32_t *pair_patch, int64_t *n_pairs, rrq_stream_t stream) {
  if (!c) return RRQ_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  rrq_status r;
  if ((r = check_device(c)) || (r = check_surface(c, s)) || (r = check_targets(c, tg))) return r;
  if (!pair_ptr || !n_pairs) return fail(c, RRQ_ERR_INVALID_ARG, "pair_ptr and n_pairs must be non-NULL");
  const int64_t T = tg->n_targets, Pn = s->n_patches;
  const int fill = pair_patch != nullptr;
  TScope ts(c, 0, st);
  if (T == 0) {
    if (!fill) {
      cudaMemsetAsync(pair_ptr, 0, sizeof(int64_t), st);
      *n_pairs = 0;
    }
    return cuda_check(c, "rrq_near_list");
  }
  if (c->prm.all_pairs) {
    if (!fill) {
      k_near_all<<<nblk(T, 256), 256, 0, st>>>(T, Pn, 0, pair_ptr, nullptr);
      if (!ensure(c, c->one, 64)) return RRQ_ERR_CUDA;
      k_scan_i64<<<1, 1024, 0, st>>>(T + 1, pair_ptr, bp<int64_t>(c->one));
      c->launches += 2;
      cudaMemcpyAsync(n_pairs, bp<int64_t>(c->one), sizeof(int64_t), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
    } else {
      k_near_all<<<nblk(T, 256), 256, 0, st>>>(T, Pn, 1, pair_ptr, pair_patch);
      c->launches++;
    }
    return cuda_check(c, "rrq_near_list(all)");
  }
  if ((r = compute_balls(c, s, st))) return r;
  std::vector<double> hb(Pn * 5);
  cudaMemcpyAsync(hb.data(), c->balls.p, Pn * 5 * sizeof(double), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300}, rmax = 0;
  for (int64_t P = 0; P < Pn; ++P) {
    for (int a = 0; a < 3; ++a) { lo[a] = std::min(lo[a], hb[P * 5 + a]); hi[a] = std::max(hi[a], hb[P * 5 + a]); }
    rmax = std::max(rmax, hb[P * 5 + 3] + c->prm.eta * hb[P * 5 + 4]);
  }
  Grid g;
  double cell = std::max(rmax, 1e-300);
  for (;;) {
    int64_t tot = 1;
    for (int a = 0; a < 3; ++a) {
      g.lo[a] = lo[a] - cell;
      g.dim[a] = (int)std::max<int64_t>(1, (int64_t)std::ceil((hi[a] - lo[a] + 2 * cell) / cell));
      tot *= g.dim[a];
    }
    if (tot <= (1 << 22)) break;
    cell *= 1.26;
  }
  g.inv_cell = 1.0 / cell;
  const int ncell = g.dim[0] * g.dim[1] * g.dim[2];
  if (!ensure(c, c->cell_cnt, (ncell + 1) * sizeof(int32_t)) || !ensure(c, c->cell_items, Pn * sizeof(int32_t)) ||
      !ensure(c, c->patch_cell, Pn * sizeof(int32_t)) || !ensure(c, c->cursor, (ncell + 1) * sizeof(int32_t)) ||
      !ensure(c, c->one, 64))
    return RRQ_ERR_CUDA;
  cudaMemsetAsync(c->cell_cnt.p, 0, (ncell + 1) * sizeof(int32_t), st);
  k_cell_count<<<nblk(Pn, 256), 256, 0, st>>>(Pn, bp<double>(c->balls), g, bp<int32_t>(c->cell_cnt), bp<int32_t>(c->patch_cell));
  k_scan_i32<<<1, 1024, 0, st>>>(ncell + 1, bp<int32_t>(c->cell_cnt), bp<int32_t>(c->one));
  cudaMemcpyAsync(c->cursor.p, c->cell_cnt.p, (ncell + 1) * sizeof(int32_t), cudaMemcpyDeviceToDevice, st);
  k_cell_fill<<<nblk(Pn, 256), 256, 0, st>>>(Pn, bp<int32_t>(c->patch_cell), bp<int32_t>(c->cursor), bp<int32_t>(c->cell_items));
  c->launches += 3;
  if (!fill) {
    k_near_targets<<<nblk(T, 128), 128, 0, st>>>(T, tg->x, tg->self_node, c->prm.n_nodes, bp<double>(c->balls),
                                                 c->prm.eta, g, bp<int32_t>(c->cell_cnt), bp<int32_t>(c->cell_items), 0,
                                                 pair_ptr, nullptr);
    cudaMemsetAsync(pair_ptr + T, 0, sizeof(int64_t), st);
    k_scan_i64<<<1, 1024, 0, st>>>(T + 1, pair_ptr, bp<int64_t>(c->one));
    c->launches += 2;
    cudaMemcpyAsync(n_pairs, c->one.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
  } else {
    k_near_targets<<<nblk(T, 128), 128, 0, st>>>(T, tg->x, tg->self_node, c->prm.n_nodes, bp<double>(c->balls),
                                                 c->prm.eta, g, bp<int32_t>(c->cell_cnt), bp<int32_t>(c->cell_items), 1,
                                                 pair_ptr, pair_patch);
    c->launches++;
  }
  return cuda_check(c, "rrq_near_list");
}

template <int P>
static size_t stride_bytes() { return (size_t)Layout<P>::STRIDE * sizeof(double); }

size_t rrq_fit_bytes(rrq_ctx c, int64_t n_patches) {
  if (!c || n_patches <= 0) return 0;
  size_t s = 0;
  switch (c->prm.p) {
    case 4: s = stride_bytes<4>(); break;
    case 6: s = stride_bytes<6>(); break;
    case 8: s = stride_bytes<8>(); break;
    case 10: s = stride_bytes<10>(); break;
    case 12: s = stride_bytes<12>(); break;
    case 14: s = stride_bytes<14>(); break;
  }
  return s * (size_t)n_patches;
}

template <int P>
static rrq_status patch_fit_impl(rrq_ctx c, const rrq_surface *s, double *fit, int32_t *status, cudaStream_t st) {
  using D = Dims<P>;
  const int64_t Pn = s->n_patches;
  rrq_status r;
  TScope ts(c, 1, st);
  if ((r = compute_balls(c, s, st))) return r;
  k_patch_geom<P><<<(unsigned)Pn, 128, 0, st>>>(Pn, s->nodes, s->verts, s->edge_x, s->edge_dx, bp<double>(c->balls), c->T, fit);
  {
    using EC = EdgeTabCfg<P>;
    k_edge_tables<P><<<(unsigned)Pn, EC::THREADS, EC::SMEM, st>>>(Pn, c->T.hc, c->d_trtab + TrCfg<P>::VLAM,
                                                                  c->d_trtab + TrCfg<P>::VTH, fit);
  }
  c->launches += 2;
  if ((r = cuda_check(c, "k_patch_geom/k_edge_tables"))) return r;
  using FC = FitCfg<P>;
  int grid = (int)std::min<int64_t>(Pn, 2 * c->num_sms);
  if (!ensure(c, c->fitwork, (size_t)grid * FC::WS * sizeof(double))) return RRQ_ERR_CUDA;
  k_patch_fit_q<P><<<grid, 256, FC::SMEM, st>>>(Pn, s->nodes, s->normals, c->T.hc, fit, bp<double>(c->fitwork), status);
  c->launches++;
  return cuda_check(c, "k_patch_fit");
}

rrq_status rrq_patch_fit(rrq_ctx c, const rrq_surface *s, void *fit, int32_t *patch_status, rrq_stream_t stream) {
  if (!c) return RRQ_ERR_INVALID_ARG;
  rrq_status r;
  if ((r = check_device(c)) || (r = check_surface(c, s))) return r;
  if (!fit) return fail(c, RRQ_ERR_INVALID_ARG, "fit is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  switch (c->prm.p) {
    case 4: return patch_fit_impl<4>(c, s, (double *)fit, patch_status, st);
    case 6: return patch_fit_impl<6>(c, s, (double *)fit, patch_status, st);
    case 8: return patch_fit_impl<8>(c, s, (double *)fit, patch_status, st);
    case 10: return patch_fit_impl<10>(c, s, (double *)fit, patch_status, st);
    case 12: return patch_fit_impl<12>(c, s, (double *)fit, patch_status, st);
    case 14: return patch_fit_impl<14>(c, s, (double *)fit, patch_status, st);
  }
  return RRQ_ERR_NOT_IMPLEMENTED;
}

template <int P>
static size_t edge_smem(int n_omega) {
  using D = Dims<P>;
  using EC = EdgeCfg<P>;
  int tab = D::Q * D::Q + 2 * D::Q + 2 * n_omega + kNDirect * D::Q + EC::WPB * 2 * kNDirect;
  tab = (tab + 1) & ~1;
  return (size_t)tab * sizeof(double) + EC::WPB * EC::PPW * sizeof(EdgePair<P>);
}

template <int P>
static rrq_status build_impl(rrq_ctx c, const rrq_surface *s, const rrq_targets *tg, const int64_t *pair_ptr,
                             const int32_t *pair_patch, int64_t row_begin, int64_t row_end, const double *fit,
                             uint32_t mask, int64_t *row_ptr, int32_t *col_idx, double *const vals[4], int32_t *pstat,
                             cudaStream_t st) {
  using D = Dims<P>;
  using QC = QmapCfg<P>;
  using CC = ContractCfg<P>;
  constexpr int TP = QC::TP;
  static_assert(QC::TP == CC::TP, "k_qmap and k_contract share the work items");
  const int64_t Pn = s->n_patches;
  const int raw = (mask & RRQ_RAW) ? 1 : 0;
  const int want_dp = (mask & RRQ_DP) ? 1 : 0;   // kernel mask: the dQ rows and the dW translation only for D
  if (!ensure_hmap(c, 2 * (size_t)(Pn + 2))) return RRQ_ERR_CUDA;
  k_pair_range<<<1, 32, 0, st>>>(pair_ptr, row_begin, row_end, c->hmap);
  c->launches++;
  {   // the mapped pair range is only valid once the kernel ran: check before consuming it
    rrq_status r0 = cuda_check(c, "k_pair_range");
    if (r0) return r0;
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(c, RRQ_ERR_CUDA, std::string("k_pair_range: ") + cudaGetErrorString(e));
  }
  const int64_t obase = c->hmap[0], total = c->hmap[1] - c->hmap[0];
  if (total == 0) {
    if (row_ptr) {
      k_row_ptr<<<nblk(row_end - row_begin + 1, 256), 256, 0, st>>>(row_begin, row_end, pair_ptr, obase, row_ptr, D::N);
      c->launches++;
    }
    return cuda_check(c, "rrq_build_correction");
  }
  if (c->timing) {
    if (!ensure(c, c->swapcnt, 64)) return RRQ_ERR_CUDA;
    cudaMemsetAsync(c->swapcnt.p, 0, 8, st);
  }
  if (!ensure(c, c->ptgt, total * sizeof(int64_t)) || !ensure(c, c->perm, total * sizeof(int64_t)) ||
      !ensure(c, c->seg, (Pn + 1) * sizeof(int64_t)) || !ensure(c, c->cursor, (Pn + 1) * sizeof(int64_t)) ||
      !ensure(c, c->items, (Pn + 1) * sizeof(int64_t)) || !ensure(c, c->ipatch, (total / TP + Pn + 1) * sizeof(int32_t)) ||
      !ensure(c, c->one, 64))
    return RRQ_ERR_CUDA;
  // ---- plumbing over the whole call: pair -> target, patch-major permutation, work items
  std::vector<int64_t> hseg(Pn + 1), hitem(Pn + 1);
  TScope tbuild(c, 7, st);   // the whole call (device time on the caller's stream)
  {
    TScope tsp(c, 6, st);
    k_pair_targets<<<nblk(row_end - row_begin + 1, 256), 256, 0, st>>>(row_begin, row_end, pair_ptr, obase,
                                                                       bp<int64_t>(c->ptgt), nullptr, D::N);
    cudaMemsetAsync(c->seg.p, 0, (Pn + 1) * sizeof(int64_t), st);
    k_patch_hist<<<nblk(total, 256), 256, 0, st>>>(total, obase, pair_patch, bp<int64_t>(c->seg));
    k_scan_i64<<<1, 1024, 0, st>>>(Pn + 1, bp<int64_t>(c->seg), bp<int64_t>(c->one));
    cudaMemcpyAsync(c->cursor.p, c->seg.p, (Pn + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, st);
    k_patch_scatter<<<nblk(total, 256), 256, 0, st>>>(total, obase, pair_patch, bp<int64_t>(c->cursor),
                                                      bp<int64_t>(c->perm));
    k_items<<<nblk(Pn, 256), 256, 0, st>>>(Pn, bp<int64_t>(c->seg), TP, bp<int64_t>(c->items));
    cudaMemsetAsync(bp<int64_t>(c->items) + Pn, 0, sizeof(int64_t), st);
    k_scan_i64<<<1, 1024, 0, st>>>(Pn + 1, bp<int64_t>(c->items), bp<int64_t>(c->one) + 1);
    k_item_patch<<<nblk(Pn, 256), 256, 0, st>>>(Pn, bp<int64_t>(c->items), bp<int32_t>(c->ipatch));
    k_copy_i64<<<nblk(Pn + 1, 256), 256, 0, st>>>(Pn + 1, bp<int64_t>(c->seg), c->hmap);
    k_copy_i64<<<nblk(Pn + 1, 256), 256, 0, st>>>(Pn + 1, bp<int64_t>(c->items), c->hmap + Pn + 1);
    c->launches += 9;
  }
  {
    rrq_status r0 = cuda_check(c, "build plumbing");
    if (r0) return r0;
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(c, RRQ_ERR_CUDA, std::string("build plumbing: ") + cudaGetErrorString(e));
  }
  std::memcpy(hseg.data(), c->hmap, (Pn + 1) * sizeof(int64_t));
  std::memcpy(hitem.data(), c->hmap + Pn + 1, (Pn + 1) * sizeof(int64_t));
  hseg[Pn] = total;
  // ---- sub-chunks: ranges of whole patches with at most `cap` pairs (scratch ~24 KB per pair at p = 8:
  // the double-buffered producer outputs plus the Q and Z rows)
  const int64_t per_pair = (int64_t)(2 * (2 * D::K + XRow<P>::STRIDE) + QRow<P>::STRIDE + CC::ZBLK / CC::TP) * 8 +
                           2 * (int64_t)(sizeof(PairSetup) + sizeof(ContractPair) + 3 * (sizeof(double2) + 1) + 8 * sizeof(double));
  const int64_t cap = std::max<int64_t>(2 * TP, (int64_t)(c->scratch_bytes / per_pair));
  // sub-chunks = contiguous ranges of work items (tiles of TP pairs of one patch): whole patches while they
  // fit, a patch with more than `cap` pairs (config 5: one patch, 10M targets) split at tile boundaries
  struct Sub { int64_t it0, it1, sA, sB; };
  std::vector<Sub> subs;
  int64_t maxsub = 0, maxitems = 0;
  {
    const int64_t capI = std::max<int64_t>(1, cap / TP);
    int64_t cur_it0 = -1, cur_sA = 0;
    auto flush = [&](int64_t it1, int64_t sB) {
      if (cur_it0 >= 0 && sB > cur_sA) subs.push_back({cur_it0, it1, cur_sA, sB});
      cur_it0 = -1;
    };
    for (int64_t P0 = 0; P0 < Pn; ++P0) {
      const int64_t np0 = hseg[P0 + 1] - hseg[P0];
      if (np0 == 0) continue;
      if (cur_it0 >= 0 && hseg[P0 + 1] - cur_sA > cap) flush(hitem[P0], hseg[P0]);
      if (np0 > cap) {
        for (int64_t it = hitem[P0]; it < hitem[P0 + 1]; it += capI) {
          const int64_t ie = std::min(it + capI, hitem[P0 + 1]);
          subs.push_back({it, ie, hseg[P0] + (it - hitem[P0]) * TP,
                          ie == hitem[P0 + 1] ? hseg[P0 + 1] : hseg[P0] + (ie - hitem[P0]) * TP});
        }
        continue;
      }
      if (cur_it0 < 0) { cur_it0 = hitem[P0]; cur_sA = hseg[P0]; }
    }
    flush(hitem[Pn], hseg[Pn]);
    for (const Sub &u : subs) {
      maxsub = std::max(maxsub, u.sB - u.sA);
      maxitems = std::max(maxitems, u.it1 - u.it0);
    }
  }
  const int nset = (c->overlap && subs.size() > 1) ? 2 : 1;
  for (int b = 0; b < nset; ++b)
    if (!ensure(c, c->Arow[b], (size_t)maxitems * QC::ABLK * 8) || !ensure(c, c->Xrow[b], (size_t)maxsub * XRow<P>::STRIDE * 8) ||
        !ensure(c, c->psetup[b], (size_t)maxsub * sizeof(PairSetup)) ||
        !ensure(c, c->cpair[b], (size_t)maxsub * sizeof(ContractPair)) ||
        !ensure(c, c->om[b], (size_t)maxsub * 8 * sizeof(double)) ||   // k_edge_lines: scalar line integrals
        !ensure(c, c->et0[b], (size_t)maxsub * 3 * (sizeof(double2) + 1) + 64))   // k_newton: t0 + flag byte per edge, batch counter
      return RRQ_ERR_CUDA;
  const void *z_before = c->Z.p;
  if (!ensure(c, c->Qrow, (size_t)maxsub * QRow<P>::STRIDE * 8) || !ensure(c, c->Z, (size_t)maxitems * CC::ZBLK * 8))
    return RRQ_ERR_CUDA;
  if (CC::KPAD && c->Z.p != z_before) cudaMemsetAsync(c->Z.p, 0, c->Z.n, st);   // the padded k-entries stay zero
  // producer stream: a second stream when overlapping, else the caller's
  cudaStream_t sp = st;
  if (nset == 2) {
    if (!c->st2) {
      if (cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking) != cudaSuccess)
        return fail(c, RRQ_ERR_CUDA, "stream creation failed");
      for (cudaEvent_t *e : {&c->ev_edge[0], &c->ev_edge[1], &c->ev_free[0], &c->ev_free[1], &c->ev_fork, &c->ev_join})
        cudaEventCreateWithFlags(e, cudaEventDisableTiming);
    }
    sp = c->st2;
    cudaEventRecord(c->ev_fork, st);   // the producer sees the plumbing above (perm, items, ...)
    cudaStreamWaitEvent(sp, c->ev_fork, 0);
  }
  rrq_status r;
  for (size_t i = 0; i < subs.size(); ++i) {
    const Sub &sr = subs[i];
    const int b = (int)(i % nset);
    const int64_t sA = sr.sA, sB = sr.sB, it0 = sr.it0, it1 = sr.it1;
    const int64_t np_ = sB - sA;
    double *Ar = bp<double>(c->Arow[b]), *Xr = bp<double>(c->Xrow[b]);
    PairSetup *ps = bp<PairSetup>(c->psetup[b]);
    ContractPair *cp = bp<ContractPair>(c->cpair[b]);
    // ---- producer: Steps 4-5 (+ scalar line integrals, gamma parts) into set b
    if (nset == 2 && i >= 2) cudaStreamWaitEvent(sp, c->ev_free[b], 0);   // sub-chunk i-2 is done with set b
    {
      TScope t1(c, 2, sp);
      k_pair_setup<P><<<nblk(np_, 256), 256, 0, sp>>>(sA, sB, bp<int64_t>(c->perm), bp<int64_t>(c->ptgt), obase,
                                                       pair_patch, fit, tg->x, tg->normal, tg->self_node, tg->side,
                                                       bp<int64_t>(c->seg), bp<int64_t>(c->items), it0, ps, cp);
      double2 *T0 = bp<double2>(c->et0[b]);
      uint8_t *EF = reinterpret_cast<uint8_t *>(T0 + 3 * np_);
      {
        TScope t8(c, 8, sp);
        unsigned long long *ctr = reinterpret_cast<unsigned long long *>(EF + ((3 * np_ + 15) / 16) * 16);
        cudaMemsetAsync(ctr, 0, 8, sp);
        // persistent warps drawing batches of 32 edges; 4 CTAs of 4 warps per SM
        const unsigned gn = (unsigned)std::min<int64_t>(nblk(3 * np_, kNewtonThreads), (int64_t)c->num_sms * 4);
        k_newton<P><<<gn, kNewtonThreads, 0, sp>>>(np_, ps, fit, c->prm.rho_swap, T0, EF, ctr);
      }
      double *OMb = bp<double>(c->om[b]);
      {
        TScope t9(c, 9, sp);
        using EC = EdgeCfg<P>;
        constexpr int PR = EC::WPB * EC::PPW;   // pairs per CTA round
        unsigned grid = (unsigned)std::min<int64_t>((np_ + PR - 1) / PR, (int64_t)c->num_sms * EC::MINB * 2);
        k_edge_lines<P><<<grid, EC::WPB * 32, edge_smem<P>(c->prm.n_omega), sp>>>(
            sA, sB, fit, c->T, c->prm.n_omega, Ar, OMb, pstat, obase,
            c->timing ? bp<unsigned long long>(c->swapcnt) : nullptr, ps, want_dp, T0, EF);
      }
      {
        TScope t10(c, 10, sp);
        using TC = TgtCfg<P>;
        constexpr int PR = TC::WPB * TC::PPW;
        unsigned grid = (unsigned)std::min<int64_t>((np_ + PR - 1) / PR, (int64_t)c->num_sms * TC::MINB * 2);
        k_target_gamma<P><<<grid, TC::WPB * 32, TC::SMEM, sp>>>(sA, sB, c->T, Xr, OMb, c->d_trtab, ps, want_dp);
      }
    }
    if ((r = cuda_check(c, "k_edge_lines / k_target_gamma"))) return r;
    if (nset == 2) {
      cudaEventRecord(c->ev_edge[b], sp);
      cudaStreamWaitEvent(st, c->ev_edge[b], 0);
    }
    // ---- consumer: Steps 6-8
    {
      TScope t2(c, 3, st);
      auto *kq = want_dp ? k_qmap<P, true> : k_qmap<P, false>;
      kq<<<(unsigned)(it1 - it0), QC::WARPS * 32, QC::SMEM, st>>>(it0, it1, bp<int64_t>(c->items), bp<int32_t>(c->ipatch),
                                                                 bp<int64_t>(c->seg), sA, fit, Ar, bp<double>(c->Qrow), c->d_trtab);
    }
    if ((r = cuda_check(c, "k_qmap"))) return r;
    {
      TScope t3(c, 4, st);
      constexpr int WPB = TrCfg<P>::WPB;
      unsigned grid = (unsigned)std::min<int64_t>((np_ + WPB - 1) / WPB, (int64_t)c->num_sms);
      auto *kt = want_dp ? k_translate<P, true> : k_translate<P, false>;
      kt<<<grid, WPB * 32, TrCfg<P>::SMEM, st>>>(sA, sB, Xr, bp<double>(c->Qrow), c->d_trtab, bp<double>(c->Z), mask);
    }
    if ((r = cuda_check(c, "k_translate"))) return r;
    {
      TScope t4(c, 5, st);
      const uint32_t km = mask & RRQ_ALL;
      auto *kc = km == RRQ_ALL ? k_contract<P, 15> : km == (RRQ_S | RRQ_D) ? k_contract<P, 3> : k_contract<P, 0>;
      kc<<<(unsigned)(it1 - it0), CC::WARPS * 32, CC::SMEM, st>>>(
          it0, it1, bp<int64_t>(c->items), bp<int32_t>(c->ipatch), bp<int64_t>(c->seg), sA, cp,
          fit, bp<double>(c->Z), s->nodes, s->normals, s->weights, mask, raw, obase, col_idx, vals[0], vals[1], vals[2],
          vals[3], pstat);
    }
    if ((r = cuda_check(c, "k_contract"))) return r;
    if (nset == 2) cudaEventRecord(c->ev_free[b], st);
    c->launches += 7;
    c->last_sA = sA;
    c->last_np = np_;
    c->last_set = b;
  }
  if (nset == 2) {   // join the producer stream
    cudaEventRecord(c->ev_join, sp);
    cudaStreamWaitEvent(st, c->ev_join, 0);
  }
  if (row_ptr) {
    k_row_ptr<<<nblk(row_end - row_begin + 1, 256), 256, 0, st>>>(row_begin, row_end, pair_ptr, obase, row_ptr, D::N);
    c->launches++;
  }
  c->last_nz = D::NZ;
  if (c->timing) {
    unsigned long long sw = 0;
    cudaMemcpyAsync(&sw, c->swapcnt.p, 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    c->stats[0] += total;
    c->stats[1] += (int64_t)sw;
  }
  return cuda_check(c, "rrq_build_correction");
}

rrq_status rrq_build_correction(rrq_ctx c, const rrq_surface *s, const rrq_targets *tg, const int64_t *pair_ptr,
                                const int32_t *pair_patch, int64_t n_pairs, int64_t row_begin, int64_t row_end,
                                const void *fit, uint32_t mask, int64_t *row_ptr, int32_t *col_idx,
                                double *const vals[4], int32_t *pstat, rrq_stream_t stream) {
  if (!c) return RRQ_ERR_INVALID_ARG;
  rrq_status r;
  if ((r = check_device(c)) || (r = check_surface(c, s)) || (r = check_targets(c, tg))) return r;
  if (!pair_ptr || (!pair_patch && n_pairs > 0) || !fit || !vals)
    return fail(c, RRQ_ERR_INVALID_ARG, "pair_ptr, pair_patch (unless n_pairs == 0), fit, vals must be non-NULL");
  if (row_begin < 0 || row_end < row_begin || row_end > tg->n_targets)
    return fail(c, RRQ_ERR_INVALID_ARG, "row range must satisfy 0 <= row_begin <= row_end <= n_targets");
  if (n_pairs < 0) return fail(c, RRQ_ERR_INVALID_ARG, "n_pairs < 0");
  if ((mask & (RRQ_SP | RRQ_DP)) && !tg->normal) return fail(c, RRQ_ERR_INVALID_ARG, "S' and D' need target normals");
  if ((mask & RRQ_ALL) == 0) return fail(c, RRQ_ERR_INVALID_ARG, "kernel_mask selects no kernel");
  {   // the contraction stores weight pairs with 16-B (8-B index) stores and stages the patch's nodes by bulk copies
    auto al = [](const void *q, uintptr_t a) { return q == nullptr || ((uintptr_t)q % a) == 0; };
    if (!al(s->nodes, 16) || !al(s->normals, 16) || !al(s->weights, 16) || !al(col_idx, 8) || !al(vals[0], 16) ||
        !al(vals[1], 16) || !al(vals[2], 16) || !al(vals[3], 16))
      return fail(c, RRQ_ERR_INVALID_ARG, "nodes/normals/weights/vals must be 16-byte aligned, col_idx 8-byte aligned");
  }
  if (row_end == row_begin) return RRQ_OK;
  cudaStream_t st = (cudaStream_t)stream;
  switch (c->prm.p) {
    case 4: return build_impl<4>(c, s, tg, pair_ptr, pair_patch, row_begin, row_end, (const double *)fit, mask, row_ptr, col_idx, vals, pstat, st);
    case 6: return build_impl<6>(c, s, tg, pair_ptr, pair_patch, row_begin, row_end, (const double *)fit, mask, row_ptr, col_idx, vals, pstat, st);
    case 8: return build_impl<8>(c, s, tg, pair_ptr, pair_patch, row_begin, row_end, (const double *)fit, mask, row_ptr, col_idx, vals, pstat, st);
    case 10: return build_impl<10>(c, s, tg, pair_ptr, pair_patch, row_begin, row_end, (const double *)fit, mask, row_ptr, col_idx, vals, pstat, st);
    case 12: return build_impl<12>(c, s, tg, pair_ptr, pair_patch, row_begin, row_end, (const double *)fit, mask, row_ptr, col_idx, vals, pstat, st);
    case 14: return build_impl<14>(c, s, tg, pair_ptr, pair_patch, row_begin, row_end, (const double *)fit, mask, row_ptr, col_idx, vals, pstat, st);
  }
  return RRQ_ERR_NOT_IMPLEMENTED;
}

rrq_status rrq_apply_smooth(rrq_ctx c, int64_t n_targets, const double *tx, const int64_t *self_node,
                            const rrq_surface *s, double alpha, double beta, const double *density, double *y,
                            rrq_stream_t stream) {
  if (!c) return RRQ_ERR_INVALID_ARG;
  rrq_status r;
  if ((r = check_device(c)) || (r = check_surface(c, s))) return r;
  if (n_targets < 0) return fail(c, RRQ_ERR_INVALID_ARG, "n_targets < 0");
  if (n_targets == 0) return RRQ_OK;
  if (!tx || !density || !y) return fail(c, RRQ_ERR_INVALID_ARG, "NULL array");
  const int64_t ns = s->n_patches * (int64_t)c->prm.n_nodes;
  k_smooth_apply<<<nblk(n_targets, 256), 256, 0, (cudaStream_t)stream>>>(n_targets, tx, self_node, ns, s->nodes,
                                                                          s->normals, s->weights, density, alpha,
                                                                          beta, y);
  c->launches++;
  return cuda_check(c, "rrq_apply_smooth");
}

rrq_status rrq_apply_correction(rrq_ctx c, int64_t n_rows, const int64_t *row_ptr, const int32_t *col_idx,
                                const double *vals, const double *density, double *y, rrq_stream_t stream) {
  if (!c) return RRQ_ERR_INVALID_ARG;
  if (check_device(c)) return RRQ_ERR_INVALID_ARG;
  if (n_rows < 0) return fail(c, RRQ_ERR_INVALID_ARG, "n_rows < 0");
  if (n_rows == 0) return RRQ_OK;
  if (!row_ptr || !col_idx || !vals || !density || !y) return fail(c, RRQ_ERR_INVALID_ARG, "NULL array");
  k_apply<<<nblk(n_rows * 32, 256), 256, 0, (cudaStream_t)stream>>>(n_rows, row_ptr, col_idx, vals, density, y);
  c->launches++;
  return cuda_check(c, "rrq_apply_correction");
}


// Dynamic shared memory limit of one kernel (the carveout is left to the driver: forcing the maximum costs
// k_qmap 3 % through the smaller L1); RRQ_DEBUG_OCC=1 prints the resulting CTAs per SM.
template <typename K>
static cudaError_t set_smem(K *kern, const char *name, size_t smem, int threads) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess && std::getenv("RRQ_DEBUG_OCC")) {
    int nb = -1;
    cudaFuncAttributes fa{};
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem);
    cudaFuncGetAttributes(&fa, kern);
    std::fprintf(stderr, "rrq: %-22s %4d threads %7zu B smem %3d regs -> %d CTAs/SM\n", name, threads, smem, fa.numRegs, nb);
  }
  return e;
}

template <int P>
static cudaError_t set_attrs(int n_omega) {
  cudaError_t e = cudaSuccess;
  auto acc = [&](cudaError_t x) { if (e == cudaSuccess) e = x; };
  acc(set_smem(k_edge_tables<P>, "k_edge_tables", EdgeTabCfg<P>::SMEM, EdgeTabCfg<P>::THREADS));
  acc(set_smem(k_patch_fit_q<P>, "k_patch_fit_q", FitCfg<P>::SMEM, 256));
  acc(set_smem(k_edge_lines<P>, "k_edge_lines", edge_smem<P>(n_omega), EdgeCfg<P>::WPB * 32));
  acc(set_smem(k_target_gamma<P>, "k_target_gamma", TgtCfg<P>::SMEM, TgtCfg<P>::WPB * 32));
  acc(set_smem(k_qmap<P, true>, "k_qmap<dp>", QmapCfg<P>::SMEM, QmapCfg<P>::WARPS * 32));
  acc(set_smem(k_qmap<P, false>, "k_qmap", QmapCfg<P>::SMEM, QmapCfg<P>::WARPS * 32));
  acc(set_smem(k_translate<P, true>, "k_translate<dp>", TrCfg<P>::SMEM, TrCfg<P>::WPB * 32));
  acc(set_smem(k_translate<P, false>, "k_translate", TrCfg<P>::SMEM, TrCfg<P>::WPB * 32));
  acc(set_smem(k_contract<P, 15>, "k_contract<15>", ContractCfg<P>::SMEM, ContractCfg<P>::WARPS * 32));
  acc(set_smem(k_contract<P, 3>, "k_contract<3>", ContractCfg<P>::SMEM, ContractCfg<P>::WARPS * 32));
  acc(set_smem(k_contract<P, 0>, "k_contract<0>", ContractCfg<P>::SMEM, ContractCfg<P>::WARPS * 32));
  if (std::getenv("RRQ_DEBUG_OCC")) {
    int nb = -1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_newton<P>, kNewtonThreads, 0);
    std::fprintf(stderr, "rrq: %-22s -> %d CTAs/SM\n", "k_newton", nb);
  }
  return e;
}

static cudaError_t set_kernel_attributes(int p, int n_omega) {
  switch (p) {
    case 4: return set_attrs<4>(n_omega);
    case 6: return set_attrs<6>(n_omega);
    case 8: return set_attrs<8>(n_omega);
    case 10: return set_attrs<10>(n_omega);
    case 12: return set_attrs<12>(n_omega);
    case 14: return set_attrs<14>(n_omega);
  }
  return cudaErrorInvalidValue;
}
