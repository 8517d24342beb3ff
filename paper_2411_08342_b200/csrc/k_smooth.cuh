// The smooth rule of the splitting D = D_smooth + D_RRQ applied to a density: the far part of
// the layer-potential operators that the correction matrix completes.  For each target t
//   y_t += alpha * sum_j w_j sigma_j / (4 pi |t - x_j|)  +  beta * sum_j w_j sigma_j (t - x_j).n_j / (4 pi |t - x_j|^3)
// over all surface nodes j except the target's own node (self_node, reading A14) -- the same smooth
// terms k_contract subtracts, so smooth + correction = the RRQ operator on near pairs and the plain rule
// elsewhere.  FMM is out of scope: a direct sum, O(N_T N_S).
// Thread per target, CTA-wide source tiles in shared memory (x, n, w sigma), 4 independent accumulators.
#pragma once
#include "rrq_device.cuh"

namespace rrq {

constexpr int kSmoothTile = 256;

__global__ void __launch_bounds__(256) k_smooth_apply(int64_t n_targets, const double *__restrict__ tx,
                                                      const int64_t *__restrict__ self_node, int64_t n_src,
                                                      const double *__restrict__ sx, const double *__restrict__ sn,
                                                      const double *__restrict__ sw, const double *__restrict__ sigma,
                                                      double alpha, double beta, double *__restrict__ y) {
  __shared__ double4 sp[kSmoothTile];   // x, y, z, w sigma
  __shared__ double4 snrm[kSmoothTile]; // n (w sigma in .w unused)
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool act = t < n_targets;
  double p0 = 0, p1 = 0, p2 = 0;
  int64_t self = -1;
  if (act) {
    p0 = tx[3 * t]; p1 = tx[3 * t + 1]; p2 = tx[3 * t + 2];
    if (self_node) self = self_node[t];
  }
  double as0 = 0, as1 = 0, ad0 = 0, ad1 = 0;
  for (int64_t j0 = 0; j0 < n_src; j0 += kSmoothTile) {
    __syncthreads();
    for (int i = threadIdx.x; i < kSmoothTile; i += blockDim.x) {
      const int64_t j = j0 + i;
      if (j < n_src) {
        sp[i] = make_double4(sx[3 * j], sx[3 * j + 1], sx[3 * j + 2], sw[j] * sigma[j]);
        snrm[i] = make_double4(sn[3 * j], sn[3 * j + 1], sn[3 * j + 2], 0.0);
      } else {
        sp[i] = make_double4(1e150, 0.0, 0.0, 0.0);   // far away (finite r^2), zero weight
        snrm[i] = make_double4(0.0, 0.0, 0.0, 0.0);
      }
    }
    __syncthreads();
    if (!act) continue;
    const int64_t sl = self - j0;   // the self node inside this tile, if any
#pragma unroll 4
    for (int i = 0; i < kSmoothTile; i += 2) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double4 s = sp[i + h], nn = snrm[i + h];
        const double d0 = p0 - s.x, d1 = p1 - s.y, d2 = p2 - s.z;
        const double r2 = d0 * d0 + d1 * d1 + d2 * d2;
        double ir = rsqrt_nr(r2);
        if (i + h == sl || !(r2 > 0)) ir = 0.0;
        const double ws = s.w * ir;
        const double dn = (d0 * nn.x + d1 * nn.y + d2 * nn.z) * ir * ir;
        if (h == 0) { as0 += ws; ad0 += ws * dn; } else { as1 += ws; ad1 += ws * dn; }
      }
    }
  }
  if (act) y[t] += (alpha * (as0 + as1) + beta * (ad0 + ad1)) * (1.0 / (4.0 * kPi));
}

}  // namespace rrq
