// Near list (reading A6; "adaptive octree or k-d tree ... omit the details"): a uniform
// cell grid over the patch-ball centres with cell size >= the largest query radius R_P + eta h_P,
// so a target only visits the 27 cells around it.  Count pass -> exclusive scan -> fill pass ->
// per-target insertion sort (patches ascending, deterministic).
#pragma once
#include "rrq_device.cuh"

namespace rrq {

struct Grid {
  double lo[3], inv_cell;
  int dim[3];
};

__device__ __forceinline__ int cell_coord(double x, double lo, double inv, int dim) {
  int c = (int)floor((x - lo) * inv);
  return c < 0 ? 0 : (c >= dim ? dim - 1 : c);
}

__global__ void k_cell_count(int64_t n_patches, const double *__restrict__ balls, Grid g, int32_t *__restrict__ cell_cnt,
                             int32_t *__restrict__ patch_cell) {
  int64_t P = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (P >= n_patches) return;
  const double *b = balls + P * 5;
  int cx = cell_coord(b[0], g.lo[0], g.inv_cell, g.dim[0]);
  int cy = cell_coord(b[1], g.lo[1], g.inv_cell, g.dim[1]);
  int cz = cell_coord(b[2], g.lo[2], g.inv_cell, g.dim[2]);
  int c = (cz * g.dim[1] + cy) * g.dim[0] + cx;
  patch_cell[P] = c;
  atomicAdd(cell_cnt + c, 1);
}

__global__ void k_cell_fill(int64_t n_patches, const int32_t *__restrict__ patch_cell, int32_t *__restrict__ cursor,
                            int32_t *__restrict__ cell_items) {
  int64_t P = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (P >= n_patches) return;
  int pos = atomicAdd(cursor + patch_cell[P], 1);
  cell_items[pos] = (int32_t)P;
}

// Pass 0: counts into cnt[t]; pass 1: fill pair_patch[pair_ptr[t] ...] and sort the segment.
__global__ void k_near_targets(int64_t n_targets, const double *__restrict__ tx, const int64_t *__restrict__ self_node,
                               int n, const double *__restrict__ balls, double eta, Grid g,
                               const int32_t *__restrict__ cell_start, const int32_t *__restrict__ cell_items,
                               int fill, int64_t *__restrict__ cnt_or_ptr, int32_t *__restrict__ pair_patch) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_targets) return;
  double x[3] = {tx[3 * t], tx[3 * t + 1], tx[3 * t + 2]};
  int64_t selfP = (self_node && self_node[t] >= 0) ? self_node[t] / n : -1;
  int cx = cell_coord(x[0], g.lo[0], g.inv_cell, g.dim[0]);
  int cy = cell_coord(x[1], g.lo[1], g.inv_cell, g.dim[1]);
  int cz = cell_coord(x[2], g.lo[2], g.inv_cell, g.dim[2]);
  int64_t base = fill ? cnt_or_ptr[t] : 0, k = base;
  bool self_found = false;
  for (int dz = -1; dz <= 1; ++dz) {
    int z = cz + dz;
    if (z < 0 || z >= g.dim[2]) continue;
    for (int dy = -1; dy <= 1; ++dy) {
      int y = cy + dy;
      if (y < 0 || y >= g.dim[1]) continue;
      for (int dx = -1; dx <= 1; ++dx) {
        int xx = cx + dx;
        if (xx < 0 || xx >= g.dim[0]) continue;
        int c = (z * g.dim[1] + y) * g.dim[0] + xx;
        for (int it = cell_start[c]; it < cell_start[c + 1]; ++it) {
          int P = cell_items[it];
          const double *b = balls + (int64_t)P * 5;
          // the A6 test in the oracle's arithmetic (k_patch_balls: separately rounded IEEE operations)
          bool near = norm3_rn(__dsub_rn(x[0], b[0]), __dsub_rn(x[1], b[1]), __dsub_rn(x[2], b[2])) <=
                      __dadd_rn(b[3], __dmul_rn(eta, b[4]));
          if (P == selfP) { near = true; self_found = true; }
          if (near) {
            if (fill) pair_patch[k] = P;
            ++k;
          }
        }
      }
    }
  }
  if (selfP >= 0 && !self_found) {   // the self patch is always near (cannot happen for sane inputs)
    if (fill) pair_patch[k] = (int32_t)selfP;
    ++k;
  }
  if (!fill) {
    cnt_or_ptr[t] = k;
    return;
  }
  // insertion sort of the segment (patches ascending)
  for (int64_t i = base + 1; i < k; ++i) {
    int32_t v = pair_patch[i];
    int64_t j = i - 1;
    while (j >= base && pair_patch[j] > v) { pair_patch[j + 1] = pair_patch[j]; --j; }
    pair_patch[j + 1] = v;
  }
}

__global__ void k_near_all(int64_t n_targets, int64_t n_patches, int fill, int64_t *__restrict__ cnt_or_ptr,
                           int32_t *__restrict__ pair_patch) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_targets) return;
  if (!fill) { cnt_or_ptr[t] = n_patches; return; }
  int64_t b = cnt_or_ptr[t];
  for (int64_t P = 0; P < n_patches; ++P) pair_patch[b + P] = (int32_t)P;
}

// Exclusive scan of int64 counts in place (single CTA, chunked; n up to ~1e8 in a few ms).
__global__ void k_scan_i64(int64_t n, int64_t *__restrict__ a, int64_t *__restrict__ total) {
  __shared__ int64_t sh[1024];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < n; base += 1024) {
    int64_t i = base + threadIdx.x;
    int64_t v = i < n ? a[i] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      int64_t w = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
      __syncthreads();
      sh[threadIdx.x] += w;
      __syncthreads();
    }
    if (i < n) a[i] = carry + sh[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += sh[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void k_scan_i32(int n, int32_t *__restrict__ a, int32_t *__restrict__ total) {
  __shared__ int32_t sh[1024];
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < n; base += 1024) {
    int i = base + threadIdx.x;
    int32_t v = i < n ? a[i] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      int32_t w = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
      __syncthreads();
      sh[threadIdx.x] += w;
      __syncthreads();
    }
    if (i < n) a[i] = carry + sh[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += sh[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

}  // namespace rrq
