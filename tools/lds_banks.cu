// Micro-benchmark: shared-memory wavefronts of one LDS.128 per lane for several address patterns
// (read with ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum).
#include <cstdio>
__global__ void k(int pat, double *out) {
  __shared__ __align__(16) double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
  __syncthreads();
  const int l = threadIdx.x & 31;
  int c;   // 16-byte chunk index
  switch (pat) {
    case 0: c = l; break;                              // contiguous 512 B
    case 1: c = 9 * l; break;                          // stride 144 B
    case 2: c = 9 * (l % 8) + 64 * (l / 8); break;     // quarters: stride 9, same groups across quarters
    case 3: c = 8 * l; break;                          // all lanes same 16-B group
    case 4: c = (l / 8) + 8 * (l % 8); break;          // quarter: same group; quarters differ
    case 5: c = (l % 8) + 64 * (l / 8); break;         // quarter contiguous 128 B, quarters in other rows
    case 6: c = 9 * (l % 16) + 200 * (l / 16); break;  // half-warps stride 9
    case 7: c = (l % 4) * 8 + (l / 4); break;          // lane%4 -> row, lane/4 -> group (fragment-like)
    default: c = (l * 5) % 32 * 9; break;
  }
  double acc = 0;
  for (int it = 0; it < 1000; ++it) {
    const double2 v = *reinterpret_cast<const double2 *>(sm + 2 * ((c + it * 0) & 2047));
    acc += v.x + v.y;
    __syncwarp();
  }
  if (acc == -1) out[0] = acc;
}
int main() {
  double *o;
  cudaMalloc(&o, 8);
  for (int p = 0; p < 9; ++p) { k<<<1, 32>>>(p, o); cudaDeviceSynchronize(); }
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
}
