// FP64 peak microbenchmarks for the roofline denominator ("measure it on the box").
// dfma: independent FMA chains on the FP64 CUDA-core pipe.  dmma: mma.sync m8n8k4 f64 (DMMA).
#include <cstdio>
#include <cuda_runtime.h>
#define CHAINS 8
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0; for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}
__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double acc[4][2];
  for (int c = 0; c < 4; ++c) { acc[c][0] = 0; acc[c][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int c = 0; c < 4; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[0] = s;
}
// mixed: even warps run DFMA chains, odd warps run DMMA; if the two units are separate the combined
// rate approaches the sum of the two peaks, if they share one pipe it stays near the larger one.
__global__ void mixed_kernel(double* out, int iters_f, int iters_m, double a, double b) {
  if ((threadIdx.x >> 5) & 1) {
    double ma = threadIdx.x * 1e-3, mb = 1.0 + threadIdx.x * 1e-4;
    double acc[4][2];
    for (int c = 0; c < 4; ++c) { acc[c][0] = 0; acc[c][1] = 0; }
    for (int i = 0; i < iters_m; ++i) {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(ma), "d"(mb));
    }
    double s = 0; for (int c = 0; c < 4; ++c) s += acc[c][0] + acc[c][1];
    if (s == 12345.678) out[0] = s;
  } else {
    double x[CHAINS];
    for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < iters_f; ++i) {
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0; for (int c = 0; c < CHAINS; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;
  }
}
int main() {
  int dev = 0; cudaDeviceProp pr; cudaGetDeviceProperties(&pr, dev);
  int sms = pr.multiProcessorCount;
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int bpsm = 1; bpsm <= 8; bpsm *= 2) {
    int threads = 256, blocks = sms * bpsm, iters = 20000;
    dfma_kernel<<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * CHAINS * (double)iters * threads * blocks;
    printf("{\"kernel\":\"dfma\",\"blocks_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n", bpsm, ms, flops / ms / 1e9);
  }
  for (int bpsm = 1; bpsm <= 8; bpsm *= 2) {
    int threads = 256, blocks = sms * bpsm, iters = 20000;
    dmma_kernel<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 4.0 * (double)iters * (threads / 32) * blocks;
    printf("{\"kernel\":\"dmma\",\"blocks_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n", bpsm, ms, flops / ms / 1e9);
  }
  for (int ratio = 1; ratio <= 8; ratio *= 2) {   // DFMA iterations per DMMA iteration
    int threads = 256, blocks = sms * 4, iters_m = 10000, iters_f = iters_m * ratio;
    mixed_kernel<<<blocks, threads>>>(out, 100, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    mixed_kernel<<<blocks, threads>>>(out, iters_f, iters_m, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ff = 2.0 * CHAINS * (double)iters_f * (threads / 2) * blocks;
    double fm = 2.0 * 8 * 8 * 4 * 4.0 * (double)iters_m * (threads / 64) * blocks;
    printf("{\"kernel\":\"mixed\",\"dfma_per_dmma_iter\":%d,\"ms\":%.3f,\"dfma_tflops\":%.3f,\"dmma_tflops\":%.3f,\"sum_tflops\":%.3f}\n",
           ratio, ms, ff / ms / 1e9, fm / ms / 1e9, (ff + fm) / ms / 1e9);
  }
  printf("err=%s sms=%d clock_khz=%d\n", cudaGetErrorString(cudaGetLastError()), sms, pr.clockRate);
  return 0;
}
