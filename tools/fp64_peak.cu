// FP64 DFMA throughput microbenchmark (roofline denominator for the ALU-bound axis passes).
// Burst: one ~50 ms launch; sustained: back-to-back launches for >= 4 s. Reports TFLOP/s (DFMA = 2 flop).
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
__global__ void dfma_kernel(double *out, int iters, double s) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999, c = s;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  double r = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (r == 12345.678) out[0] = r;
}
int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  double *out; CK(cudaMalloc(&out, 8));
  const int threads = 256, blocks = p.multiProcessorCount * 8; const int iters = 2000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) dfma_kernel<<<blocks, threads>>>(out, iters, 1e-9);
  CK(cudaDeviceSynchronize());
  double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
  float best = 1e30f;
  for (int rep = 0; rep < 10; ++rep) {
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters, 1e-9); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  printf("{\"fp64_tflops_burst\": %.3f, \"burst_ms\": %.3f, ", flops / best / 1e9, best);
  int nl = 0; cudaEventRecord(e0);
  float ms = 0;
  while (ms < 5000.f) { for (int k = 0; k < 20; ++k) { dfma_kernel<<<blocks, threads>>>(out, iters, 1e-9); ++nl; }
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); }
  printf("\"fp64_tflops_sustained\": %.3f, \"sustained_s\": %.2f, \"sms\": %d}\n", flops * nl / ms / 1e9, ms / 1e3, p.multiProcessorCount);
  return 0;
}
