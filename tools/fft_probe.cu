// Microbenchmark: FP64 pipe utilisation of the in-register DFT building blocks alone (no SMEM, no
// syncs), at the axis kernel's occupancy (THREADS per CTA, one CTA per SM, 255 registers).
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_1901_07275_b200/csrc tools/fft_probe.cu -o tools/fft_probe
#include <cstdio>
#include <cuda_runtime.h>
#include "fft_regs.cuh"
using namespace jtk;

template <int M, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) probe(double *out, int iters, double seed) {
  double xr[32], xi[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) { xr[i] = seed * (i + threadIdx.x); xi[i] = seed * (i - (int)threadIdx.x); }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int b = 0; b < 32 / M; ++b) dft<M>(&xr[b * M], &xi[b * M]);
#pragma unroll
    for (int i = 0; i < 32; ++i) { xr[i] *= 0.03125; xi[i] *= 0.03125; }   // keep values bounded
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += xr[i] + xi[i];
  out[blockIdx.x * THREADS + threadIdx.x] = s;
}

template <int M, int THREADS>
void run(int iters) {
  double *d;
  cudaMalloc(&d, 148 * THREADS * 8);
  probe<M, THREADS><<<148, THREADS>>>(d, iters, 1e-3);
  cudaDeviceSynchronize();
  cudaFree(d);
}

// Run under ncu: --metrics sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum
int main() {
  run<32, 256>(2000);
  run<16, 256>(2000);
  run<32, 384>(2000);
  run<16, 384>(2000);
  run<16, 512>(2000);
  run<8, 256>(2000);
  printf("done\n");
  return 0;
}
