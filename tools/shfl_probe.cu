// Throughput of warp shuffles vs shared-memory loads per SM (do SHFLs share the L1/SMEM data pipe's 128 B/clk?).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/shfl_probe tools/shfl_probe.cu && tools/shfl_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_shfl(double *out, int iters) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __shfl_xor_sync(0xffffffffu, a[i], 1 + (i & 3)) + 1.0;  // 2 SHFL.32 per double
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_lds(double *out, int iters) {
  __shared__ __align__(16) double2 sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_double2(i, i);
  __syncthreads();
  double s = 0;
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {  // LDS.128, 32 distinct consecutive 16 B addresses = 4 wavefronts
      const double2 v = sm[((it * 8 + i) * 32 + lane) & 2047];
      s += v.x;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_mix(double *out, int iters) {  // half SHFL, half LDS: do they overlap (separate pipes)?
  __shared__ __align__(16) double2 sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_double2(i, i);
  __syncthreads();
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
  double s = 0;
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      a[i] = __shfl_xor_sync(0xffffffffu, a[i], 1 + (i & 3)) + 1.0;
      const double2 v = sm[((it * 8 + i) * 32 + lane) & 2047];
      s += v.x;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double *d;
  cudaMalloc(&d, 148 * 1024 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096, nt = 1024;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int rep = 0; rep < 2; ++rep) {
    for (int which = 0; which < 3; ++which) {
      cudaEventRecord(e0);
      if (which == 0) k_shfl<<<148, nt>>>(d, iters);
      else if (which == 1) k_lds<<<148, nt>>>(d, iters);
      else k_mix<<<148, nt>>>(d, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      // per SM: (nt / 32) warps x iters x 8 ops (SHFL: x2 instructions per double)
      const double warp_ops = (double)(nt / 32) * iters * 8;
      const double cyc = ms * 1e-3 * 1.965e9;
      const char *nm[3] = {"shfl (2 SHFL.32 per op)", "lds.128 (4 wavefronts)", "mix: 1 shfl-op + 1 lds.128"};
      printf("%-28s %.3f ms  %.2f SM-cycles per warp-op\n", nm[which], ms, cyc / warp_ops);
    }
  }
  return 0;
}
