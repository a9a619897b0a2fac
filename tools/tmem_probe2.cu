// TMEM -> register throughput with several tcgen05.ld in flight before one wait::ld (x16 shape), per-SM B/clk.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1901_07275_b200/csrc/tmem.cuh"
using namespace jtk;

template <int WARPS, int INFLIGHT>
__global__ void __launch_bounds__(WARPS * 32, 1) probe(unsigned *out, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&slot, 512);
  tmem_fence_before_sync();
  __syncthreads();
  tmem_fence_after_sync();
  const uint32_t base = slot;
  const int cols = 512 / (WARPS / 4);
  const uint32_t ta = base + ((uint32_t)(32 * (warp % 4)) << 16) + (uint32_t)((warp / 4) * cols);
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint32_t r[INFLIGHT][16];
#pragma unroll
    for (int j = 0; j < INFLIGHT; ++j) tmem_ld16(ta + (uint32_t)((16 * j) % cols), r[j]);
    tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < INFLIGHT; ++j) acc += r[j][0] ^ r[j][15] ^ r[j][7];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tmem_fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc(base, 512);
}

template <int WARPS, int INFLIGHT>
void run(int iters) {
  unsigned *d;
  cudaMalloc(&d, 148 * WARPS * 32 * 4);
  probe<WARPS, INFLIGHT><<<148, WARPS * 32>>>(d, 10);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<WARPS, INFLIGHT><<<148, WARPS * 32>>>(d, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double bytes = 148.0 * WARPS * 32 * 16 * 4.0 * INFLIGHT * iters;
  printf("warps=%2d inflight=%d  %.3f ms  %.1f B/clk/SM  %s\n", WARPS, INFLIGHT, ms, bytes / 148.0 / (ms * 1e-3 * 1.965e9),
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<8, 1>(20000);
  run<8, 2>(20000);
  run<8, 4>(10000);
  run<8, 8>(5000);
  run<16, 4>(10000);
  return 0;
}
