// Microbenchmark: TMEM <-> register throughput with tcgen05.ld / tcgen05.st (32x32b shape, x32 columns),
// one CTA per SM of WARPS warps, each warp streaming its own 32-column slice of its lane quadrant.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a tools/tmem_probe.cu -o tools/tmem_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int WARPS, bool LOAD>
__global__ void __launch_bounds__(WARPS * 32, 1) probe(unsigned *out, int iters) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&taddr_s)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = taddr_s;
  // lane quadrant of this warp (warp % 4), column slice (warp / 4) * 32 .. + 32
  const uint32_t ta = base + ((uint32_t)(32 * (warp % 4)) << 16) + (uint32_t)((warp / 4) * 32 % 512);
  unsigned r[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) r[i] = threadIdx.x * 7 + i;
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
    if (LOAD) {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
          "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
            "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
            "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(ta));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc += r[it & 31];
    } else {
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
          "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
          "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
          "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
          "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
          : "memory");
      r[it & 31] += 1;
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + r[5];
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(512));
}

template <int WARPS, bool LOAD>
void run(int iters) {
  unsigned *d;
  cudaMalloc(&d, 148 * WARPS * 32 * 4);
  probe<WARPS, LOAD><<<148, WARPS * 32>>>(d, 10);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<WARPS, LOAD><<<148, WARPS * 32>>>(d, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double bytes = 148.0 * WARPS * 32 * 32 * 4.0 * iters;  // per SM: warps x 32 lanes x 32 cols x 4 B
  double cyc = ms * 1e-3 * 1.965e9;
  printf("%s warps=%2d  %.3f ms  %.1f B/clk/SM  err=%s\n", LOAD ? "tcgen05.ld" : "tcgen05.st", WARPS, ms,
         bytes / 148.0 / cyc, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<4, true>(20000);
  run<8, true>(20000);
  run<16, true>(20000);
  run<4, false>(20000);
  run<8, false>(20000);
  run<16, false>(20000);
  return 0;
}
