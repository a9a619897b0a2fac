// Probe: can tcgen05.cp (SMEM -> TMEM) replicate an 8-row core matrix down the 32 lanes of a quadrant with a
// zero stride-dimension byte offset (SBO = 0), and what do .32x128b.warpx4 / .64x128b.warpx2::02_13 write where?
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tmem_cp_probe tools/tmem_cp_probe.cu && tools/tmem_cp_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // fixed 0b001 (sm100 descriptor version)
  return d;               // base offset 0, LBO mode 0, swizzle none
}

template <int MODE>
__global__ void probe(uint32_t *out, uint32_t sbo) {
  __shared__ __align__(128) uint32_t sm[1024];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 0x10000u + i;  // word i of row i/4
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tslot;
  // zero the 32 columns of every lane first (each warp its quadrant)
  {
    const uint32_t ta = tbase + ((uint32_t)(32 * (threadIdx.x / 32)) << 16);
    uint32_t z[4] = {0, 0, 0, 0};
    for (int c = 0; c < 32; c += 4)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(ta + c), "r"(z[0]), "r"(z[1]),
                   "r"(z[2]), "r"(z[3]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    const uint64_t d = sdesc((uint32_t)__cvta_generic_to_shared(sm), 0, sbo);
    if (MODE == 0) asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(tbase), "l"(d) : "memory");
    else if (MODE == 1) asm volatile("tcgen05.cp.cta_group::1.64x128b.warpx2::02_13 [%0], %1;" ::"r"(tbase), "l"(d) : "memory");
    else asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(tbase), "l"(d) : "memory");
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
  }
  {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok) : "r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t ta = tbase + ((uint32_t)(32 * (threadIdx.x / 32)) << 16);
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(ta));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int i = 0; i < 4; ++i) out[threadIdx.x * 4 + i] = r[i];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tbase) : "memory");
}

int main() {
  uint32_t *d, h[128 * 4];
  cudaMalloc(&d, sizeof(h));
  const char *names[3] = {"32x128b.warpx4", "64x128b.warpx2::02_13", "128x128b"};
  for (int mode = 0; mode < 3; ++mode)
    for (uint32_t sbo : {128u, 0u, 256u}) {
      cudaMemset(d, 0xff, sizeof(h));
      if (mode == 0) probe<0><<<1, 128>>>(d, sbo);
      else if (mode == 1) probe<1><<<1, 128>>>(d, sbo);
      else probe<2><<<1, 128>>>(d, sbo);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("%s SBO=%u (%s): lane -> source row (word0 - 0x10000) / 4:\n ", names[mode], sbo, cudaGetErrorString(e));
      for (int lane = 0; lane < 128; ++lane) {
        const uint32_t w = h[lane * 4];
        if (w == 0) printf(" .");
        else printf(" %d", (int)(w - 0x10000u) / 4);
        if (lane % 32 == 31) printf("\n ");
      }
      printf("\n");
      if (e != cudaSuccess) return 1;
    }
  return 0;
}
