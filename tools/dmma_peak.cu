// FP64 tensor-core (DMMA, mma.sync .f64) throughput probe on sm_100a, alone and concurrently with DFMA.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void mma884(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma16816(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}
// mode 0: DMMA m8n8k4 only; 1: DFMA only; 2: half warps DMMA, half DFMA; 3: m16n8k16
__global__ void k(double *out, int iters, int mode) {
  int w = threadIdx.x / 32;
  double a = threadIdx.x * 1e-3, b = 1.0 - a;
  double acc[8][2];
  for (int i = 0; i < 8; ++i) { acc[i][0] = i; acc[i][1] = -i; }
  double f[8]; for (int i = 0; i < 8; ++i) f[i] = a + i;
  bool do_mma = (mode == 0) || (mode == 2 && (w & 1) == 0);
  bool do_fma = (mode == 1) || (mode == 2 && (w & 1) == 1);
  if (mode == 3) {
    double d[4][4] = {}; double A[8], B[4];
    for (int i = 0; i < 8; ++i) A[i] = a + i; for (int i = 0; i < 4; ++i) B[i] = b - i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int u = 0; u < 4; ++u) mma16816(d[u], A, B);
    double s = 0; for (int u = 0; u < 4; ++u) for (int i = 0; i < 4; ++i) s += d[u][i];
    if (s == 1234.5) out[0] = s;
    return;
  }
  for (int it = 0; it < iters; ++it) {
    if (do_mma) {
#pragma unroll
      for (int u = 0; u < 8; ++u) mma884(acc[u][0], acc[u][1], a, b);
    }
    if (do_fma) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = fma(f[i], 0.999999, 1e-9);
    }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1] + f[i];
  if (s == 1234.5) out[0] = s;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double *out; cudaMalloc(&out, 8);
  int blocks = p.multiProcessorCount * 4, threads = 256, iters = 4000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char *names[4] = {"dmma_m8n8k4", "dfma", "mixed(half warps each)", "dmma_m16n8k16"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int w = 0; w < 2; ++w) k<<<blocks, threads>>>(out, iters, mode);
    cudaEventRecord(e0); k<<<blocks, threads>>>(out, iters, mode); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double warps = blocks * threads / 32.0;
    double flop_mma = 0, flop_fma = 0;
    if (mode == 0) flop_mma = warps * iters * 8 * 512.0;
    if (mode == 1) flop_fma = warps * iters * 32 * 32 * 2.0;
    if (mode == 2) { flop_mma = warps / 2 * iters * 8 * 512.0; flop_fma = warps / 2 * iters * 32 * 32 * 2.0; }
    if (mode == 3) flop_mma = warps * iters * 4 * 16 * 8 * 16 * 2.0;
    printf("%-24s %.3f ms  mma %.2f TF  fma %.2f TF  total %.2f TF  err=%s\n", names[mode], ms, flop_mma / ms / 1e9,
           flop_fma / ms / 1e9, (flop_mma + flop_fma) / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
}
