// L1 / SMEM data-pipe probe (dev tool): cycles per warp-instruction per SM for the access patterns the
// axis kernels use.  Every kernel runs 148*8 CTAs x 256 threads, ITER loads per thread, with the loaded
// data folded into a result so nothing is dead.  Reported: ns per launch and SM-cycles per warp-instr.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITER = 4096;
constexpr int TBL = 2048;  // double2 entries = 32 KB (L1 resident)

template <int MODE>
__global__ void __launch_bounds__(256) probe(const double2 *__restrict__ tbl, double *out, int salt) {
  __shared__ double2 sm[TBL];
  for (int i = threadIdx.x; i < TBL; i += blockDim.x) sm[i] = tbl[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double ax = 0, ay = 0;
  int base = (w * 64 + salt) & (TBL - 1);
#pragma unroll 8
  for (int it = 0; it < ITER; ++it) {
    int idx;
    if (MODE == 0 || MODE == 1) idx = lane;            // 32 distinct consecutive
    else if (MODE == 2 || MODE == 3) idx = lane >> 2;  // 8 distinct consecutive (4 lanes each)
    else if (MODE == 4) idx = 0;                       // uniform
    else if (MODE == 5) idx = lane >> 1;               // 16 distinct
    else idx = lane;
    idx = (idx + base + it * 37) & (TBL - 1);
    double2 v;
    if (MODE == 0 || MODE == 2) v = sm[idx];
    else if (MODE == 6) { v.x = __shfl_sync(0xffffffffu, ax, (lane + it) & 31); v.y = __shfl_sync(0xffffffffu, ay, (lane + 3) & 31); }
    else v = __ldg(&tbl[idx]);
    ax += v.x;
    ay += v.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = ax + ay;
}

template <int MODE>
void run(const char *name, const double2 *tbl, double *out) {
  const int grid = 148 * 8;
  probe<MODE><<<grid, 256>>>(tbl, out, 1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) probe<MODE><<<grid, 256>>>(tbl, out, r);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 5;
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double warp_instr_per_sm = (double)grid * 8 * ITER / 148.0;
  const double cyc = ms * 1e-3 * clk * 1e3;
  printf("%-34s %8.3f ms  %6.2f SM-cycles per warp-instr\n", name, ms, cyc / warp_instr_per_sm);
}

int main() {
  double2 *tbl;
  double *out;
  cudaMalloc(&tbl, TBL * sizeof(double2));
  cudaMemset(tbl, 0, TBL * sizeof(double2));
  cudaMalloc(&out, 148 * 8 * 256 * sizeof(double));
  run<0>("LDS.128 32 distinct", tbl, out);
  run<2>("LDS.128 8 distinct", tbl, out);
  run<1>("LDG.128 32 distinct (L1 hit)", tbl, out);
  run<3>("LDG.128 8 distinct (L1 hit)", tbl, out);
  run<5>("LDG.128 16 distinct (L1 hit)", tbl, out);
  run<4>("LDG.128 uniform (L1 hit)", tbl, out);
  run<6>("SHFL x2 (64-bit pair)", tbl, out);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
