// Shared-memory wavefronts per warp instruction for the access patterns of the axis kernels (run under ncu
// with l1tex__data_pipe_lsu_wavefronts_mem_shared.sum and smsp__inst_executed_op_shared_ld.sum).
#include <cstdio>
#include <cuda_runtime.h>

template <int BYTES, int DISTINCT>
__global__ void probe(double *out, int iters) {
  __shared__ __align__(128) double s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int idx = (lane % DISTINCT);  // DISTINCT distinct elements, consecutive
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    const int base = (it * 64) & 2047;
    if (BYTES == 8) {
      acc += s[base + idx];
    } else {
      const double2 v = reinterpret_cast<const double2 *>(s)[(base >> 1) + idx];
      acc += v.x * v.y;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  double *d;
  cudaMalloc(&d, 148 * 256 * 8);
  probe<8, 32><<<148, 256>>>(d, 1000);
  probe<8, 8><<<148, 256>>>(d, 1000);
  probe<8, 1><<<148, 256>>>(d, 1000);
  probe<16, 32><<<148, 256>>>(d, 1000);
  probe<16, 8><<<148, 256>>>(d, 1000);
  probe<16, 4><<<148, 256>>>(d, 1000);
  probe<16, 1><<<148, 256>>>(d, 1000);
  cudaDeviceSynchronize();
  printf("done\n");
  return 0;
}
