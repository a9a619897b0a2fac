// Fused axis-pass kernels (K4 forward, K5 inverse).
//
// One CTA owns a tile of LINES complete lines along the transformed axis (lines are the paper's
// "n^{d-1} 1D transforms").  For every line it computes, entirely on chip,
//
//   forward (eq:oneJ):   y = W V a_V  +  Re sum_{l<r} D_{u~_l} F_N D_{v_l} a_G
//   inverse (eq:oneJinv): a_V = (W V)^T y,  a_G = Re sum_{l<r} D_{v_l} F_N^T D_{u~_l} y
//
// with one HBM read and one HBM write of the line per axis pass; the r rank terms are batched in one
// pass (north star: "batches several rank terms per pass to cut HBM round trips").
//
// Per rank term l:
//   forward:  x[k] = v_l[k] a[k]                            (A1: column scale + pack, registers)
//             X = F_N x  (positive exponent)                (A2: Stockham radix-R passes, SMEM exchange)
//             y_j += Re(u~_l[j] X[m_j]) for rows j of bin m  (A3: gather + row scale + Re + accumulate)
//   inverse:  b[m] = sum_{j: m_j = m} u~_l[j] y_j            (bin sums; monotone m_j -> segmented, no atomics)
//             B = F_N b                                      (same sign)
//             a[k] += Re(v_l[k] B[k])
//
// Thread layout: tid = vt * LINES + line.  A thread owns R points of one line ("virtual thread" vt of
// TPL = N / R per line); lanes of a warp that share vt read the same u~, v, twiddle entries.
// Shared memory holds the complex exchange buffer [pos][line] (split re / im planes) and the per-row
// accumulators; the a (forward) or accumulated a (inverse) values live in registers across terms.
#pragma once
#include <cuda_runtime.h>

#include "fft_regs.cuh"

namespace jtk {

struct AxisDev {
  int n;        // axis length
  int N;        // FFT length (power of two >= n)
  int k0;       // dense low-degree block width
  int r;        // rank
  const double2 *u;     // r x n   u~_l[j]     at u[l * n + j]
  const double2 *v;     // r x N   v_l[k]      at v[l * N + k]  (zero for k < k0 and k >= n)
  const double *phiv;   // n x k0  (W V)[j,k]  at phiv[j * k0 + k]
  const int *bstart;    // N/2 + 2 row offsets of the bins (rows of bin m: bstart[m] .. bstart[m+1]-1)
  const double2 *tw;    // N twiddles e^{+2 pi i q / N}
};

template <int N, int R, int LINES>
struct Geo {
  static constexpr int TPL = N / R;               // threads per line
  static constexpr int NT = TPL * LINES;          // threads per CTA
  static constexpr int PADDED = (LINES >= 8);     // [pos][LINES+1] rows, else linear + 1 pad / 16
  static constexpr int LDL = PADDED ? LINES + 1 : LINES;
  static constexpr int BUF = PADDED ? N * LDL : N * LINES + (N * LINES) / 16 + 1;  // doubles per plane
  __device__ static __forceinline__ int sidx(int pos, int line) {
    if constexpr (PADDED) {
      return pos * LDL + line;
    } else {
      int p = pos * LINES + line;
      return p + (p >> 4);
    }
  }
  static constexpr size_t smem_bytes(int k0) {
    // exchange re + im planes, per-row accumulators / y tile (N rows), a_V block (inverse)
    return sizeof(double) * (size_t)(3 * BUF + k0 * LINES + 8);
  }
};

// Radix of the Stockham pass that starts at sub-transform size NS.
template <int N, int R, int NS>
struct Pass {
  static constexpr int RS = (N / NS < R) ? N / NS : R;
  static constexpr int B = R / RS;                // butterflies per thread
  static constexpr bool LAST = (NS * RS == N);
};

// Pass at NS > 1: read R points from the exchange buffer, twiddle, radix-RS butterflies.
template <int N, int R, int LINES, int NS>
__device__ __forceinline__ void pass_load_compute(double (&xr)[R], double (&xi)[R], const double *__restrict__ bre,
                                                  const double *__restrict__ bim, int vt, int line,
                                                  const double2 *__restrict__ tw) {
  using G = Geo<N, R, LINES>;
  using P = Pass<N, R, NS>;
  constexpr int RS = P::RS;
#pragma unroll
  for (int i = 0; i < P::B; ++i) {
    const int v = vt + i * G::TPL;
#pragma unroll
    for (int r = 0; r < RS; ++r) {
      const int pos = v + r * (N / RS);
      xr[i * RS + r] = bre[G::sidx(pos, line)];
      xi[i * RS + r] = bim[G::sidx(pos, line)];
    }
    if constexpr (NS > 1) {
      const int base = (v % NS) * (N / (NS * RS));
#pragma unroll
      for (int r = 1; r < RS; ++r) {
        const double2 w = __ldg(&tw[r * base]);
        const double tr = xr[i * RS + r] * w.x - xi[i * RS + r] * w.y;
        xi[i * RS + r] = fma(xr[i * RS + r], w.y, xi[i * RS + r] * w.x);
        xr[i * RS + r] = tr;
      }
    }
    dft<RS>(&xr[i * RS], &xi[i * RS]);
  }
}

// First pass (NS == 1): the R points are already in registers (input positions vt + r * TPL).
template <int N, int R, int LINES>
__device__ __forceinline__ void pass0_compute(double (&xr)[R], double (&xi)[R]) {
  using P = Pass<N, R, 1>;
#pragma unroll
  for (int i = 0; i < P::B; ++i) dft<P::RS>(&xr[i * P::RS], &xi[i * P::RS]);
}

template <int N, int R, int LINES, int NS>
__device__ __forceinline__ void pass_store(const double (&xr)[R], const double (&xi)[R], double *__restrict__ bre,
                                           double *__restrict__ bim, int vt, int line) {
  using G = Geo<N, R, LINES>;
  using P = Pass<N, R, NS>;
  constexpr int RS = P::RS;
#pragma unroll
  for (int i = 0; i < P::B; ++i) {
    const int v = vt + i * G::TPL;
    const int idxD = (v / NS) * NS * RS + (v % NS);
#pragma unroll
    for (int s = 0; s < RS; ++s) {
      bre[G::sidx(idxD + s * NS, line)] = xr[i * RS + s];
      bim[G::sidx(idxD + s * NS, line)] = xi[i * RS + s];
    }
  }
}

// Runs passes NS, NS*RS, ... to completion.  On entry xr/xi hold the outputs of the pass that ended at
// sub-size NS (still in registers, not yet stored).  On exit they hold the final outputs of the
// last pass, at positions (see out_pos) vt + i TPL + s N / RS_last.
template <int N, int R, int LINES, int NS>
__device__ __forceinline__ void run_passes(double (&xr)[R], double (&xi)[R], double *bre, double *bim, int vt, int line,
                                           const double2 *__restrict__ tw) {
  if constexpr (NS < N) {
    // the previous pass (which ended at sub-size NS) has stored; the pass at NS reads
    pass_load_compute<N, R, LINES, NS>(xr, xi, bre, bim, vt, line, tw);
    if constexpr (!Pass<N, R, NS>::LAST) {
      __syncthreads();
      pass_store<N, R, LINES, NS>(xr, xi, bre, bim, vt, line);
      __syncthreads();
      run_passes<N, R, LINES, NS * Pass<N, R, NS>::RS>(xr, xi, bre, bim, vt, line, tw);
    }
  }
}

// Full FFT of one term whose first-pass inputs are in registers.  Leaves the outputs in registers.
template <int N, int R, int LINES>
__device__ __forceinline__ void fft_term(double (&xr)[R], double (&xi)[R], double *bre, double *bim, int vt, int line,
                                         const double2 *__restrict__ tw) {
  pass0_compute<N, R, LINES>(xr, xi);
  if constexpr (!Pass<N, R, 1>::LAST) {
    pass_store<N, R, LINES, 1>(xr, xi, bre, bim, vt, line);
    __syncthreads();
    run_passes<N, R, LINES, Pass<N, R, 1>::RS>(xr, xi, bre, bim, vt, line, tw);
  }
}

// Last-pass geometry: find the NS at which the last pass starts.
template <int N, int R, int NS = 1>
struct LastPass {
  static constexpr int value = Pass<N, R, NS>::LAST ? NS : LastPass<N, R, NS * Pass<N, R, NS>::RS>::value;
};
template <int N, int R>
struct LastPass<N, R, N> {
  static constexpr int value = N;
};

// Position (frequency index) of output register e = i * RS + s after the last pass.
template <int N, int R, int LINES>
__device__ __forceinline__ int out_pos(int vt, int e) {
  constexpr int NSL = LastPass<N, R>::value;
  constexpr int RS = Pass<N, R, NSL>::RS;
  using G = Geo<N, R, LINES>;
  const int i = e / RS, s = e % RS;
  return vt + i * G::TPL + s * (N / RS);
}

// Global address of element `pos` of tile line `line` (lines are indexed (outer, inner) with inner
// fastest; the transformed axis has stride `inner`).
struct LineAddr {
  long long base;
  __device__ __forceinline__ LineAddr(long long L, long long inner, int n) {
    long long o = L / inner, i = L - o * inner;
    base = o * (long long)n * inner + i;
  }
};

// Copy a tile of LINES lines (n points each) from global to the exchange-layout buffer dst (zero-padding
// positions n..N-1 and lines past the end).
template <int N, int R, int LINES>
__device__ __forceinline__ void load_tile(const double *__restrict__ g, double *dst, long long L0, long long nlines,
                                          long long inner, int n) {
  using G = Geo<N, R, LINES>;
  if (inner == 1) {
    for (int idx = threadIdx.x; idx < LINES * N; idx += G::NT) {
      const int line = idx / N, pos = idx % N;
      const long long L = L0 + line;
      double val = 0.0;
      if (pos < n && L < nlines) val = g[L * n + pos];
      dst[G::sidx(pos, line)] = val;
    }
  } else {
    for (int idx = threadIdx.x; idx < LINES * N; idx += G::NT) {
      const int line = idx % LINES, pos = idx / LINES;
      const long long L = L0 + line;
      double val = 0.0;
      if (pos < n && L < nlines) {
        LineAddr la(L, inner, n);
        val = g[la.base + (long long)pos * inner];
      }
      dst[G::sidx(pos, line)] = val;
    }
  }
}

template <int N, int R, int LINES>
__device__ __forceinline__ void store_tile(double *__restrict__ g, const double *src, long long L0, long long nlines,
                                           long long inner, int n) {
  using G = Geo<N, R, LINES>;
  if (inner == 1) {
    for (int idx = threadIdx.x; idx < LINES * N; idx += G::NT) {
      const int line = idx / N, pos = idx % N;
      const long long L = L0 + line;
      if (pos < n && L < nlines) g[L * n + pos] = src[G::sidx(pos, line)];
    }
  } else {
    for (int idx = threadIdx.x; idx < LINES * N; idx += G::NT) {
      const int line = idx % LINES, pos = idx / LINES;
      const long long L = L0 + line;
      if (pos < n && L < nlines) {
        LineAddr la(L, inner, n);
        g[la.base + (long long)pos * inner] = src[G::sidx(pos, line)];
      }
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Forward axis pass (K4).
// ------------------------------------------------------------------------------------------------
template <int N, int R, int LINES>
__global__ void __launch_bounds__(Geo<N, R, LINES>::NT, 2)
    fwd_axis_kernel(AxisDev ax, const double *in, double *out, long long nlines, long long inner) {
  using G = Geo<N, R, LINES>;
  extern __shared__ double smem[];
  double *bre = smem;
  double *bim = smem + G::BUF;
  double *ys = smem + 2 * G::BUF;
  const int line = threadIdx.x % LINES;
  const int vt = threadIdx.x / LINES;
  const long long L0 = (long long)blockIdx.x * LINES;
  const int n = ax.n, k0 = ax.k0;

  load_tile<N, R, LINES>(in, bre, L0, nlines, inner, n);
  __syncthreads();

  // coefficients at this thread's first-pass input positions k = vt + r TPL
  double a[R];
#pragma unroll
  for (int r = 0; r < R; ++r) a[r] = bre[G::sidx(vt + r * G::TPL, line)];

  // A4: V block for the rows this thread owns (rows of its output bins m <= N/2)
#pragma unroll
  for (int e = 0; e < R; ++e) {
    const int m = out_pos<N, R, LINES>(vt, e);
    if (m <= N / 2) {
      const int j0 = ax.bstart[m], j1 = ax.bstart[m + 1];
      for (int j = j0; j < j1; ++j) {
        double acc = 0.0;
        const double *pv = ax.phiv + (long long)j * k0;
        for (int k = 0; k < k0; ++k) acc = fma(__ldg(&pv[k]), bre[G::sidx(k, line)], acc);
        ys[G::sidx(j, line)] = acc;
      }
    }
  }
  __syncthreads();  // bre is reused as the FFT exchange buffer below

  for (int l = 0; l < ax.r; ++l) {
    const double2 *vl = ax.v + (long long)l * N;
    const double2 *ul = ax.u + (long long)l * n;
    double xr[R], xi[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {  // A1: x = v_l (.) a
      const double2 vv = __ldg(&vl[vt + r * G::TPL]);
      xr[r] = vv.x * a[r];
      xi[r] = vv.y * a[r];
    }
    fft_term<N, R, LINES>(xr, xi, bre, bim, vt, line, ax.tw);  // A2
#pragma unroll
    for (int e = 0; e < R; ++e) {  // A3: rows of bin m: y_j += Re(u~_l[j] X[m])
      const int m = out_pos<N, R, LINES>(vt, e);
      if (m <= N / 2) {
        const int j0 = ax.bstart[m], j1 = ax.bstart[m + 1];
        for (int j = j0; j < j1; ++j) {
          const double2 uu = __ldg(&ul[j]);
          double y = ys[G::sidx(j, line)];
          y = fma(uu.x, xr[e], y);
          y = fma(-uu.y, xi[e], y);
          ys[G::sidx(j, line)] = y;
        }
      }
    }
    __syncthreads();  // next term's first pass store overwrites the exchange buffer
  }
  __syncthreads();
  store_tile<N, R, LINES>(out, ys, L0, nlines, inner, n);
}

// ------------------------------------------------------------------------------------------------
// Inverse axis pass (K5).
// ------------------------------------------------------------------------------------------------
template <int N, int R, int LINES>
__global__ void __launch_bounds__(Geo<N, R, LINES>::NT, 2)
    inv_axis_kernel(AxisDev ax, const double *in, double *out, long long nlines, long long inner) {
  using G = Geo<N, R, LINES>;
  extern __shared__ double smem[];
  double *bre = smem;
  double *bim = smem + G::BUF;
  double *ys = smem + 2 * G::BUF;
  double *avs = smem + 3 * G::BUF;  // k0 x LINES
  const int line = threadIdx.x % LINES;
  const int vt = threadIdx.x / LINES;
  const long long L0 = (long long)blockIdx.x * LINES;
  const int n = ax.n, k0 = ax.k0;

  load_tile<N, R, LINES>(in, ys, L0, nlines, inner, n);
  __syncthreads();

  // a_V = (W V)^T y: per-thread partial sums over the rows of its first-pass bins, then a reduction
  // over the TPL threads of the line through the (not yet used) exchange buffer.
  {
    double *scratch = bre;  // k0 * TPL * LINES doubles (fits in the 2 * BUF of bre + bim)
    for (int k = 0; k < k0; ++k) {
      double acc = 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int m = vt + r * G::TPL;
        if (m <= N / 2) {
          const int j0 = ax.bstart[m], j1 = ax.bstart[m + 1];
          for (int j = j0; j < j1; ++j) acc = fma(__ldg(&ax.phiv[(long long)j * k0 + k]), ys[G::sidx(j, line)], acc);
        }
      }
      scratch[(k * G::TPL + vt) * LINES + line] = acc;
    }
    __syncthreads();
    for (int k = vt; k < k0; k += G::TPL) {
      double s = 0.0;
      for (int t = 0; t < G::TPL; ++t) s += scratch[(k * G::TPL + t) * LINES + line];
      avs[k * LINES + line] = s;
    }
    __syncthreads();
  }

  double acc[R];
#pragma unroll
  for (int e = 0; e < R; ++e) acc[e] = 0.0;

  for (int l = 0; l < ax.r; ++l) {
    const double2 *vl = ax.v + (long long)l * N;
    const double2 *ul = ax.u + (long long)l * n;
    double xr[R], xi[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {  // bin sums b[m] = sum_{j in bin m} u~_l[j] y_j at m = vt + r TPL
      const int m = vt + r * G::TPL;
      double sr = 0.0, si = 0.0;
      if (m <= N / 2) {
        const int j0 = ax.bstart[m], j1 = ax.bstart[m + 1];
        for (int j = j0; j < j1; ++j) {
          const double2 uu = __ldg(&ul[j]);
          const double y = ys[G::sidx(j, line)];
          sr = fma(uu.x, y, sr);
          si = fma(uu.y, y, si);
        }
      }
      xr[r] = sr;
      xi[r] = si;
    }
    fft_term<N, R, LINES>(xr, xi, bre, bim, vt, line, ax.tw);
#pragma unroll
    for (int e = 0; e < R; ++e) {  // a[k] += Re(v_l[k] B[k])
      const int k = out_pos<N, R, LINES>(vt, e);
      const double2 vv = __ldg(&vl[k]);
      acc[e] = fma(vv.x, xr[e], acc[e]);
      acc[e] = fma(-vv.y, xi[e], acc[e]);
    }
    __syncthreads();
  }
  // assemble the output tile in bre: a_G from registers, a_V from avs
#pragma unroll
  for (int e = 0; e < R; ++e) {
    const int k = out_pos<N, R, LINES>(vt, e);
    double val = acc[e];
    if (k < k0) val += avs[k * LINES + line];
    bre[G::sidx(k, line)] = val;
  }
  __syncthreads();
  store_tile<N, R, LINES>(out, bre, L0, nlines, inner, n);
}

}  // namespace jtk
