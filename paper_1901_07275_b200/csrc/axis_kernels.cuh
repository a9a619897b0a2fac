// Fused axis-pass kernels, warp-group design (K4 forward, K5 inverse).
//
// Every line along the transformed axis is one of the paper's "n^{d-1} 1D transforms" (PAPER.md:676,
// 724).  A GROUP of threads owns LG complete lines (LG = 32 / TPL lines per warp when a line needs
// TPL <= 32 threads, else one line spread over GW = TPL / 32 warps) and computes, entirely on chip,
//
//   forward (eq:oneJ):    y = W V a_V  +  Re sum_{l<r} D_{u~_l} F_N D_{v_l} a_G
//   inverse (eq:oneJinv): a_V = (W V)^T y,  a_G = Re sum_{l<r} D_{v_l} F_N^T D_{u~_l} y
//
// with ONE HBM read and ONE HBM write of each line per axis pass (all r rank terms batched in the pass,
// north star: "batches several rank terms per pass to cut HBM round trips").  Groups never wait on one
// another: the only barriers are __syncwarp (GW == 1) or a named barrier of the group's GW warps, so the
// load / FFT / exchange phases of different groups on one SM overlap freely.
//
// Per rank term l (registers unless noted):
//   forward:  x[k] = v_l[k] a[k]                               (A1: column scale + pack)
//             X = F_N x  (positive exponent, unnormalised)     (A2: Stockham passes; radix-R first pass in
//                                                                registers, exchange through SMEM)
//             y_{m,c} += Re(u~_l[m,c] X[m])  for bins m <= N/2  (A3: row scale + Re + accumulate; rows of
//                                                                bin m are bstart[m] + c, c < MAXR)
//   inverse:  b[m] = sum_c u~_l[m,c] y_{m,c}                   (bin sums, m <= N/2; no atomics)
//             B = F_N b                                        (same sign)
//             a[k] += Re(v_l[k] B[k])
//
// Register ownership (thread vt of TPL on its line): first-pass inputs at positions vt + r TPL (r < R);
// last-pass outputs at v + s (N / RS_L), v = vt + i TPL.  The forward keeps its accumulators y per OUTPUT
// BIN of the last pass (only bins m <= N/2 are ever read, t in (0, pi), so the dead half of the last
// butterflies is removed by the compiler); the inverse keeps its y per INPUT bin of the first pass.
// Both hold at most R/2 + 1 bins x MAXR rows per thread.
#pragma once
#include <cuda_runtime.h>

#include "fft_regs.cuh"

namespace jtk {

struct AxisDev {
  int n;      // axis length
  int N;      // FFT length (power of two >= max(n, 16))
  int k0;     // width of the dense low-degree block W V (<= 32)
  int r;      // rank (FFT terms per line)
  int nbins;  // N / 2 + 1
  const double2 *v;      // r x N        v_l[k] at v[l N + k] (zero for k < k0 and k >= n)
  const double2 *ub;     // r x nbins x MAXR   u~_l of row bstart[m] + c at ub[(l nbins + m) MAXR + c] (0-padded)
  const double *phivb;   // k0 x nbins x MAXR  (W V)[bstart[m] + c, k] at phivb[(k nbins + m) MAXR + c] (0-padded)
  const int *bstart;     // nbins + 1 row offsets: rows of bin m are bstart[m] .. bstart[m+1]-1
  const double2 *tw;     // per-pass twiddle tables, see TwOff (pass NS, radix RS: (RS-1) NS entries,
                         // entry (r-1) NS + j = e^{+2 pi i j r / (NS RS)})
};

constexpr int K0MAX = 32;

// Radix of the Stockham pass that starts at sub-transform size NS.
template <int N, int R, int NS>
struct Pass {
  static constexpr int RS = (N / NS < R) ? N / NS : R;
  static constexpr int B = R / RS;  // butterflies per thread in this pass
  static constexpr bool LAST = (NS * RS == N);
};

template <int N, int R, int NS = 1>
struct LastNS {
  static constexpr int value = Pass<N, R, NS>::LAST ? NS : LastNS<N, R, NS * Pass<N, R, NS>::RS>::value;
};
template <int N, int R>
struct LastNS<N, R, N> {
  static constexpr int value = N;
};

// Offset of pass NS's twiddle table in AxisDev::tw: the tables of the passes after the first, in
// pass order, each laid out [r-1][j] so that the threads of a pass read consecutive entries.
template <int N, int R, int NS, int P = Pass<N, R, 1>::RS>
struct TwOff {
  static constexpr int value = (P >= NS) ? 0 : (Pass<N, R, P>::RS - 1) * P + TwOff<N, R, NS, P * Pass<N, R, P>::RS>::value;
};
template <int N, int R, int NS>
struct TwOff<N, R, NS, N> {
  static constexpr int value = 0;
};
template <int N, int R>
constexpr int tw_entries() { return TwOff<N, R, N>::value; }

template <int N_, int R_, int MAXR_>
struct Cfg {
  static constexpr int N = N_, R = R_, MAXR = MAXR_;
  static constexpr int TPL = N / R;                      // threads per line
  static constexpr int LG = TPL >= 32 ? 1 : 32 / TPL;    // lines per group
  static constexpr int GT = TPL * LG;                    // threads per group
  static constexpr int GW = GT / 32;                     // warps per group
  static constexpr int GPC = GW >= 4 ? 1 : 4 / GW;       // groups per CTA
  static constexpr int NT = GPC * GT;                    // threads per CTA
  // Register budget (32-bit registers): a thread holds x (4R), its persistent input state (the
  // coefficients a, or the inverse's input-bin values: 2R resp. 2 NB MAXR) and its output accumulators
  // (the forward's bin rows y: 2 NB MAXR, or the inverse's acc: 2R).  For R >= 32 that exceeds 255, so
  // the input state lives in a thread-private SMEM area (PRIV), read once per term (8 B per point).
  static constexpr bool PRIV = R >= 32;
  static constexpr int REGS = R >= 32 ? 255 : (MAXR > 2 ? 200 : 168);
  static constexpr int MINB = 65536 / (REGS * NT) > 0 ? 65536 / (REGS * NT) : 1;  // CTAs per SM
  static constexpr int NSL = LastNS<N, R>::value;        // the last pass starts at sub-size NSL
  static constexpr int RSL = Pass<N, R, NSL>::RS;        // ... with radix RSL
  static constexpr int NB = R / 2 + 1;                   // bins per thread (R/2 + the Nyquist slot)
  // exchange buffer: double2 slots [pos][line], LG pad slots after every R positions -> the strided
  // first-pass stores and the unit-stride loads are both free of bank conflicts
  static constexpr int SLOTS = Pass<N, R, 1>::LAST ? 0 : (N + N / R) * LG;
  static constexpr int PSLOTS = PRIV ? (R > NB * MAXR ? R : NB * MAXR) : 0;  // private doubles per thread
  static constexpr int GROUP_BYTES = SLOTS * 16 + K0MAX * LG * 8 + PSLOTS * GT * 8;
  static constexpr size_t smem_bytes() { return (size_t)GPC * GROUP_BYTES; }
  __device__ static __forceinline__ int sidx(int pos, int line) { return (pos + pos / R) * LG + line; }
  static_assert(GT % 32 == 0, "group must be whole warps");
  static_assert(RSL >= 2, "last pass radix");
};

template <class C>
__device__ __forceinline__ void group_sync() {
  if constexpr (C::GW == 1) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)(threadIdx.x / C::GT)), "r"(C::GT) : "memory");
  }
}

// ---- Stockham passes over the group's exchange buffer -------------------------------------------------

template <class C, int NS>
__device__ __forceinline__ void pass_store(const double (&xr)[C::R], const double (&xi)[C::R], double2 *buf, int vt,
                                           int line) {
  using P = Pass<C::N, C::R, NS>;
#pragma unroll
  for (int i = 0; i < P::B; ++i) {
    const int v = vt + i * C::TPL;
    const int idxD = (v / NS) * NS * P::RS + (v % NS);
#pragma unroll
    for (int s = 0; s < P::RS; ++s) buf[C::sidx(idxD + s * NS, line)] = make_double2(xr[i * P::RS + s], xi[i * P::RS + s]);
  }
}

template <class C, int NS>
__device__ __forceinline__ void pass_load_compute(double (&xr)[C::R], double (&xi)[C::R], const double2 *buf, int vt,
                                                  int line, const double2 *__restrict__ tw) {
  using P = Pass<C::N, C::R, NS>;
  constexpr int RS = P::RS;
#pragma unroll
  for (int i = 0; i < P::B; ++i) {
    const int v = vt + i * C::TPL;
#pragma unroll
    for (int r = 0; r < RS; ++r) {
      const double2 d = buf[C::sidx(v + r * (C::N / RS), line)];
      xr[i * RS + r] = d.x;
      xi[i * RS + r] = d.y;
    }
    const double2 *twp = tw + TwOff<C::N, C::R, NS>::value + (v % NS);
#pragma unroll
    for (int r = 1; r < RS; ++r) {
      const double2 w = __ldg(&twp[(r - 1) * NS]);
      const double tr = xr[i * RS + r] * w.x - xi[i * RS + r] * w.y;
      xi[i * RS + r] = fma(xr[i * RS + r], w.y, xi[i * RS + r] * w.x);
      xr[i * RS + r] = tr;
    }
    dft<RS>(&xr[i * RS], &xi[i * RS]);
  }
}

template <class C, int NS>
__device__ __forceinline__ void run_passes(double (&xr)[C::R], double (&xi)[C::R], double2 *buf, int vt, int line,
                                           const double2 *__restrict__ tw) {
  if constexpr (NS < C::N) {
    pass_load_compute<C, NS>(xr, xi, buf, vt, line, tw);
    if constexpr (!Pass<C::N, C::R, NS>::LAST) {
      group_sync<C>();
      pass_store<C, NS>(xr, xi, buf, vt, line);
      group_sync<C>();
      run_passes<C, NS * Pass<C::N, C::R, NS>::RS>(xr, xi, buf, vt, line, tw);
    }
  }
}

// Full FFT of one term; first-pass inputs (positions vt + r TPL) in registers on entry, last-pass
// outputs (positions out_pos) in registers on exit.  The caller syncs the group before the next call.
template <class C>
__device__ __forceinline__ void fft(double (&xr)[C::R], double (&xi)[C::R], double2 *buf, int vt, int line,
                                    const double2 *__restrict__ tw) {
  using P0 = Pass<C::N, C::R, 1>;
#pragma unroll
  for (int i = 0; i < P0::B; ++i) dft<P0::RS>(&xr[i * P0::RS], &xi[i * P0::RS]);
  if constexpr (!P0::LAST) {
    pass_store<C, 1>(xr, xi, buf, vt, line);
    group_sync<C>();
    run_passes<C, P0::RS>(xr, xi, buf, vt, line, tw);
  }
}

// Frequency index of last-pass output register e = i RSL + s.
template <class C>
__device__ __forceinline__ int out_pos(int vt, int e) {
  return vt + (e / C::RSL) * C::TPL + (e % C::RSL) * (C::N / C::RSL);
}

// Forward: the thread's output bins q = i (RSL/2) + s (s < RSL/2) -> register e = i RSL + s; q = R/2 is the
// Nyquist bin N/2 = output s = RSL/2 of butterfly i = 0 (that bin only when vt == 0).
template <class C>
__device__ __forceinline__ constexpr int fwd_reg_of_bin(int q) {
  return q < C::R / 2 ? (q / (C::RSL / 2)) * C::RSL + (q % (C::RSL / 2)) : C::RSL / 2;
}

// Group geometry shared by both kernels.
template <class C>
struct GroupCtx {
  int grp, line, vt;
  long long L, base;
  bool live;
  double2 *buf;
  double *alow;
  double *priv;  // thread-private slots [slot][gt] (C::PRIV)
  int gt;
  __device__ __forceinline__ GroupCtx(double2 *smem, long long nlines, long long inner, int n) {
    grp = threadIdx.x / C::GT;
    gt = threadIdx.x % C::GT;
    line = gt % C::LG;
    vt = gt / C::LG;
    L = ((long long)blockIdx.x * C::GPC + grp) * C::LG + line;
    live = L < nlines;
    const long long o = L / inner, i = L - o * inner;
    base = o * (long long)n * inner + i;
    char *gb = reinterpret_cast<char *>(smem) + grp * C::GROUP_BYTES;
    buf = reinterpret_cast<double2 *>(gb);
    alow = reinterpret_cast<double *>(gb + C::SLOTS * sizeof(double2));
    priv = alow + K0MAX * C::LG;
  }
};

// S doubles of per-thread state: registers, or (C::PRIV) the thread's private SMEM slots.  Indices are
// compile-time constants after unrolling.
template <class C, int S>
struct State {
  double reg[C::PRIV ? 1 : S];
  double *sm;
  int gt;
  __device__ __forceinline__ State(double *p, int t) : sm(p), gt(t) {}
  __device__ __forceinline__ double get(int i) const {
    if constexpr (C::PRIV) return sm[i * C::GT + gt];
    else return reg[i];
  }
  __device__ __forceinline__ void set(int i, double v) {
    if constexpr (C::PRIV) sm[i * C::GT + gt] = v;
    else reg[i] = v;
  }
};

template <int MAXR>
__device__ __forceinline__ void load_rows(const double *__restrict__ p, double (&o)[MAXR]) {
  if constexpr (MAXR % 2 == 0) {
#pragma unroll
    for (int c = 0; c < MAXR; c += 2) {
      const double2 t = __ldg(reinterpret_cast<const double2 *>(p + c));
      o[c] = t.x;
      o[c + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int c = 0; c < MAXR; ++c) o[c] = __ldg(p + c);
  }
}

// ------------------------------------------------------------------------------------------------
// Forward axis pass (K4).
// ------------------------------------------------------------------------------------------------
template <class C>
__global__ void __launch_bounds__(C::NT, C::MINB) fwd_axis_kernel(AxisDev ax, const double *in, double *out, long long nlines,
                                                          long long inner) {
  constexpr int R = C::R, TPL = C::TPL, LG = C::LG, NB = C::NB, MAXR = C::MAXR;
  extern __shared__ double2 smem[];
  GroupCtx<C> g(smem, nlines, inner, ax.n);
  const int n = ax.n, k0 = ax.k0, nbins = ax.nbins;
  const int vt = g.vt, line = g.line;

  // coefficients at the first-pass input positions k = vt + r TPL
  State<C, R> a(g.priv, g.gt);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int k = vt + r * TPL;
    const double ak = (g.live && k < n) ? in[g.base + (long long)k * inner] : 0.0;
    a.set(r, ak);
    if (r * TPL < K0MAX && k < k0) g.alow[k * LG + line] = ak;
  }

  int m[NB];
#pragma unroll
  for (int q = 0; q < NB; ++q) m[q] = q < R / 2 ? out_pos<C>(vt, fwd_reg_of_bin<C>(q)) : C::N / 2;

  // A4: y = W V a_V on the rows of the thread's bins
  double y[NB][MAXR];
#pragma unroll
  for (int q = 0; q < NB; ++q)
#pragma unroll
    for (int c = 0; c < MAXR; ++c) y[q][c] = 0.0;
  group_sync<C>();
  for (int k = 0; k < k0; ++k) {
    const double ak = g.alow[k * LG + line];
    const double *pk = ax.phivb + (long long)k * nbins * MAXR;
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      double pv[MAXR];
      load_rows<MAXR>(pk + m[q] * MAXR, pv);
#pragma unroll
      for (int c = 0; c < MAXR; ++c) y[q][c] = fma(pv[c], ak, y[q][c]);
    }
  }

  for (int l = 0; l < ax.r; ++l) {
    const double2 *vl = ax.v + (long long)l * C::N;
    const double2 *ul = ax.ub + (long long)l * nbins * MAXR;
    double xr[R], xi[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {  // A1
      const double2 vv = __ldg(&vl[vt + r * TPL]);
      const double ar = a.get(r);
      xr[r] = vv.x * ar;
      xi[r] = vv.y * ar;
    }
    fft<C>(xr, xi, g.buf, vt, line, ax.tw + (l >> 30));  // A2 (see Cfg::REGS)
#pragma unroll
    for (int q = 0; q < NB; ++q) {  // A3
      const int e = fwd_reg_of_bin<C>(q);
#pragma unroll
      for (int c = 0; c < MAXR; ++c) {
        const double2 uu = __ldg(&ul[m[q] * MAXR + c]);
        y[q][c] = fma(uu.x, xr[e], y[q][c]);
        y[q][c] = fma(-uu.y, xi[e], y[q][c]);
      }
    }
    group_sync<C>();  // the next term's first store overwrites the exchange buffer
  }

  if (g.live) {
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      if (q < R / 2 || vt == 0) {
        const int j0 = __ldg(&ax.bstart[m[q]]), cnt = __ldg(&ax.bstart[m[q] + 1]) - j0;
#pragma unroll
        for (int c = 0; c < MAXR; ++c)
          if (c < cnt) out[g.base + (long long)(j0 + c) * inner] = y[q][c];
      }
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Inverse axis pass (K5).
// ------------------------------------------------------------------------------------------------
template <class C>
__global__ void __launch_bounds__(C::NT, C::MINB) inv_axis_kernel(AxisDev ax, const double *in, double *out, long long nlines,
                                                          long long inner) {
  constexpr int R = C::R, TPL = C::TPL, LG = C::LG, NB = C::NB, MAXR = C::MAXR;
  extern __shared__ double2 smem[];
  GroupCtx<C> g(smem, nlines, inner, ax.n);
  const int n = ax.n, k0 = ax.k0, nbins = ax.nbins;
  const int vt = g.vt, line = g.line;

  // input bins: q < R/2 -> first-pass position vt + q TPL; q = R/2 -> position vt + N/2 (Nyquist, vt == 0)
  int m[NB];
  State<C, NB * MAXR> yb(g.priv, g.gt);  // yb(q MAXR + c): row c of input bin q
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    const bool own = q < R / 2 || vt == 0;
    m[q] = q < R / 2 ? vt + q * TPL : C::N / 2;
    const int j0 = __ldg(&ax.bstart[m[q]]), cnt = __ldg(&ax.bstart[m[q] + 1]) - j0;
#pragma unroll
    for (int c = 0; c < MAXR; ++c)
      yb.set(q * MAXR + c, (g.live && own && c < cnt) ? in[g.base + (long long)(j0 + c) * inner] : 0.0);
  }

  // a_V = (W V)^T y: thread partial sums over its rows, reduced over the TPL threads of the line
  for (int k = 0; k < k0; ++k) {
    const double *pk = ax.phivb + (long long)k * nbins * MAXR;
    double p = 0.0;
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      double pv[MAXR];
      load_rows<MAXR>(pk + m[q] * MAXR, pv);
#pragma unroll
      for (int c = 0; c < MAXR; ++c) p = fma(pv[c], yb.get(q * MAXR + c), p);
    }
    if constexpr (C::GW == 1) {
#pragma unroll
      for (int off = LG; off < 32; off *= 2) p += __shfl_xor_sync(0xffffffffu, p, off);
      if (vt == 0) g.alow[k * LG + line] = p;
    } else {
#pragma unroll
      for (int off = 1; off < 32; off *= 2) p += __shfl_xor_sync(0xffffffffu, p, off);
      if ((threadIdx.x & 31) == 0) reinterpret_cast<double *>(g.buf)[k * C::GW + vt / 32] = p;
    }
  }
  if constexpr (C::GW > 1) {
    group_sync<C>();
    if (vt < k0) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < C::GW; ++w) s += reinterpret_cast<double *>(g.buf)[vt * C::GW + w];
      g.alow[vt] = s;
    }
  }
  group_sync<C>();

  double acc[R];
#pragma unroll
  for (int e = 0; e < R; ++e) acc[e] = 0.0;

  for (int l = 0; l < ax.r; ++l) {
    const double2 *vl = ax.v + (long long)l * C::N;
    const double2 *ul = ax.ub + (long long)l * nbins * MAXR;
    double xr[R], xi[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      xr[r] = 0.0;
      xi[r] = 0.0;
      if (r <= R / 2) {  // bin sums (positions > N/2 hold no rows)
#pragma unroll
        for (int c = 0; c < MAXR; ++c) {
          const double2 uu = __ldg(&ul[m[r] * MAXR + c]);
          const double yv = yb.get(r * MAXR + c);
          xr[r] = fma(uu.x, yv, xr[r]);
          xi[r] = fma(uu.y, yv, xi[r]);
        }
      }
    }
    fft<C>(xr, xi, g.buf, vt, line, ax.tw + (l >> 30));
#pragma unroll
    for (int e = 0; e < R; ++e) {  // a[k] += Re(v_l[k] B[k])
      const double2 vv = __ldg(&vl[out_pos<C>(vt, e)]);
      acc[e] = fma(vv.x, xr[e], acc[e]);
      acc[e] = fma(-vv.y, xi[e], acc[e]);
    }
    group_sync<C>();
  }

  if (g.live) {
#pragma unroll
    for (int e = 0; e < R; ++e) {
      const int k = out_pos<C>(vt, e);
      double val = acc[e];
      if (k < k0) val += g.alow[k * LG + line];
      if (k < n) out[g.base + (long long)k * inner] = val;
    }
  }
}

}  // namespace jtk
