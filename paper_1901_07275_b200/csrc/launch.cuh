// The axis-pass launch layer of libjt.so: configuration choice per FFT length (radix, term split, clusters) and
// the kernel launches.  Each FFT length's kernel instantiations live in their own translation unit
// (launch_n<N> explicitly instantiated in launch_<N>.cu, compiled in parallel by build.py); jt_api.cu sees only the
// extern declarations at the end.  Everything here is internal (not part of the C ABI, include/jt.h).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/jt.h"
#include "axis_kernels.cuh"

namespace jtl {

// Per-plan launch state: kernels enqueued by the latest call (jt_last_launches) and the term-split workspace
// (few-line launches without a cluster, jtk::TermSplit), grown stream-ordered (cudaMallocAsync)
struct LaunchState {
  int launches = 0;
  double *ts_work = nullptr;
  size_t ts_elems = 0;
  // fused term-split reduction (jt_api.cu transform_body): mode 1 = only report what the launch would do (q_S term
  // slices, q_cluster: reduced in a cluster), mode 2 = a workspace term split that leaves its q_S partials in ts_work
  // (no ts_reduce); in_S > 0: the next launch's input is the sum of those partials (TermSplit::in_part)
  int mode = 0;
  int q_S = 1;
  bool q_cluster = false;
  const double *in_part = nullptr;
  long long in_stride = 0;
  int in_S = 0;
};

inline thread_local std::string g_last_error;

inline jt_status fail(jt_status s, const std::string &msg) {
  g_last_error = msg;
  return s;
}

#define JT_CUDA_TRY(expr)                                                                      \
  do {                                                                                         \
    cudaError_t e_ = (expr);                                                                   \
    if (e_ != cudaSuccess) return fail(JT_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)



// SM count of the current device (cached: a driver query per launch costs microseconds on the latency-bound
// few-line transforms).
inline int sm_count() {
  static int cache[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) return 148;
    cache[dev] = v;
  }
  return cache[dev];
}

// cudaFuncSetAttribute once per (kernel, attribute, device) instead of on every launch.
struct AttrKey {
  const void *kern;
  int attr, dev;
};
inline std::mutex g_attr_mu;
inline std::vector<AttrKey> g_attr_done;
inline cudaError_t ensure_attr(const void *kern, cudaFuncAttribute attr, int value) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_attr_mu);
  for (auto &k : g_attr_done)
    if (k.kern == kern && k.attr == (int)attr && k.dev == dev) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, attr, value);
  if (e == cudaSuccess) g_attr_done.push_back(AttrKey{kern, (int)attr, dev});
  return e;
}
inline cudaError_t ensure_smem_attr(const void *kern, int smem) {
  return ensure_attr(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

// Largest cluster size S <= want (down to 2) with which kernel `kern` (smem bytes per CTA) runs `need` clusters at
// once on this device (one wave: a second wave would double the latency-bound launch); 0 if none (then the caller
// uses the workspace + ts_reduce path).  Cached per kernel, device and request.
struct ClusterKey {
  const void *kern;
  int dev, want, need, got;
};
inline std::vector<ClusterKey> g_cluster_fit;
inline int cluster_fit(const void *kern, int NT, size_t smem, int want, int need) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    for (auto &k : g_cluster_fit)
      if (k.kern == kern && k.dev == dev && k.want == want && k.need == need) return k.got;
  }
  int got = 0;
  if (ensure_smem_attr(kern, (int)smem) == cudaSuccess &&
      (want <= 8 || ensure_attr(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess)) {
    for (int S = want; S >= 2 && !got; --S) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)S);
      cfg.blockDim = dim3((unsigned)NT);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = (unsigned)S;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int nc = 0;
      if (cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) == cudaSuccess && nc >= need) got = S;
    }
  }
  cudaGetLastError();  // (a refused query is not an error of the caller's)
  std::lock_guard<std::mutex> lk(g_attr_mu);
  g_cluster_fit.push_back(ClusterKey{kern, dev, want, need, got});
  return got;
}

// Resident CTAs per SM of kernel `kern` (NT threads, smem bytes), at most 2 and at least 1 (cached).
struct OccKey {
  const void *kern;
  int dev, nt;
  size_t smem;
  int got;
};
inline std::vector<OccKey> g_occ;
inline int blocks_per_sm(const void *kern, int NT, size_t smem) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 1;
  std::lock_guard<std::mutex> lk(g_attr_mu);
  for (auto &k : g_occ)
    if (k.kern == kern && k.dev == dev && k.nt == NT && k.smem == smem) return k.got;
  int nb = 1;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, NT, smem) != cudaSuccess || nb < 1)
    nb = 1;
  cudaGetLastError();
  nb = std::min(nb, 2);
  g_occ.push_back(OccKey{kern, dev, NT, smem, nb});
  return nb;
}

// Is stream s being captured into a CUDA graph?  (Then the calls skip their cross-call ordering events and
// timing marks, and must not grow workspaces: capture after one uncaptured call of the same shape.)
inline bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(s, &st) == cudaSuccess && st == cudaStreamCaptureStatusActive;
}

// Radix of the first (register) pass for FFT length N: one SMEM exchange per term for N <= 1024
// (16x16, 32x16, 32x32), two for 2048 and 4096 (16x16x8, 32x32x4); see DESIGN.md "Kernels".
// MAXR = 4 (more than two nodes in some bin: only for (a, b) near the ends of (-1, 1)) always uses
// radix 16, whose accumulators fit in registers.
constexpr int radix_of(int64_t N, int maxr) {
  return maxr > 2    ? 16
         : N == 16   ? 16
         : N == 32   ? 32
         : N == 64   ? JT_R64
         : N == 128  ? JT_R128
         : N == 256  ? JT_R256
         : N == 512  ? JT_R512
         : N == 1024 ? JT_R1024
         : N == 2048 ? JT_R2048
                     : JT_R4096;
}
// the term-split (few-line, latency-bound) launches may use another radix (Cfg::WG instantiations)
constexpr int radix_ts_of(int64_t N, int maxr) { return maxr <= 2 && N == 128 ? JT_R128_TS : radix_of(N, maxr); }
template <int N, int MAXR>
constexpr int radix_for() {
  return radix_of(N, MAXR);
}

// Launch of an axis-pass kernel (all of them go through here): an optional cluster dimension, and (JT_PDL) the
// programmatic-dependent-launch attribute, so the kernel's prologue (TMEM allocation, twiddles, the first factor
// stages) overlaps the previous kernel's tail; the kernels wait (griddepcontrol.wait) before touching the arrays.
template <class K>
cudaError_t launch_axis_kernel(K kern, unsigned grid, int nt, size_t smem, cudaStream_t s, unsigned cluster,
                               const jtk::AxisDev &ax, const double *in, double *out, long long nlines,
                               const jtk::Layout &lay, const jtk::TermSplit &ts) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3((unsigned)nt);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (cluster > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = cluster;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  if (JT_PDL) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, ax, in, out, nlines, lay, ts);
}

// The term-split instantiation of configuration C's kernel.
template <class C>
auto ts_kernel() {
  if constexpr (C::INV) return jtk::inv_axis_kernel<C, false, true>;
  else return jtk::fwd_axis_kernel<C, false, true>;
}

// Persistent launch: one CTA per SM (C::GPC groups each), looping over batches of GPC x LG lines.
template <class C>
jt_status launch_cfg(LaunchState &st, const jtk::AxisDev &ax, const double *in, double *out, long long nlines,
                     const jtk::Layout &lay, cudaStream_t s, bool allow_ts) {
  const size_t smem = C::smem_bytes();
  const long long lines_per_batch = (long long)C::GPC * C::LG;
  const long long batches = (nlines + lines_per_batch - 1) / lines_per_batch;
  if (batches == 0) return JT_OK;
  const int sms = sm_count();
  const bool split = lay.in_cs != ax.n || lay.out_cs != ax.n;
  // few lines (fewer batches than half the SMs): split the rank terms over S CTAs per batch and sum the
  // partials (jtk::TermSplit, jtk::ts_reduce), so a latency-bound launch uses more of the GPU
  jtk::TermSplit ts{1, nullptr, 0};
  if (allow_ts && !split && nlines == lay.outer * lay.inner && ax.r >= 2 && batches * 2 <= sms) {
    // (CTAs of the term-split kernel that fit on one SM: two for the one-warp-group kernels capped by JT_WG_GPC)
    const int bps = C::MINB > 1 ? blocks_per_sm((const void *)ts_kernel<C>(), C::NT, smem) : 1;
    const int S = (int)std::min<long long>(ax.r, (long long)sms * bps / batches);
    if constexpr (C::CLUSTER_FIT && JT_TS_CLUSTER) {
      // the batch's S CTAs as one thread-block cluster, partials summed through distributed shared memory inside
      // the kernel (jtk::cluster_reduce): one launch, no workspace round trip through L2 / HBM
      auto kern = ts_kernel<C>();
      const int Sc = S > 1 ? cluster_fit((const void *)kern, C::NT, smem, std::min(S, JT_TS_CLUSTER_MAX), (int)batches)
                           : 0;
      if (Sc > 1 && st.mode == 1) {
        st.q_S = Sc;
        st.q_cluster = true;
        return JT_OK;
      }
      if (Sc > 1 && st.mode != 2) {
        // group term split (jtk::TermSplit::gsl): batches of GPC/2 groups' lines, two groups per line group dealing
        // the terms, when that needs fewer rounds of terms per group than the plain split (one-wave clusters)
        long long nb = batches;
        int Sg = Sc, gsl = 1;
        if constexpr (JT_GSPLIT >= 2 && C::GPC % 2 == 0) {
          const long long b2 = (nlines + lines_per_batch / 2 - 1) / (lines_per_batch / 2);
          const int S2 = (int)std::min<long long>(ax.r, (long long)sms * bps / b2);
          const int Sc2 = S2 > 1 ? cluster_fit((const void *)kern, C::NT, smem, std::min(S2, JT_TS_CLUSTER_MAX), (int)b2)
                                 : 0;
          const int rounds1 = (ax.r + Sc - 1) / Sc;
          const int rounds2 = Sc2 > 1 ? ((ax.r + Sc2 - 1) / Sc2 + 1) / 2 : rounds1;
          if (rounds2 < rounds1) {
            nb = b2;
            Sg = Sc2;
            gsl = 2;
          }
        }
        ts = jtk::TermSplit{Sg, nullptr, 1, gsl, st.in_part, st.in_stride, st.in_S};
        JT_CUDA_TRY(launch_axis_kernel(kern, (unsigned)(nb * Sg), C::NT, smem, s, (unsigned)Sg, ax, in, out,
                                       nlines, lay, ts));
        ++st.launches;
        return JT_OK;
      }
    }
    const size_t need = (size_t)S * nlines * ax.n;
    if (st.mode == 1) {
      st.q_S = S;
      st.q_cluster = false;
      return JT_OK;
    }
    if (S > 1) {
      if (st.ts_elems < need) {
        if (capturing(s)) return fail(JT_ERR_ARG, "term-split workspace must grow: run the call once before capturing it");
        // stream-ordered: no implicit device synchronisation in the middle of a pipelined call (a ragged later
        // chunk may need more than an earlier one), and valid under CUDA graph capture
        if (st.ts_work) cudaFreeAsync(st.ts_work, s);
        st.ts_work = nullptr;
        st.ts_elems = 0;
        if (cudaMallocAsync((void **)&st.ts_work, need * sizeof(double), s) != cudaSuccess)
          return fail(JT_ERR_ALLOC, "term-split workspace");
        st.ts_elems = need;
      }
      ts = jtk::TermSplit{S, st.ts_work, 0, 1, st.in_part, st.in_stride, st.in_S};
    }
  }
  if (st.mode == 1) {  // (not a term-split launch)
    st.q_S = 1;
    st.q_cluster = false;
    return JT_OK;
  }
  if (st.in_S > 0 && ts.S <= 1) return fail(JT_ERR_ARG, "internal: fused partial input on a launch without term split");
  const unsigned grid = ts.S > 1 ? (unsigned)(batches * ts.S) : (unsigned)std::min<long long>(batches, sms);
  if constexpr (C::WG && !JT_WG_LARGE) {  // (only reached for term-split launches: see launch_nmd)
    if (ts.S <= 1) return fail(JT_ERR_ARG, "internal: one-warp-group configuration without term split");
    if constexpr (C::INV) {
      JT_CUDA_TRY(ensure_smem_attr((const void *)jtk::inv_axis_kernel<C, false, true>, (int)smem));
      JT_CUDA_TRY(launch_axis_kernel(jtk::inv_axis_kernel<C, false, true>, grid, C::NT, smem, s, 0, ax, in, out, nlines,
                                     lay, ts));
    } else {
      JT_CUDA_TRY(ensure_smem_attr((const void *)jtk::fwd_axis_kernel<C, false, true>, (int)smem));
      JT_CUDA_TRY(launch_axis_kernel(jtk::fwd_axis_kernel<C, false, true>, grid, C::NT, smem, s, 0, ax, in, out, nlines,
                                     lay, ts));
    }
  } else if constexpr (C::INV) {
    auto kern = ts.S > 1 ? jtk::inv_axis_kernel<C, false, true>
                         : (split ? jtk::inv_axis_kernel<C, true> : jtk::inv_axis_kernel<C, false>);
    JT_CUDA_TRY(ensure_smem_attr((const void *)kern, (int)smem));
    JT_CUDA_TRY(launch_axis_kernel(kern, grid, C::NT, smem, s, 0, ax, in, out, nlines, lay, ts));
  } else {
    auto kern = ts.S > 1 ? jtk::fwd_axis_kernel<C, false, true>
                         : (split ? jtk::fwd_axis_kernel<C, true> : jtk::fwd_axis_kernel<C, false>);
    JT_CUDA_TRY(ensure_smem_attr((const void *)kern, (int)smem));
    JT_CUDA_TRY(launch_axis_kernel(kern, grid, C::NT, smem, s, 0, ax, in, out, nlines, lay, ts));
  }
  JT_CUDA_TRY(cudaGetLastError());
  ++st.launches;
  if (ts.S > 1 && st.mode == 2) {  // partials left in the workspace for the next pass to sum
    st.q_S = ts.S;
    return JT_OK;
  }
  if (ts.S > 1) {
    ++st.launches;
    const long long total = nlines * ax.n;
    const int thr = 256;
    const unsigned g = (unsigned)std::min<long long>((total + thr - 1) / thr, 4LL * sms);
    jtk::ts_reduce<<<g, thr, 0, s>>>(ts.part, out, ts.S, nlines, ax.n, lay.inner);
    JT_CUDA_TRY(cudaGetLastError());
  }
  return JT_OK;
}

// Would launch_cfg<C> split the rank terms (few lines)?  Same test as inside launch_cfg.
template <class C>
bool term_split_applies(const jtk::AxisDev &ax, long long nlines, const jtk::Layout &lay, bool allow_ts, int sms) {
  const long long batches = (nlines + (long long)C::GPC * C::LG - 1) / ((long long)C::GPC * C::LG);
  const bool split = lay.in_cs != ax.n || lay.out_cs != ax.n;
  return allow_ts && !split && nlines == lay.outer * lay.inner && ax.r >= 2 && batches > 0 && batches * 2 <= sms &&
         std::min<long long>(ax.r, sms / batches) > 1;
}

template <int N, int MAXR, bool INV>
jt_status launch_nmd(LaunchState &st, const jtk::AxisDev &ax, const double *in, double *out, long long nlines,
                     const jtk::Layout &lay, cudaStream_t s, bool allow_ts) {
  using C = jtk::Cfg<N, radix_for<N, MAXR>(), MAXR, INV>;
  using CW = jtk::Cfg<N, radix_ts_of(N, MAXR), MAXR, INV, true>;
  if constexpr (JT_TS_WG && (CW::LG != C::LG || CW::R != C::R)) {  // term-split launches: one-warp groups / radix
    const int sms = sm_count();
    if (term_split_applies<CW>(ax, nlines, lay, allow_ts, sms)) {
      jtk::AxisDev axt = ax;
      axt.tw = ax.tw_ts;
      return launch_cfg<CW>(st, axt, in, out, nlines, lay, s, true);
    }
    if constexpr (JT_WG_LARGE && N == JT_WG_LARGE && CW::R == C::R) {  // (A/B: one-warp groups for every launch)
      jtk::AxisDev axt = ax;
      axt.tw = ax.tw_ts;
      return launch_cfg<CW>(st, axt, in, out, nlines, lay, s, allow_ts);
    }
  }
  return launch_cfg<C>(st, ax, in, out, nlines, lay, s, allow_ts);
}

template <int N, int MAXR>
jt_status launch_nm(LaunchState &st, bool inverse, const jtk::AxisDev &ax, const double *in, double *out,
                    long long nlines, const jtk::Layout &lay, cudaStream_t s, bool allow_ts) {
  if (inverse) return launch_nmd<N, MAXR, true>(st, ax, in, out, nlines, lay, s, allow_ts);
  return launch_nmd<N, MAXR, false>(st, ax, in, out, nlines, lay, s, allow_ts);
}

// FFT lengths with Cfg::PAIR forward kernels (the last Stockham pass must hold an even number of butterflies per
// thread, so that a thread owns bin m and its conjugate mirror N - 1 - m): 512 = 32 x 16 (2 butterflies), 4096 =
// 32 x 32 x 4 (8), 2048 = 16 x 16 x 8 (2), and 256 as 32 x 8 (4; the unpaired N = 256 kernels are radix 16 = 16 x 16,
// one butterfly)
constexpr bool pair_length(int64_t N) { return JT_PAIR && (N == 512 || N == 256 || N == 4096 || (JT_PAIR_2048 && N == 2048)); }
constexpr int pair_radix(int64_t N) { return N == 256 ? 32 : radix_of(N, 2); }

template <int N>
jt_status launch_n(LaunchState &st, bool inverse, int maxr, const jtk::AxisDev &ax, const double *in, double *out,
                   long long nlines, const jtk::Layout &lay, cudaStream_t s, bool allow_ts) {
  if (maxr == -2) {  // paired real rank terms (jt_api.cu launch_axis)
    if constexpr (pair_length(N)) {
      using CP = jtk::Cfg<N, pair_radix(N), 2, false, false, true>;
      using CI = jtk::Cfg<N, pair_radix(N), 2, true, false, true>;
      if (inverse) return launch_cfg<CI>(st, ax, in, out, nlines, lay, s, allow_ts);
      return launch_cfg<CP>(st, ax, in, out, nlines, lay, s, allow_ts);
    } else {
      return fail(JT_ERR_ARG, "no pair kernels for this FFT length");
    }
  }
  if (maxr <= 2) return launch_nm<N, 2>(st, inverse, ax, in, out, nlines, lay, s, allow_ts);
  if (maxr == 3) return launch_nm<N, 3>(st, inverse, ax, in, out, nlines, lay, s, allow_ts);
  return launch_nm<N, 4>(st, inverse, ax, in, out, nlines, lay, s, allow_ts);
}

// JT_CHECKS counters of this translation unit's device module (each launch_<N>.cu has its own): read into *c / *l
// (added / first nonzero kept), then reset
template <int N>
jt_status checks_io(unsigned long long *c, int *l) {
  unsigned long long v = 0;
  int ln = 0;
  JT_CUDA_TRY(cudaMemcpyFromSymbol(&v, jtk::jt_check_count, sizeof(v)));
  JT_CUDA_TRY(cudaMemcpyFromSymbol(&ln, jtk::jt_check_line, sizeof(ln)));
  *c += v;
  if (!*l) *l = ln;
  const unsigned long long z = 0;
  const int zl = 0;
  JT_CUDA_TRY(cudaMemcpyToSymbol(jtk::jt_check_count, &z, sizeof(z)));
  JT_CUDA_TRY(cudaMemcpyToSymbol(jtk::jt_check_line, &zl, sizeof(zl)));
  return JT_OK;
}

extern template jt_status launch_n<16>(LaunchState &, bool, int, const jtk::AxisDev &, const double *, double *, long long, const jtk::Layout &, cudaStream_t, bool);
extern template jt_status launch_n<32>(LaunchState &, bool, int, const jtk::AxisDev &, const double *, double *, long long, const jtk::Layout &, cudaStream_t, bool);
extern template jt_status launch_n<64>(LaunchState &, bool, int, const jtk::AxisDev &, const double *, double *, long long, const jtk::Layout &, cudaStream_t, bool);
extern template jt_status launch_n<128>(LaunchState &, bool, int, const jtk::AxisDev &, const double *, double *, long long, const jtk::Layout &, cudaStream_t, bool);
extern template jt_status launch_n<256>(LaunchState &, bool, int, const jtk::AxisDev &, const double *, double *, long long, const jtk::Layout &, cudaStream_t, bool);
extern template jt_status launch_n<512>(LaunchState &, bool, int, const jtk::AxisDev &, const double *, double *, long long, const jtk::Layout &, cudaStream_t, bool);
extern template jt_status launch_n<1024>(LaunchState &, bool, int, const jtk::AxisDev &, const double *, double *, long long, const jtk::Layout &, cudaStream_t, bool);
extern template jt_status launch_n<2048>(LaunchState &, bool, int, const jtk::AxisDev &, const double *, double *, long long, const jtk::Layout &, cudaStream_t, bool);
extern template jt_status launch_n<4096>(LaunchState &, bool, int, const jtk::AxisDev &, const double *, double *, long long, const jtk::Layout &, cudaStream_t, bool);

extern template jt_status checks_io<16>(unsigned long long *, int *);
extern template jt_status checks_io<32>(unsigned long long *, int *);
extern template jt_status checks_io<64>(unsigned long long *, int *);
extern template jt_status checks_io<128>(unsigned long long *, int *);
extern template jt_status checks_io<256>(unsigned long long *, int *);
extern template jt_status checks_io<512>(unsigned long long *, int *);
extern template jt_status checks_io<1024>(unsigned long long *, int *);
extern template jt_status checks_io<2048>(unsigned long long *, int *);
extern template jt_status checks_io<4096>(unsigned long long *, int *);

}  // namespace jtl
