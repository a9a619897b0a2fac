// Fused axis-pass kernels (K4 forward, K5 inverse).
//
// Every line along the transformed axis is one of the paper's "n^{d-1} 1D transforms" (PAPER.md:676,
// 724).  A GROUP of threads owns LG complete lines (TPL threads per line, thread gt = vt LG + line) and
// computes, entirely on chip,
//
//   forward (eq:oneJ):    y = W V a_V  +  Re sum_{l<r} D_{u~_l} F_N D_{v_l} a_G
//   inverse (eq:oneJinv): a_V = (W V)^T y,  a_G = Re sum_{l<r} D_{v_l} F_N^T D_{u~_l} y
//
// with ONE HBM read and ONE HBM write of each line per axis pass: all r rank terms are batched in the
// pass (north star: "batches several rank terms per pass to cut HBM round trips").
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
// Execution structure:
//   * Persistent CTAs (one per SM) of GPC independent groups loop over batches of GPC x LG lines.
//   * The per-term factors (v_l: N complex; u~_l: MAXR x (N/2+1) complex) are streamed by the TMA
//     bulk-copy engine into a 2-stage SMEM ring shared by the CTA's groups (mbarrier full/empty pairs,
//     thread 0 is the producer).  Measured on B200 (tools/l1_probe.cu): an LDG.128 costs the L1 data
//     pipe 4 cycles per warp whatever the address sharing and misses L1 here (SMEM takes it), while a
//     broadcast LDS.128 costs ~2; the ring turns long-latency global factor loads into short SMEM ones.
//   * Groups synchronise only among themselves (__syncwarp, or a named barrier of the group's warps), so
//     the FP64-heavy FFT phases of one group overlap the SMEM-heavy exchange phases of another.
//   * Register ownership (thread vt of TPL on its line): first-pass inputs at positions vt + r TPL
//     (r < R); last-pass outputs at v + s (N / RS_L), v = vt + i TPL.  The forward keeps its y per OUTPUT
//     bin of the last pass (only bins m <= N/2 are read, t in (0, pi), so the dead half of the last
//     butterflies is removed by the compiler); the inverse keeps its y per INPUT bin of the first pass.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fft_regs.cuh"
#include "tmem.cuh"
#include "tuning.h"

namespace jtk {

struct AxisDev {
  int n;      // axis length
  int N;      // FFT length (power of two >= max(n, 16))
  int k0;     // width of the dense low-degree block W V (<= 32)
  int r;      // rank (FFT terms per line)
  int nbins;  // N / 2 + 1
  const double2 *v;      // r x N        v_l[k] at v[l N + k] (zero for k < k0 and k >= n)
  const double2 *ub;     // r x MAXR x nbins   u~_l of row bstart[m] + c at ub[(l MAXR + c) nbins + m] (0-padded)
  const double *phivb;   // k0 x MAXR x nbins  (W V)[bstart[m] + c, k] at phivb[(k MAXR + c) nbins + m] (0-padded)
  const double *phivc;   // the same in chunks of 2 degrees: (W V)[bstart[m] + c, 2 h + kk] at
                         // phivc[((h nbins + m) MAXR + c) 2 + kk], h < ceil(k0 / KPT) KPT / 2 (0-padded); a ring stage
                         // takes the KPT / 2 consecutive chunks of its term
  const int *bstart;     // nbins + 1 row offsets: rows of bin m are bstart[m] .. bstart[m+1]-1
  const double2 *tw;     // per-pass twiddle tables, see TwOff (pass NS, radix RS: (RS-1) NS entries,
                         // entry (r-1) NS + j = e^{+2 pi i j r / (NS RS)})
  const double2 *tw_ts;  // the same for the radix of the term-split launches where it differs (else == tw)
};

// Term split (few lines: latency-bound launches).  S > 1: CTA b handles batch b / S and only the rank terms
// [s r / S, (s + 1) r / S) of slice s = b % S (the W V block in the slices of its degrees), writing its
// partial line results to part[(s nlines + L) n + j]; ts_reduce sums the S partials in slice order.
struct TermSplit {
  int S;
  double *part;
  // cluster != 0: the grid is launched in clusters of the S CTAs of a batch (cluster rank = slice), and the
  // partial lines are summed through distributed shared memory at the end of the kernel (cluster_reduce): no
  // workspace, no ts_reduce launch
  int cluster;
  // gsl == 2 (cluster launches only): group term split -- a batch is GPC/2 groups' lines, and each line group is
  // processed by two groups that deal the CTA's terms between them (Ctx::gsl), so twice the CTAs' worth of terms run
  // at once where a one-wave cluster grid cannot take more slices (256^2: 3 -> 2 terms per group)
  int gsl = 1;
  // in_S > 0 (term-split launches only): the input is the sum, in slice order, of in_S arrays at in_part + s in_stride
  // (the previous pass's partials, not reduced by a launch of their own: the reduction fused into this pass's loads)
  const double *in_part = nullptr;
  long long in_stride = 0;
  int in_S = 0;
};

// Input element at offset idx: the plain input, or (fused reduction) the sum of the previous pass's partials.
// (compiled only with JT_TS_FUSE: the runtime branch alone cost the 1D forward 3 us -- the plain input loads no longer
// all issue before the first use)
template <bool TSPLIT>
__device__ __forceinline__ double load_in(const double *in, const TermSplit &ts, long long idx) {
  if constexpr (TSPLIT && JT_TS_FUSE) {
    if (ts.in_S > 0) {
      double v[4], sum = 0.0;
      for (int s0 = 0; s0 < ts.in_S; s0 += 4) {  // four partials' loads in flight per round
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = s0 + q < ts.in_S ? __ldg(&ts.in_part[(s0 + q) * ts.in_stride + idx]) : 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (s0 + q < ts.in_S) sum += v[q];
      }
      return sum;
    }
  }
  return __ldg(&in[idx]);
}

// (build-time tuning knobs JT_*: tuning.h)

// ---- JT_CHECKS builds (build.py `checks`: libjt_checks.so): bounds checks on every global index, shared-memory
// slot and tensor-memory column the kernels touch.  A violation is counted (jt_check_count, the first one's
// source line in jt_check_line; read by jt_debug_checks) and the access is SKIPPED, so a checks run never
// faults the GPU (the substitute for compute-sanitizer, which is closed on this pool).  Off: JT_CHK(c) is true.
#ifndef JT_CHECKS
#define JT_CHECKS 0
#endif
// (static: one copy per translation unit / device module -- the launch_<N>.cu units each own one, summed by
// jt_debug_checks through jtl::checks_io<N>)
static __device__ unsigned long long jt_check_count;
static __device__ int jt_check_line;
__device__ __forceinline__ bool chk(bool ok, int line) {
  if (!ok && atomicAdd(&jt_check_count, 1ull) == 0ull) jt_check_line = line;
  return ok;
}
#if JT_CHECKS
#define JT_CHK(cond) (::jtk::chk((cond), __LINE__))
#else
#define JT_CHK(cond) true
#endif
// Schedule fuzzing (checks build only): before every synchronisation point (group barriers, ring waits and releases,
// cluster barriers) a thread sometimes sleeps for up to ~1 us, so warps reach shared data in orders the normal build
// rarely produces; a missing barrier then shows up as a parity failure or as two runs that differ (the checks test
// runs every case twice and compares the bits).
#ifndef JT_JITTER
#define JT_JITTER JT_CHECKS
#endif
__device__ __forceinline__ void jitter() {
#if JT_JITTER
  unsigned t = (unsigned)clock64() * 2654435761u + threadIdx.x * 40503u + blockIdx.x * 977u;
  t ^= t >> 13;
  if ((t & 7u) == 0u) __nanosleep(t & 1023u);
  __syncwarp();
#endif
}

// Phase trace (dev builds only, -DJT_PHASES=1, tools/phases.py): thread 0 of every CTA records clock64 at the
// phase boundaries of its first batch and prints them with the kernel's globaltimer start / end, so the critical
// path of the latency-bound launches (configs 1-2) can be split into prologue, loads, terms and reduction.
#ifndef JT_PHASES
#define JT_PHASES 0
#endif
struct Phases {
#if JT_PHASES
  long long t[11] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long g0 = 0;
  __device__ __forceinline__ Phases() {
    if (threadIdx.x == 0) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
      t[0] = clock64();
    }
  }
  __device__ __forceinline__ void mark(int i, bool on = true) {
    if (threadIdx.x == 0 && on && t[i] == 0) t[i] = clock64();
  }
  __device__ __forceinline__ void print(int kind, int n, int terms, long long inner) {
    if (threadIdx.x == 0) {
      unsigned long long g1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
      const long long e = clock64();
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      printf("PH k%d_i%lld n%d cta%d sm%u terms%d g0 %llu g1 %llu d %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld\n",
             kind, inner, n, (int)blockIdx.x, smid, terms, g0, g1, t[1] - t[0], t[2] - t[0], t[3] - t[0], t[4] - t[0],
             t[5] - t[0], t[6] - t[0], t[8] ? t[8] - t[0] : 0, t[9] ? t[9] - t[0] : 0, t[10] ? t[10] - t[0] : 0,
             t[7] - t[0], e - t[0]);
    }
  }
#else
  __device__ __forceinline__ void mark(int, bool = true) {}
  __device__ __forceinline__ void print(int, int, int, long long) {}
#endif
};

// Programmatic dependent launch (JT_PDL, launch.cuh launch_axis_kernel): every axis kernel lets the next kernel of
// the stream launch at once (its CTAs are placed as this one's exit) and waits for the previous kernel's completion
// and memory before its first access to the arrays; without the launch attribute both are no-ops.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

constexpr int K0MAX = 32;   // largest dense low-degree block (jt_opts.k0)
constexpr int VST_KPT = 2;  // degrees of W V staged per rank term (N <= 512), read as double2 pairs
constexpr int VST_KPT_PAIR = 4;  // ... per FFT of the PAIR kernels (half as many terms: the whole block stays in the ring)
                            // (4 measured slower: a bigger stage leaves room for only 2 ring stages)
constexpr int SMEM_LIMIT = 227 * 1024;

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

// Total entries of the per-pass twiddle tables (TwOff of the pass after the last).
template <int N, int R, int P = Pass<N, R, 1>::RS>
struct TwTotal {
  static constexpr int value = (Pass<N, R, P>::RS - 1) * P + TwTotal<N, R, P * Pass<N, R, P>::RS>::value;
};
template <int N, int R>
struct TwTotal<N, R, N> {
  static constexpr int value = 0;
};

// Twiddles a thread applies per FFT (complex values): passes after the first, B butterflies of RS - 1 each.
template <int N, int R, int P = Pass<N, R, 1>::RS>
struct TwPerThread {
  static constexpr int value = Pass<N, R, P>::B * (Pass<N, R, P>::RS - 1) + TwPerThread<N, R, P * Pass<N, R, P>::RS>::value;
};
template <int N, int R>
struct TwPerThread<N, R, N> {
  static constexpr int value = 0;
};
// ... of the passes before the one at sub-size NS
template <int N, int R, int NS, int P = Pass<N, R, 1>::RS>
struct TwPrefix {
  static constexpr int value =
      (P >= NS) ? 0 : Pass<N, R, P>::B * (Pass<N, R, P>::RS - 1) + TwPrefix<N, R, NS, P * Pass<N, R, P>::RS>::value;
};
template <int N, int R, int NS>
struct TwPrefix<N, R, NS, N> {
  static constexpr int value = 0;
};

template <int N_, int R_, int MAXR_, bool INV_, bool WG_ = false, bool PAIR_ = false>
struct Cfg {
  static constexpr int N = N_, R = R_, MAXR = MAXR_;
  static constexpr bool INV = INV_;
  // PAIR (forward only): two REAL rank terms per complex FFT.  The plan's paired factor set (jt_internal.h
  // AxisHost::pair) has real v'_l, so X_l = F_N(v'_l (.) a) is conjugate-symmetric and the terms (l, l') share the FFT
  // Z = F_N((v'_l + i v'_l') e^{i pi k / N} (.) a) on the half-integer bin grid m + 1/2:
  //   Re(u_l X_l[m] + u_l' X_l'[m]) = Re(P Z[m]) + Re(conj(Q) Z[N - 1 - m]),  P = (u_l - i u_l') / 2, Q = (u_l + i u_l') / 2.
  // A1 and the FFT are unchanged (the "v" of a pair is complex); the last pass's butterflies are dealt so that a thread
  // owns bin m and its mirror N - 1 - m (last_v), nothing of the last butterflies is pruned, and A3 reads two factor
  // rows (P, conj(Q)) per node: UROWS = 2 MAXR rows per bin in u~.  Bins are 0 .. N/2 - 1 (no Nyquist slot).
  static constexpr bool PAIR = PAIR_;
  static constexpr int UROWS = PAIR_ ? 2 * MAXR_ : MAXR_;
  // WG: one warp per group (LG = 32 / TPL lines) -- only for the term-split launches of few lines, which are
  // latency-bound (no named barriers: 256^2 0.041 -> 0.033 ms); the large launches keep 4 lines per group,
  // whose factor loads serve twice the lines per wavefront (one-warp groups measured +15 % at 512^3)
  static constexpr bool WG = WG_;
  static constexpr int TPL = N / R;                                     // threads per line
  // lines per group (2 lines at TPL = 128 was measured 6 % slower at N = 4096: one 8-warp barrier domain)
  // (WG applies to TPL = 16 only: at TPL = 32 one-line warps measured slower, 1024 x 64 inverse +7 %)
  static constexpr int LG = TPL <= 8 ? 32 / TPL : (TPL <= 32 ? (WG && TPL == 16 ? 2 : 4) : (N == 4096 && R == 32 ? JT_LG4096 : 1));
  static constexpr int GT = TPL * LG;                                   // threads per group
  static constexpr int GW = GT / 32;                                    // warps per group
  static constexpr int NSL = LastNS<N, R>::value;                       // the last pass starts at sub-size NSL
  static constexpr int RSL = Pass<N, R, NSL>::RS;                       // ... with radix RSL
  static constexpr int NB = R / 2 + 1;                                  // bins per thread (R/2 + Nyquist slot)
  static constexpr int NBINS = N / 2 + 1;
  // bin slots per thread in the row-range table and (inverse) the input state: the PAIR inverse also holds the rows
  // of its first-pass MIRROR positions' bins (slots R/2 .. R-1, see inv_axis_kernel)
  static constexpr int NBT = (PAIR_ && INV_) ? R_ : R_ / 2 + 1;
  // Register budget (32-bit registers): a thread holds x (4R), its persistent input state (the
  // coefficients a, or the inverse's input-bin values: 2R resp. 2 NB MAXR) and its output accumulators
  // (the forward's bin rows y: 2 NB MAXR, or the inverse's acc: 2R).  For R >= 32 that exceeds 255, so
  // the input state lives in a thread-private SMEM area (PRIV), read once per term (8 B per point), and
  // the exchange runs one real plane at a time (SPLITX) to leave SMEM for the factor ring.
  static constexpr bool PRIV = R >= 32 || (JT_PRIV16 && N >= 64);
  // PRIV state in tensor memory (TPRIV, tcgen05.ld/st): frees the SMEM crossbar of the per-term state re-reads
  static constexpr bool TPRIV = PRIV && JT_TPRIV && N <= JT_TPRIV_NMAX;
  // exchange one real plane at a time (3 group barriers per exchange) only while SMEM is short: with the state
  // in TMEM the full complex exchange (1 barrier) fits
  // (SUB: the split exchange halves the exchange buffers, room for a ring deeper than one term)
  static constexpr bool SPLITX = R >= 32 && (!TPRIV || JT_SPLITX_TPRIV || (N == 4096 && MAXR == 2 && JT_SUB && JT_SUB_SPLITX));

  static constexpr int XB = SPLITX ? 8 : 16;  // bytes per exchange slot
  // (MAXR = 4: twice the row accumulators / bin rows per thread)
  static constexpr int REGS = R >= 32 ? 255
                                      : (PRIV ? (MAXR > 3 ? JT_REGS16M4 : MAXR == 3 ? JT_REGS16M3 : (INV ? JT_REGS16 : JT_REGS16F))
                                              : (MAXR > 2 ? 200 : 168));
  // exchange buffer: slots [pos][line], LG pad slots after every R positions -> the strided first-pass
  // stores and the unit-stride loads are both free of bank conflicts
  static constexpr int SLOTS = Pass<N, R, 1>::LAST ? 0 : (N + N / R) * LG;
  static constexpr int PSTATE = PRIV ? (INV ? NBT * MAXR : R) : 0;  // private doubles per thread (inverse: bin rows)
  static constexpr int PSLOTS = TPRIV ? 0 : PSTATE;                           // ... of them in SMEM
  // + (inverse) the per-warp partial sums of (W V)^T y (K0MAX x GW x LG)
  static constexpr int VRED = INV ? K0MAX * GW * LG : 0;
  static constexpr int GROUP_BYTES = ((SLOTS * XB + K0MAX * LG * 8 + PSLOTS * GT * 8 + VRED * 8) + 127) / 128 * 128;
  // factor ring: stage = v_l (N complex) + u~_l (MAXR x NBINS complex) [+ chunk l of W V (VST): KPT degrees,
  // layout [m][c][kk], so the dense low-degree block is applied inside the term loop from SMEM]
  static constexpr bool STAGED = N <= 1024;
  // N > 1024 forward: u~_l (the epilogue's factor, 32-64 KB) through a one-stage TMA ring in the SMEM left
  // next to the exchange buffers (URING), filled a whole term ahead of its use; v_l still through L1
// (measured: N = 2048 forward -5 %; N = 4096 +8 %: its 64 KB stage leaves too little L1 for the v_l loads)
  static constexpr bool URING_WANT = !STAGED && !INV && JT_URING && N <= JT_URING_NMAX;
  // N = 4096 (SUB): a term's factors (128 KB) do not fit a stage, so they stream through a ring of 16 KB SUB-stages
  // shared by the CTA's groups, in the order the term consumes them -- forward: v_l in 4 blocks of 1024 positions
  // (A1), then u~_l in 4 blocks of bins (A3); inverse: u~_l in 4 bin blocks (bin sums), then v_l in 4 blocks
  // (accumulate) -- each released per WARP as soon as its values are in registers (no extra group barrier); the
  // last warp to release a slot refills it NSTAGE sub-stages ahead.  Replaces the L1/L2 factor loads (the top
  // stall of these passes, long-scoreboard, 40x the algorithmic bytes through L2).
  static constexpr bool SUB = N == 4096 && R == 32 && MAXR == 2 && JT_SUB;
  static constexpr int SUBB = 16384, NSUB = 8;  // bytes per sub-stage, sub-stages per term
  static constexpr bool VST = N <= 512;
  static constexpr int VUN = VST ? 1 : JT_VUNROLL;  // unroll of the batch-start W V loops
  static constexpr int KPT = VST ? (PAIR ? VST_KPT_PAIR : VST_KPT) : 0;
  static constexpr int V_BYTES = N * 16, U_BYTES = UROWS * NBINS * 16, PH_BYTES = KPT * MAXR * NBINS * 8;
  static constexpr int SV_BYTES = STAGED ? V_BYTES : 0;  // v_l bytes in a ring stage (URING stages hold u~_l only)
  static constexpr int STAGE_BYTES =
      SUB ? SUBB
          : (STAGED ? (V_BYTES + U_BYTES + PH_BYTES + 127) / 128 * 128 : (URING_WANT ? (U_BYTES + 127) / 128 * 128 : 0));
  // twiddle tables of the passes after the first, copied to SMEM (TWS): every twiddle is one broadcast
  // LDS.128 instead of a chain of complex multiplies
  static constexpr bool TWS = N <= 1024;
  // ... and with the state in TMEM, each thread's own twiddles (constant for the kernel) in its TMEM slice (TWT)
  static constexpr int TWPT = TwPerThread<N, R>::value;  // complex twiddles per thread
  // (MAXR 4: slice too small; the R = 32 inverse measured 2 % slower with it)
// twiddles per TMEM wait in the N > 1024 passes (measured: forward 4 -5 % vs 8 at N = 4096; inverse 8 -3 % at 2048)
  // N > 1024 (no SMEM table, TWS off): the twiddles in TMEM too, one copy per lane quadrant shared by the warps
  // of that quadrant (TW_SHARED: warps w and w + 4 have the same thread positions vt when the group size
  // divides 128), after all the warps' state slices
  static constexpr bool TWT_LARGE = !TWS && JT_TWT_LARGE && 128 % GT == 0 && (!INV || N <= JT_TWT_LARGE_INV_NMAX);
  static constexpr bool TWT = (TWS || TWT_LARGE) && TPRIV && JT_TWT && TWPT > 0 && MAXR == 2 &&
                              (!INV || R == 16 || JT_TWT_INV32 || !TWS);
  static constexpr bool TW_SHARED = TWT && !TWS;
  static constexpr bool VTM_PRE = JT_VTM && N == 512 && R == 32 && MAXR == 2 && !INV && !WG;  // (see VTM)
  // VTM (N = 512 forward): the rank term's v_l read from tensor memory instead of broadcast LDS.128s (64 of the 456
  // shared-memory wavefronts per warp and term): one thread copies the ring stage's v_l into TMEM with tcgen05.cp
  // (.32x128b.warpx4, stride-0 core matrices: each 8-row block of v repeated down a lane quadrant), so the lanes are
  // mapped line-major (lane = 8 line + vt % 8) and the exchange slots line-major too; block A (vt 0..7) and B
  // (vt 8..15) both go to every quadrant, quadrants 0, 2 read A and 1, 3 read B; the twiddles are one copy per
  // quadrant (its two warps have the same vt) -- 64 + 64 (states) + 128 (twiddles) + 2 x 128 (v) = 512 columns.
  static constexpr bool VTM = VTM_PRE && LG == 4 && GT == 64 && STAGED && TWT && TWS;
  static constexpr bool TW_QSHARE = TW_SHARED || VTM;  // one twiddle copy per lane quadrant
  static constexpr int TW_BYTES = (TWS && !TWT) ? (TwTotal<N, R>::value * 16 + 127) / 128 * 128 : 0;
  // per-CTA table of the row range of every (thread position vt, bin slot q): (j0 << 4) | count
  static constexpr int BINFO_BYTES = STAGED ? (TPL * NBT * 4 + 127) / 128 * 128 : 0;
  static constexpr int VTM_BYTES = VTM_PRE ? 16 : 0;  // (VTM: v-ready mbarrier + v-consumed counter after the ring)
  static constexpr int hdr_bytes(int nstage) {
    return (nstage * STAGE_BYTES + 3 * nstage * 8 + VTM_BYTES + 127) / 128 * 128 + BINFO_BYTES + TW_BYTES;
  }
  static constexpr int gpc_fit(int g, int nstage) {
    return (g > 1 && (((g * GT + 127) / 128) * 128 * REGS > 65536 || g * GROUP_BYTES + hdr_bytes(nstage) > SMEM_LIMIT ||
                      g > 15 || g * GT > 1024))  // named barriers 1..15 (one per group)
               ? gpc_fit(g - 1, nstage)
               : g;
  }
  // groups per CTA (one CTA per SM; the one-warp-group term-split configurations can cap it at JT_WG_GPC so that
  // two CTAs share an SM: twice the CTAs, each with fewer rank terms)
  static constexpr int GPC = (WG && JT_WG_GPC < gpc_fit(8, STAGED ? 2 : (SUB ? 4 : 1))) ? JT_WG_GPC
                                                                                   : gpc_fit(8, STAGED ? 2 : (SUB ? 4 : 1));
  static constexpr int MINB = WG && JT_WG_GPC < 8 ? 2 : 1;  // __launch_bounds__ min blocks
  // LATE: no group barrier at the end of a rank term; the exchange buffer's reuse is guarded by a barrier just
  // before the next term's first exchange store (and a ring stage, where there is one, is released per warp), so a
  // warp can run into the next term's column scale and first DFT pass ahead of its group's other warps.  Measured
  // (tools/ab_time.py, r02i): N = 4096 forward (no ring) 3.54 -> 3.45 ms at 4096^2; everywhere else slower (the
  // per-warp ring releases cost more than the barrier: 512^3 +3.8 %, 4096 inverse +6 %), so only there.
  static constexpr bool LATE = JT_LATE_SYNC && !SUB && !INV && !STAGED && !URING_WANT;
  // forward column scale folded into the radix-32 first pass's first butterfly layer (fft_regs.cuh dft4_pre): 32 fewer
  // FP64 instructions per thread and term; measured (r02x) 4096^2 forward 3.46 -> 3.37 ms, but 512^3 +0.75 %, 1024
  // +1.2 %, 128 +1.6 % (the MUL -> FMA chain lengthens the dependent path), so only for N >= JT_A1_FOLD_NMIN
  static constexpr bool A1FOLD = JT_A1_FOLD && N >= JT_A1_FOLD_NMIN && !INV && R == 32 && Pass<N, R, 1>::RS == 32 &&
                                 Pass<N, R, 1>::B == 1 &&
                                 PRIV && !SUB && (!(JT_LOADS_FIRST & 1) || STAGED || !TPRIV);
  static constexpr bool URING = URING_WANT && GPC * GROUP_BYTES + hdr_bytes(1) <= SMEM_LIMIT;
  static constexpr int sub_fit(int s) { return (s > 4 && GPC * GROUP_BYTES + hdr_bytes(s) > SMEM_LIMIT) ? sub_fit(s - 1) : s; }
  // a third ring stage when it fits next to the GPC groups; SUB: as many sub-stages as fit (<= one term)
  static constexpr int NSTAGE = SUB ? sub_fit(12)
                                    : ((STAGED && GPC * GROUP_BYTES + hdr_bytes(3) <= SMEM_LIMIT) ? 3 : (URING ? 1 : 2));
  static_assert(!SUB || GPC * GROUP_BYTES + hdr_bytes(NSTAGE) <= SMEM_LIMIT, "SUB ring");
  static constexpr int RING_BYTES = NSTAGE * STAGE_BYTES + 3 * NSTAGE * 8;  // stages + full/empty barriers + counters
  static constexpr int BINFO_OFF = (RING_BYTES + VTM_BYTES + 127) / 128 * 128;
  static constexpr int TW_OFF = BINFO_OFF + BINFO_BYTES;
  static constexpr int HDR_BYTES = hdr_bytes(NSTAGE);
  static constexpr int NT = GPC * GT;  // threads per CTA
  static constexpr size_t smem_bytes() { return (size_t)HDR_BYTES + (size_t)GPC * GROUP_BYTES; }
  // term-split partial lines of a batch (GPC LG lines x N doubles) fit in the group areas (cluster reduction)
  static constexpr bool CLUSTER_FIT = (long long)GPC * LG * N * 8 <= (long long)GPC * GROUP_BYTES;
  __device__ static __forceinline__ int sidx(int pos, int line) {
    // (VTM: line-major with one pad slot per 32 -- conflict-free for its lane = 8 line + vt % 8 mapping)
    if constexpr (VTM) return line * (N + N / 32) + pos + pos / 32;
    else return (pos + pos / R) * LG + line;
  }
  static_assert(GT % 32 == 0, "group must be whole warps");
  static_assert(!PAIR || INV || (MAXR == 2 && Pass<N, R, NSL>::B % 2 == 0 && Pass<N, R, NSL>::B * TPL == N / RSL &&
                                 NSL > 1 && !VTM_PRE && !SUB),
                "PAIR forward: an even number of last-pass butterflies per thread");
  static_assert(!PAIR || !INV || (MAXR == 2 && Pass<N, R, 1>::B == 1 && Pass<N, R, 1>::RS == R && PRIV && !SUB),
                "PAIR inverse: one radix-R first-pass butterfly per thread (positions vt + r TPL)");
  static_assert(RSL >= 2, "last pass radix");
  static_assert(smem_bytes() <= SMEM_LIMIT, "shared memory");
  // TMEM: 512 columns; the NT/32 warps share the 4 lane quadrants, each warp a column slice of TCOLS
  static constexpr int NWARP = NT / 32;
  static constexpr int TCOLS = NWARP >= 4 ? 512 / (NWARP / 4) : 512;  // column slice per warp (upper bound)
  static constexpr int TW_COL0 = (PSTATE + 15) / 16 * 32;          // twiddles after the state chunks
  static constexpr int TW_COLS = TWT ? (4 * TWPT + 31) / 32 * 32 : 0;
  static constexpr int pow2_ge(int v, int p = 32) { return p >= v ? p : pow2_ge(v, 2 * p); }
  static constexpr int WPQ = (NWARP + 3) / 4;  // warps per lane quadrant
  // columns of a quadrant: WPQ slices [state | own twiddles], or (TW_SHARED) WPQ state slices + one twiddle copy
  // (+32: a butterfly's twiddle loads are whole 8-complex chunks and may read past the last one)
  static constexpr int V_COLA = WPQ * TW_COL0 + TW_COLS, V_COLB = V_COLA + 4 * R;  // VTM: v blocks A / B
  static constexpr int TUSED = VTM ? V_COLB + 4 * R
                                   : (TW_SHARED ? WPQ * TW_COL0 + TW_COLS + 32 : (TW_COL0 + TW_COLS) * WPQ);
  // allocate only what the slices use (a power of two >= 32), so CTAs that co-reside on an SM can all allocate
  static constexpr int TALLOC = pow2_ge(TUSED > 512 ? 512 : TUSED);
  static constexpr int TSTRIDE = TW_QSHARE ? TW_COL0 : TALLOC / WPQ / 16 * 16;
  static constexpr int TW_BASE = TW_QSHARE ? WPQ * TW_COL0 : TW_COL0;  // twiddles: from the quadrant / slice base
  static constexpr bool TMEM_OK =
      !TPRIV || (NWARP % 4 == 0 && (TW_QSHARE ? TUSED <= 512 : TW_COL0 + TW_COLS <= TCOLS));
  static_assert(!TPRIV || TW_QSHARE || TW_COL0 + TW_COLS <= TSTRIDE, "TMEM slice stride");
  static_assert(!VTM || (NWARP == 8 && TUSED == 512 && TW_COL0 == 64 && TW_COLS == 128), "VTM TMEM layout");
#ifndef JT_NO_TMEM_ASSERT
  static_assert(TMEM_OK, "TMEM state slice");
#endif
};

__device__ __forceinline__ const double2 *tw_smem_base(int off) {
  extern __shared__ __align__(128) char smem_raw[];
  return reinterpret_cast<const double2 *>(smem_raw + off);
}

template <class C>
__device__ __forceinline__ void group_sync() {
  jitter();
  if constexpr (C::GW == 1) {
    __syncwarp();
  } else {
    // non-.aligned form: correct even if a warp arrives diverged (PTX ISA, barrier.sync)
    asm volatile("barrier.sync %0, %1;" ::"r"(1 + (int)(threadIdx.x / C::GT)), "r"(C::GT) : "memory");
    // the threads a non-aligned barrier releases need not run converged: reconverge before the warp-collective
    // (.sync.aligned) tcgen05 loads that may follow (found by the checks build's schedule fuzzing)
    __syncwarp();
  }
}

// ---- mbarrier / TMA bulk-copy helpers (PTX ISA: mbarrier, cp.async.bulk) ---------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra WAIT;\n"
      "DONE:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Shared-memory matrix descriptor of a tcgen05.cp source (no swizzle; 8-row x 16-byte core matrices, rows 16 bytes
// apart): start address, leading / stride-dimension byte offsets 0 (a 128-bit-wide copy has one core matrix along K;
// stride 0 repeats the first core matrix down the copy's rows -- measured, tools/tmem_cp_probe.cu), version 1.
__device__ __forceinline__ uint64_t tmem_cp_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 46);
}

// The CTA's factor ring.  Sequence number seq = (batch iteration) r + l walks the terms of every batch
// the CTA processes; term seq lives in stage seq % NSTAGE, phase (seq / NSTAGE) & 1.
template <class C>
struct Ring {
  char *base;
  uint64_t *full, *empty;
  unsigned *cnt;    // per stage: groups that released it in the current phase (the last one refills it)
  long long total;  // terms this CTA will consume
  const double2 *gv, *gu;
  const double *gph;
  int r, k0;
  int l0 = 0, rs = 1;  // term range of this CTA: l0 .. l0 + rs - 1
  __device__ __forceinline__ double2 *v(long long seq) const {
    return reinterpret_cast<double2 *>(base + (seq % C::NSTAGE) * C::STAGE_BYTES);
  }
  __device__ __forceinline__ double2 *u(long long seq) const {
    return reinterpret_cast<double2 *>(base + (seq % C::NSTAGE) * C::STAGE_BYTES + C::SV_BYTES);
  }
  __device__ __forceinline__ const double *ph(long long seq) const {
    return reinterpret_cast<const double *>(base + (seq % C::NSTAGE) * C::STAGE_BYTES + C::SV_BYTES + C::U_BYTES);
  }
  __device__ __forceinline__ void issue(long long seq) const {  // producer: one thread
    if constexpr (C::SUB) {
      issue_sub(seq);
      return;
    }
    const int s = (int)(seq % C::NSTAGE);
    const int l = l0 + (int)(seq % rs);
    const bool kc = C::VST && l * C::KPT < k0;  // chunk l of W V exists (zero-padded to KPT degrees)
    const uint32_t ph_bytes = kc ? C::PH_BYTES : 0;
    if (!JT_CHK(l >= 0 && l < r)) {  // (checks build: complete the phase without copying, so nobody hangs)
      mbar_arrive_expect_tx(&full[s], 0);
      return;
    }
    mbar_arrive_expect_tx(&full[s], C::SV_BYTES + C::U_BYTES + ph_bytes);
    if constexpr (C::STAGED) tma_load_1d(v(seq), gv + (long long)l * C::N, C::V_BYTES, &full[s]);
    tma_load_1d(u(seq), gu + (long long)l * C::UROWS * C::NBINS, C::U_BYTES, &full[s]);
    if (kc)
      tma_load_1d(const_cast<double *>(ph(seq)), gph + (long long)l * C::KPT * C::MAXR * C::NBINS, ph_bytes, &full[s]);
  }
  // SUB: sub-stage seq = 8 t + part of the CTA's t-th term (term l0 + t % rs); 16 KB, laid out for the consumer:
  //   forward  part j < 4: v_l[1024 j .. 1024 j + 1023]                         (A1 of positions r in [8j, 8j + 8))
  //            part 4 + i: [c][h][256] = u~_l rows c of bins h 1024 + 256 i + [0, 256) (A3 of bins q in [4i, 4i + 4))
  //   inverse  part i < 4: [c][512]    = u~_l rows c of bins 512 i + [0, 512)          (bin sums of q in [4i, 4i + 4))
  //            part 4 + j: [h][256]    = v_l[1024 h + 256 j + [0, 256)]              (outputs e with e / 4 in {2j, 2j + 1})
  __device__ __forceinline__ void issue_sub(long long seq) const {
    const int s = (int)(seq % C::NSTAGE);
    const long long t = seq / C::NSUB;
    const int part = (int)(seq % C::NSUB);
    const int l = l0 + (int)(t % rs);
    if (!JT_CHK(l >= 0 && l < r)) {  // (checks build: complete the phase without copying, so nobody hangs)
      mbar_arrive_expect_tx(&full[s], 0);
      return;
    }
    mbar_arrive_expect_tx(&full[s], C::SUBB);
    char *dst = base + (long long)s * C::STAGE_BYTES;
    const double2 *vl = gv + (long long)l * C::N;
    const double2 *ul = gu + (long long)l * C::MAXR * C::NBINS;
    const int j = part & 3;
    if (C::INV ? part >= 4 : part < 4) {  // v_l
      if constexpr (!C::INV) {
        tma_load_1d(dst, vl + 1024 * j, 16384, &full[s]);
      } else {
#pragma unroll
        for (int h = 0; h < 4; ++h) tma_load_1d(dst + 4096 * h, vl + 1024 * h + 256 * j, 4096, &full[s]);
      }
    } else {  // u~_l
      if constexpr (!C::INV) {
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            tma_load_1d(dst + 4096 * (2 * c + h), ul + (long long)c * C::NBINS + 1024 * h + 256 * j, 4096, &full[s]);
      } else {
#pragma unroll
        for (int c = 0; c < 2; ++c) tma_load_1d(dst + 8192 * c, ul + (long long)c * C::NBINS + 512 * j, 8192, &full[s]);
      }
    }
  }
  __device__ __forceinline__ void wait_full(long long seq) const {
    jitter();
    mbar_wait(&full[seq % C::NSTAGE], (uint32_t)((seq / C::NSTAGE) & 1));
    __syncwarp();  // lanes may leave the try_wait loop in different iterations: reconverge
  }
  // SUB: every warp releases each sub-stage once its lanes' values are in registers; the last of the CTA's warps
  // refills the slot with sub-stage seq + NSTAGE (same acq_rel counter / proxy fence protocol as release()).
  __device__ __forceinline__ void release_warp(long long seq) const {
    jitter();
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      const int s = (int)(seq % C::NSTAGE);
      unsigned old;
      asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(smem_u32(&cnt[s])) : "memory");
      if (old == C::NWARP - 1) {
        cnt[s] = 0;
        if (seq + C::NSTAGE < total) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(seq + C::NSTAGE);
        }
      }
    }
    __syncwarp();
  }
  __device__ __forceinline__ const double2 *slot(long long seq) const {
    return reinterpret_cast<const double2 *>(base + (seq % C::NSTAGE) * C::STAGE_BYTES);
  }
  // Called by every thread of every group after its end-of-term group_sync.  The group's thread 0 counts the
  // release; the LAST group to release the stage refills it (no thread ever blocks on the slowest group).
  // The counter is a CTA-scope acq_rel atomic: every group's reads of the stage happen before its
  // increment, the refill after the last one; the proxy fence orders those generic-proxy reads before
  // the async-proxy (TMA) writes of the refill.
  __device__ __forceinline__ void release(long long seq, int gt) const {
    jitter();
    if (gt == 0) {
      const int s = (int)(seq % C::NSTAGE);
      unsigned old;
      asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(smem_u32(&cnt[s])) : "memory");
      if (old == C::GPC - 1) {
        cnt[s] = 0;
        if (seq + C::NSTAGE < total) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(seq + C::NSTAGE);
        }
      }
    }
    // reconverge before the group's next (warp-aligned) bar.sync: bar.sync from a diverged warp is
    // undefined and released the barrier early (a race seen on 512^3 axis-0 lines)
    __syncwarp();
  }
};

// ---- Stockham passes over the group's exchange buffer -------------------------------------------------

// Butterfly index (0 .. N/RS - 1) of a thread's i-th butterfly in the pass at sub-size NS: vt + i TPL, except in
// the LAST pass of the PAIR kernels, where butterflies 2h and 2h + 1 are v and its mirror N/RS - 1 - v, so that the
// thread's outputs v + s N/RS and (N/RS - 1 - v) + (RS - 1 - s) N/RS = N - 1 - (v + s N/RS) are a conjugate-mirror pair.
template <class C, int NS>
__device__ __forceinline__ int pass_v(int vt, int i) {
  using P = Pass<C::N, C::R, NS>;
  if constexpr (C::PAIR && !C::INV && P::LAST) {
    const int v = vt + (i / 2) * C::TPL;
    return (i & 1) ? C::N / P::RS - 1 - v : v;
  } else {
    return vt + i * C::TPL;
  }
}

// Store one real plane (SPLITX) or both (interleaved double2) of the outputs of the pass at sub-size NS.
template <class C, int NS>
__device__ __forceinline__ void pass_store(const double (&xr)[C::R], const double (&xi)[C::R], void *buf, int vt,
                                           int line, int plane) {
  using P = Pass<C::N, C::R, NS>;
#pragma unroll
  for (int i = 0; i < P::B; ++i) {
    const int v = vt + i * C::TPL;
    const int idxD = (v / NS) * NS * P::RS + (v % NS);
#pragma unroll
    for (int s = 0; s < P::RS; ++s) {
      const int sl = C::sidx(idxD + s * NS, line);
      if (!JT_CHK(sl >= 0 && sl < C::SLOTS)) continue;
      if constexpr (C::SPLITX) {
        static_cast<double *>(buf)[sl] = plane == 0 ? xr[i * P::RS + s] : xi[i * P::RS + s];
      } else {
        static_cast<double2 *>(buf)[sl] = make_double2(xr[i * P::RS + s], xi[i * P::RS + s]);
      }
    }
  }
}

// Load the inputs of the pass at sub-size NS (one plane, or both).
template <class C, int NS>
__device__ __forceinline__ void pass_load(double (&xr)[C::R], double (&xi)[C::R], const void *buf, int vt, int line,
                                          int plane) {
  using P = Pass<C::N, C::R, NS>;
  constexpr int RS = P::RS;
#pragma unroll
  for (int i = 0; i < P::B; ++i) {
    const int v = pass_v<C, NS>(vt, i);
#pragma unroll
    for (int r = 0; r < RS; ++r) {
      const int sl = C::sidx(v + r * (C::N / RS), line);
      if (!JT_CHK(sl >= 0 && sl < C::SLOTS)) continue;
      if constexpr (C::SPLITX) {
        if (plane == 0) xr[i * RS + r] = static_cast<const double *>(buf)[sl];
        else xi[i * RS + r] = static_cast<const double *>(buf)[sl];
      } else {
        const double2 d = static_cast<const double2 *>(buf)[sl];
        xr[i * RS + r] = d.x;
        xi[i * RS + r] = d.y;
      }
    }
  }
}

// Twiddle and radix-RS butterflies of the pass at sub-size NS (inputs already in registers).
template <class C, int NS>
__device__ __forceinline__ void pass_compute(double (&xr)[C::R], double (&xi)[C::R], int vt,
                                             const double2 *__restrict__ tw, uint32_t ttw) {
  using P = Pass<C::N, C::R, NS>;
  constexpr int RS = P::RS;
  if constexpr (C::TW_SHARED) {
    // this thread's twiddles of the pass (butterfly i, r = 1..RS-1, consecutive in TMEM), TCH complex per wait
    // across butterfly boundaries (the radix-2 / radix-4 last passes of N > 1024 have 1 / 3 per butterfly),
    // then the DFTs
    constexpr int NTW = P::B * (RS - 1);
    constexpr int TCH = C::INV ? JT_TWT_CH_LARGE_I : JT_TWT_CH_LARGE_F;
    const uint32_t t0 = ttw + 4 * TwPrefix<C::N, C::R, NS>::value;
#pragma unroll
    for (int ch = 0; ch < (NTW + TCH - 1) / TCH; ++ch) {
      double w[16];
      tmem_ld_d8(t0 + 4 * TCH * ch, &w[0]);
      if constexpr (TCH == 8) tmem_ld_d8(t0 + 4 * TCH * ch + 16, &w[8]);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < TCH; ++j) {
        const int k = TCH * ch + j;
        if (k < NTW) {
          const int e = (k / (RS - 1)) * RS + 1 + k % (RS - 1);
          const double pr = w[2 * j], pim = w[2 * j + 1];
          const double tr = xr[e] * pr - xi[e] * pim;
          xi[e] = fma(xr[e], pim, xi[e] * pr);
          xr[e] = tr;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < P::B; ++i) dft<RS>(&xr[i * RS], &xi[i * RS]);
  } else if constexpr (C::TWT && JT_TW_PREISSUE) {
    // as below, but each chunk's TMEM loads are issued one chunk ahead, so the loads of butterfly i + 1's first chunk
    // are in flight during butterfly i's DFT (one exposed TMEM latency per pass instead of one per chunk)
    constexpr int NCHK = (RS - 1 + 7) / 8;
    const uint32_t tb = ttw + 4 * TwPrefix<C::N, C::R, NS>::value;
    double w[16];
    tmem_ld_d8(tb, &w[0]);
    tmem_ld_d8(tb + 16, &w[8]);
#pragma unroll
    for (int i = 0; i < P::B; ++i) {
#pragma unroll
      for (int ch = 0; ch < NCHK; ++ch) {
        tmem_wait_ld();
        double wc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) wc[j] = w[j];
        if (ch + 1 < NCHK || i + 1 < P::B) {
          const uint32_t tn = ch + 1 < NCHK ? tb + 4 * (i * (RS - 1)) + 32 * (ch + 1) : tb + 4 * ((i + 1) * (RS - 1));
          tmem_ld_d8(tn, &w[0]);
          tmem_ld_d8(tn + 16, &w[8]);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int r = 1 + 8 * ch + j;
          if (r < RS) {
            const double pr = wc[2 * j], pim = wc[2 * j + 1];
            const double tr = xr[i * RS + r] * pr - xi[i * RS + r] * pim;
            xi[i * RS + r] = fma(xr[i * RS + r], pim, xi[i * RS + r] * pr);
            xr[i * RS + r] = tr;
          }
        }
      }
      dft<RS>(&xr[i * RS], &xi[i * RS]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < P::B; ++i) {
      const int v = pass_v<C, NS>(vt, i);
      if constexpr (C::TWT) {
        // this thread's twiddles w^r, r = 1..RS-1, from its TMEM slice, 8 complex per tcgen05.ld pair
        constexpr int NCHK = (RS - 1 + 7) / 8;
        const uint32_t t0 = ttw + 4 * (TwPrefix<C::N, C::R, NS>::value + i * (RS - 1));
#pragma unroll
        for (int ch = 0; ch < NCHK; ++ch) {
          double w[16];
          tmem_ld_d8(t0 + 32 * ch, &w[0]);
          tmem_ld_d8(t0 + 32 * ch + 16, &w[8]);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int r = 1 + 8 * ch + j;
            if (r < RS) {
              const double pr = w[2 * j], pim = w[2 * j + 1];
              const double tr = xr[i * RS + r] * pr - xi[i * RS + r] * pim;
              xi[i * RS + r] = fma(xr[i * RS + r], pim, xi[i * RS + r] * pr);
              xr[i * RS + r] = tr;
            }
          }
        }
        dft<RS>(&xr[i * RS], &xi[i * RS]);
        continue;
      }
      // Twiddles w^r, w = e^{2 pi i (v mod NS) / (NS RS)}: every one from the SMEM table (TWS), or exact table
      // values at the anchors r = 1 (mod 8) and the chain w^r = w^{r-1} w in between (from global / L1).
      double pr = 1.0, pim = 0.0;
      double2 w1;
      const double2 *twp;
      if constexpr (C::TWS) {
        twp = tw_smem_base(C::TW_OFF) + TwOff<C::N, C::R, NS>::value + (v % NS);
      } else {
        twp = tw + TwOff<C::N, C::R, NS>::value + (v % NS);
        w1 = __ldg(&twp[0]);
      }
#pragma unroll
      for (int r = 1; r < RS; ++r) {
        if constexpr (C::TWS) {  // every twiddle from the SMEM table
          const double2 wa = twp[(r - 1) * NS];
          pr = wa.x;
          pim = wa.y;
        } else if (r % 8 == 1) {
          const double2 wa = r == 1 ? w1 : __ldg(&twp[(r - 1) * NS]);
          pr = wa.x;
          pim = wa.y;
        } else {
          const double t = pr * w1.x - pim * w1.y;
          pim = fma(pr, w1.y, pim * w1.x);
          pr = t;
        }
        const double tr = xr[i * RS + r] * pr - xi[i * RS + r] * pim;
        xi[i * RS + r] = fma(xr[i * RS + r], pim, xi[i * RS + r] * pr);
        xr[i * RS + r] = tr;
      }
      dft<RS>(&xr[i * RS], &xi[i * RS]);
    }
  }
}

// Fill this thread's TMEM twiddle slice (C::TWT): for each pass after the first, for each of its butterflies i,
// w^r (r = 1..RS-1) with w = e^{2 pi i (v mod NS) / (NS RS)}, v = vt + i TPL, copied from the global tables.
template <class C, int NS>
__device__ __forceinline__ void tw_fill(double *buf, int vt, const double2 *__restrict__ tw) {
  if constexpr (NS < C::N) {
    using P = Pass<C::N, C::R, NS>;
#pragma unroll
    for (int i = 0; i < P::B; ++i) {
      const int v = pass_v<C, NS>(vt, i);
#pragma unroll
      for (int r = 1; r < P::RS; ++r) {
        const double2 w = __ldg(&tw[TwOff<C::N, C::R, NS>::value + (r - 1) * NS + (v % NS)]);
        const int k = TwPrefix<C::N, C::R, NS>::value + i * (P::RS - 1) + (r - 1);
        buf[2 * k] = w.x;
        buf[2 * k + 1] = w.y;
      }
    }
    tw_fill<C, NS * P::RS>(buf, vt, tw);
  }
}

// Exchange the outputs of the pass that started at NSS (in registers) into the inputs of the pass at
// NS = NSS RS(NSS).  On entry every thread of the group has finished reading the buffer.
template <class C, int NSS>
__device__ __forceinline__ void do_exchange(double (&xr)[C::R], double (&xi)[C::R], void *buf, int vt, int line) {
  constexpr int NS = NSS * Pass<C::N, C::R, NSS>::RS;
  if constexpr (C::SPLITX) {
    pass_store<C, NSS>(xr, xi, buf, vt, line, 0);
    group_sync<C>();
    pass_load<C, NS>(xr, xi, buf, vt, line, 0);
    group_sync<C>();
    pass_store<C, NSS>(xr, xi, buf, vt, line, 1);
    group_sync<C>();
    pass_load<C, NS>(xr, xi, buf, vt, line, 1);
  } else {
    pass_store<C, NSS>(xr, xi, buf, vt, line, 0);
    group_sync<C>();
    pass_load<C, NS>(xr, xi, buf, vt, line, 0);
  }
}

template <class C, int NS>
__device__ __forceinline__ void run_passes(double (&xr)[C::R], double (&xi)[C::R], void *buf, int vt, int line,
                                           const double2 *__restrict__ tw, uint32_t ttw) {
  if constexpr (NS < C::N) {
    pass_compute<C, NS>(xr, xi, vt, tw, ttw);
    if constexpr (!Pass<C::N, C::R, NS>::LAST) {
      group_sync<C>();
      do_exchange<C, NS>(xr, xi, buf, vt, line);
      run_passes<C, NS * Pass<C::N, C::R, NS>::RS>(xr, xi, buf, vt, line, tw, ttw);
    }
  }
}

// Full FFT of one term; first-pass inputs (positions vt + r TPL) in registers on entry, last-pass
// outputs (positions out_pos) in registers on exit.  The caller syncs the group before the next call.
// Z: the first-pass inputs above position R/2 of the thread are zero (the inverse: bins > N/2 hold no rows)
template <class C, bool PRE = false, bool Z = false>
__device__ __forceinline__ void fft(double (&xr)[C::R], double (&xi)[C::R], void *buf, int vt, int line,
                                    const double2 *__restrict__ tw, uint32_t ttw) {
  using P0 = Pass<C::N, C::R, 1>;
  static_assert(!PRE || (P0::RS == 32 && P0::B == 1), "PRE: one radix-32 first pass");
  constexpr bool ZZ = Z && JT_ZFIRST && P0::B == 1 && (P0::RS == 16 || P0::RS == 32);
#pragma unroll
  for (int i = 0; i < P0::B; ++i) dft<P0::RS, PRE, ZZ>(&xr[i * P0::RS], &xi[i * P0::RS]);
  if constexpr (!P0::LAST) {
    if constexpr (C::LATE) group_sync<C>();  // every thread of the group has read the previous term's exchange
    do_exchange<C, 1>(xr, xi, buf, vt, line);
    run_passes<C, P0::RS>(xr, xi, buf, vt, line, tw, ttw);
  }
}

// Frequency index of last-pass output register e = i RSL + s.
template <class C>
__device__ __forceinline__ int out_pos(int vt, int e) {
  return pass_v<C, C::NSL>(vt, e / C::RSL) + (e % C::RSL) * (C::N / C::RSL);
}

// PAIR: the register holding the conjugate-mirror bin N - 1 - m of last-pass output register e = i RSL + s:
// butterfly i ^ 1 (pass_v), output RSL - 1 - s.
template <class C>
__device__ __forceinline__ constexpr int mirror_reg(int e) {
  return ((e / C::RSL) ^ 1) * C::RSL + (C::RSL - 1 - e % C::RSL);
}

// Forward: the thread's output bins q = i (RSL/2) + s (s < RSL/2) -> register e = i RSL + s; q = R/2 is the
// Nyquist bin N/2 = output s = RSL/2 of butterfly i = 0 (that bin only when vt == 0).
template <class C>
__device__ __forceinline__ constexpr int fwd_reg_of_bin(int q) {
  return q < C::R / 2 ? (q / (C::RSL / 2)) * C::RSL + (q % (C::RSL / 2)) : C::RSL / 2;
}

// Per-CTA shared-memory carve-up and per-thread group geometry.
template <class C, bool TSPLIT = false>
struct Ctx {
  int grp, gt, line, vt;
  uint32_t tbase = 0, taddr = 0;  // TMEM allocation base / this thread's state slice (C::TPRIV)
  uint32_t ttw = 0;               // this thread's twiddles (C::TWT)
  uint32_t tv = 0;                // C::VTM: this warp's v_l block (A or B) in its lane quadrant
  uint64_t *vbar = nullptr;       // C::VTM: v_l copied into TMEM (tcgen05.commit), one phase per term
  unsigned *vcnt = nullptr;       // C::VTM: warps done reading v_l (monotonic: NWARP per term)
  void *buf;     // group exchange buffer
  double *alow;  // group: k0 x LG low-degree coefficients (forward) / reduced a_V (inverse)
  double *priv;  // group: thread-private slots [slot][gt] (C::PRIV)
  double *vred;  // group: K0MAX x GW x LG per-warp partials of (W V)^T y (inverse)
  Ring<C> ring;
  long long nbatch, bt0, btstep;
  int slice = 0, S = 1, l0 = 0, l1 = 0;
  // Group term split (TermSplit::gsl == 2, chosen by the launch): a batch is GU = GPC/2 groups' lines; group grp works
  // on line group lgrp = grp % GU as slice group sg = grp / GU, the CTA's terms dealt round-robin to the gsl (<= 2)
  // slice groups, each keeping its own partials (summed by cluster_reduce); groups sg >= gsl, and groups whose lines
  // are all past the end (dead), only take part in the factor ring.
  int gsl = 1, lgrp = 0, sg = 0, GU = C::GPC;
  bool dead = false;
  // first line of this group in batch bt
  __device__ __forceinline__ long long batch_line(long long bt) const {
    return (bt * (TSPLIT ? GU : C::GPC) + lgrp) * C::LG + line;
  }
  const double2 *gv, *gu;
  __device__ __forceinline__ Ctx(char *smem, const AxisDev &ax, long long nlines, const TermSplit &ts) {
    grp = threadIdx.x / C::GT;
    gt = threadIdx.x % C::GT;
    if constexpr (C::VTM) {  // lane = 8 line + vt % 8 (the TMEM v blocks repeat 8 rows down the quadrant)
      line = (gt & 31) >> 3;
      vt = ((gt >> 5) << 3) | (gt & 7);
    } else {
      line = gt % C::LG;
      vt = gt / C::LG;
    }
    gv = ax.v;
    gu = ax.ub;
    ring.base = smem;
    ring.full = reinterpret_cast<uint64_t *>(smem + C::NSTAGE * C::STAGE_BYTES);
    ring.empty = ring.full + C::NSTAGE;
    ring.cnt = reinterpret_cast<unsigned *>(ring.empty + C::NSTAGE);
    if constexpr (C::VTM) {
      vbar = reinterpret_cast<uint64_t *>(ring.cnt + C::NSTAGE + (C::NSTAGE & 1));  // (8-byte aligned)
      vcnt = reinterpret_cast<unsigned *>(vbar + 1);
    }
    ring.gv = ax.v;
    ring.gu = ax.ub;
    ring.r = ax.r;
    ring.gph = ax.phivc;
    ring.k0 = ax.k0;
    char *gb = smem + C::HDR_BYTES + grp * C::GROUP_BYTES;
    buf = gb;
    alow = reinterpret_cast<double *>(gb + C::SLOTS * C::XB);
    priv = alow + K0MAX * C::LG;
    vred = priv + C::PSLOTS * C::GT;
    if (TSPLIT && ts.gsl == 2) GU = C::GPC / 2;
    nbatch = (nlines + (long long)GU * C::LG - 1) / ((long long)GU * C::LG);
    S = TSPLIT ? ts.S : 1;
    long long mine;
    if (TSPLIT) {  // one (batch, term slice) per CTA
      slice = blockIdx.x % S;
      bt0 = blockIdx.x / S;
      btstep = nbatch;
      l0 = (int)((long long)slice * ax.r / S);
      l1 = (int)((long long)(slice + 1) * ax.r / S);
      mine = bt0 < nbatch ? 1 : 0;
    } else {
      bt0 = blockIdx.x;
      btstep = gridDim.x;
      l0 = 0;
      l1 = ax.r;
      mine = blockIdx.x < nbatch ? (nbatch - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    }
    lgrp = grp;
    if (TSPLIT && ts.gsl == 2) {
      lgrp = grp % GU;
      sg = grp / GU;
      gsl = min(2, max(l1 - l0, 1));
    }
    // (term-split launches only: one batch per CTA; the persistent launches keep the plain loop)
    dead = TSPLIT && (sg >= gsl || (bt0 * GU + lgrp) * C::LG >= nlines);
    ring.l0 = l0;
    ring.rs = l1 - l0 > 0 ? l1 - l0 : 1;
    ring.total = mine * (l1 - l0) * (C::SUB ? C::NSUB : 1);
  }
  // CTA table: TPL x NB packed row ranges (j0 << 4) | count of the bins binof(vt, q) (staged configs;
  // the others read bstart from global: their register budget has no room for the extra live state)
  __device__ static __forceinline__ int *binfo() {
    extern __shared__ __align__(128) char smem_raw[];
    return reinterpret_cast<int *>(smem_raw + C::BINFO_OFF);
  }
  __device__ __forceinline__ void rows_of(const int *__restrict__ bstart, int q, int m, int &j0, int &cnt) const {
    if constexpr (C::STAGED) {
      const int bi = binfo()[vt * C::NBT + q];
      j0 = bi >> 4;
      cnt = bi & 15;
    } else {
      j0 = __ldg(&bstart[m]);
      cnt = __ldg(&bstart[m + 1]) - j0;
    }
  }
  // Ring set-up: barriers initialised and the first NSTAGE terms in flight before anyone waits; the
  // row-range table of the bins binof(vt, q) filled.
  template <class BinOf>
  __device__ __forceinline__ void start(const int *__restrict__ bstart, const double2 *__restrict__ tw, BinOf binof) {
    if constexpr (C::TWS && !C::TWT) {
      extern __shared__ __align__(128) char smem_raw[];
      double2 *t = reinterpret_cast<double2 *>(smem_raw + C::TW_OFF);
      for (int i = threadIdx.x; i < TwTotal<C::N, C::R>::value; i += C::NT) t[i] = __ldg(&tw[i]);
    }
    if constexpr (C::STAGED || C::URING || C::SUB) {
      if (threadIdx.x == 0) {
        for (int s = 0; s < C::NSTAGE; ++s) {
          mbar_init(&ring.full[s], 1);
          ring.cnt[s] = 0;
        }
        if constexpr (C::VTM) {
          mbar_init(vbar, 1);
          *vcnt = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (long long q = 0; q < C::NSTAGE && q < ring.total; ++q) ring.issue(q);
      }
    }
    if constexpr (C::STAGED) for (int i = threadIdx.x; i < C::TPL * C::NBT; i += C::NT) {
      const int m = binof(i / C::NBT, i % C::NBT);
      if (!JT_CHK(m >= 0 && m < C::NBINS)) continue;
      const int j0 = __ldg(&bstart[m]);
      binfo()[i] = (j0 << 4) | (__ldg(&bstart[m + 1]) - j0);
    }
    __shared__ uint32_t tslot;
    if constexpr (C::TPRIV) {
      if (threadIdx.x < 32) tmem_alloc(&tslot, C::TALLOC);
      tmem_fence_before_sync();
    }
    __syncthreads();
    if constexpr (C::TPRIV) {
      tmem_fence_after_sync();
      tbase = tslot;
      const int w = threadIdx.x / 32;
      taddr = tbase + ((uint32_t)(32 * (w % 4)) << 16) + (uint32_t)((w / 4) * C::TSTRIDE);
      ttw = C::TW_QSHARE ? tbase + ((uint32_t)(32 * (w % 4)) << 16) + (uint32_t)C::TW_BASE : taddr + C::TW_BASE;
      if constexpr (C::VTM)  // quadrants 0, 2 hold the group's first warps (vt 0..7: block A), 1, 3 the second (B)
        tv = tbase + ((uint32_t)(32 * (w % 4)) << 16) + (uint32_t)(((w & 1) == 0) ? C::V_COLA : C::V_COLB);
    }
    if constexpr (C::TWT) {  // the thread's twiddles, once for the whole kernel
      // (TW_QSHARE: the quadrant's first warp writes the copy; the others read it after the barrier below)
      if (!C::TW_QSHARE || threadIdx.x < 128) {
        constexpr int NV = (2 * C::TWPT + 7) / 8 * 8;
        double t[NV];
#pragma unroll
        for (int i = 2 * C::TWPT; i < NV; ++i) t[i] = 0.0;
        tw_fill<C, Pass<C::N, C::R, 1>::RS>(t, vt, tw);
#pragma unroll
        for (int c = 0; c < NV / 8; ++c)
          if (JT_CHK((int)(ttw & 0xffff) + 16 * c + 16 <= C::TALLOC)) tmem_st_d8(ttw + 16 * c, &t[8 * c]);
        tmem_wait_st();
      }
      if constexpr (C::TW_QSHARE) {
        tmem_fence_before_sync();
        __syncthreads();
        tmem_fence_after_sync();
      }
    }
    if constexpr (C::VTM)
      if (threadIdx.x == 0 && ring.total > 0) v_issue(0);  // the first term's v_l (its TMA stage issued above)
  }
  // C::VTM: copy term sq's v_l from its ring stage into TMEM blocks A (v[16r .. 16r + 7]) and B (v[16r + 8 ..]),
  // r = 0..31, each 8-row core matrix repeated down the 32 lanes of every quadrant (stride-dimension offset 0); one
  // thread, after the stage has landed and every warp has read the previous term's v_l.
  __device__ __forceinline__ void v_issue(long long sq) const {
    if constexpr (C::VTM) {
      mbar_wait(&ring.full[sq % C::NSTAGE], (uint32_t)((sq / C::NSTAGE) & 1));
      tmem_fence_after_sync();
      const uint32_t st = smem_u32(ring.v(sq));
#pragma unroll 8
      for (int r = 0; r < C::R; ++r) {
        const uint64_t da = tmem_cp_desc(st + 256 * r), db = tmem_cp_desc(st + 256 * r + 128);
        asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(tbase + C::V_COLA + 4 * r), "l"(da)
                     : "memory");
        asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(tbase + C::V_COLB + 4 * r), "l"(db)
                     : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(vbar))
                   : "memory");
    }
  }
  // C::VTM: wait until term seq's v_l is in TMEM
  __device__ __forceinline__ void v_wait(long long seq) const {
    if constexpr (C::VTM) {
      jitter();
      mbar_wait(vbar, (uint32_t)(seq & 1));
      __syncwarp();
      tmem_fence_after_sync();
    }
  }
  // C::VTM: this warp is done reading term seq's v_l; the last of the CTA's warps copies term seq + 1's
  __device__ __forceinline__ void v_free(long long seq) const {
    if constexpr (C::VTM) {
      tmem_fence_before_sync();
      jitter();
      __syncwarp();
      if ((threadIdx.x & 31) == 0) {
        unsigned old;
        asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(smem_u32(vcnt)) : "memory");
        if (old + 1 == (unsigned)(C::NWARP * (seq + 1)) && seq + 1 < ring.total) v_issue(seq + 1);
      }
      __syncwarp();
    }
  }
  // end of the kernel: every warp's TMEM traffic done, then warp 0 frees the allocation
  __device__ __forceinline__ void finish() {
    if constexpr (C::TPRIV) {
      tmem_fence_before_sync();
      __syncthreads();
      if (threadIdx.x < 32) tmem_dealloc(tbase, C::TALLOC);
    }
  }
  // Degrees [kv0, kv1) of the dense block's batch-start part [kin, k0) handled by this CTA: all of them, or (term
  // split) this slice's share -- the partials of every slice are summed anyway, so the block need not wait on one CTA
  // (slice 0 alone: 10 us of the 20 us 1D n = 1024 forward, tools/phases.py r02zb)
  // (group term split: the slice's degrees divided again among its gsl groups)
  __device__ __forceinline__ int kv0(int kin, int k0) const {
    if (!TSPLIT) return kin;
    const int a = kin + (int)((long long)(k0 - kin) * slice / S), b = kin + (int)((long long)(k0 - kin) * (slice + 1) / S);
    return gsl > 1 && sg < gsl ? a + (b - a) * sg / gsl : a;
  }
  __device__ __forceinline__ int kv1(int kin, int k0) const {
    if (TSPLIT && dead) return kv0(kin, k0);
    if (!TSPLIT) return k0;
    const int a = kin + (int)((long long)(k0 - kin) * slice / S), b = kin + (int)((long long)(k0 - kin) * (slice + 1) / S);
    return gsl > 1 ? a + (b - a) * (sg + 1) / gsl : b;
  }
  // does this group process rank term l (of this CTA's l0 .. l1 - 1)?
  __device__ __forceinline__ bool mine(int l) const {
    return !TSPLIT || (!dead && (gsl == 1 || (l - l0) % gsl == sg));
  }
  __device__ __forceinline__ const double2 *vfac(long long seq, int l) const {
    if constexpr (C::STAGED) return ring.v(seq);
    else return gv + (long long)l * C::N;
  }
  __device__ __forceinline__ const double2 *ufac(long long seq, int l) const {
    if constexpr (C::STAGED || C::URING) return ring.u(seq);
    else return gu + (long long)l * C::UROWS * C::NBINS;
  }
  __device__ __forceinline__ void acquire(long long seq) const {
    if constexpr (C::STAGED) ring.wait_full(seq);
  }
  __device__ __forceinline__ void acquire_u(long long seq) const {  // URING: u~_l just before the epilogue
    if constexpr (C::URING) ring.wait_full(seq);
  }
  __device__ __forceinline__ void release(long long seq) const {
    if constexpr ((C::STAGED || C::URING) && C::LATE) ring.release_warp(seq);
    else if constexpr (C::STAGED || C::URING) ring.release(seq, gt);
  }
};

// S doubles of per-thread state: registers, or (C::PRIV) private slots in tensor memory (C::TPRIV: the
// thread's TMEM lane, 16 doubles per tcgen05.ld pair) or in SMEM.  Written once per batch (store), read once
// per rank term in chunks of CH = 16 (chunk: includes the wait for the TMEM load).
template <class C, int S>
struct State {
  static constexpr int CH = 16, NCH = (S + CH - 1) / CH;
  double reg[C::PRIV ? 1 : S];
  double *sm;
  int gt;
  uint32_t taddr;
  __device__ __forceinline__ State(double *p, int t, uint32_t ta) : sm(p), gt(t), taddr(ta) {}
  __device__ __forceinline__ void store(const double (&v)[S]) {
    if constexpr (!C::PRIV) {
#pragma unroll
      for (int i = 0; i < S; ++i) reg[i] = v[i];
    } else if constexpr (C::TPRIV) {
#pragma unroll
      for (int c = 0; c < 2 * NCH; ++c) {  // 8 doubles (16 columns) per store, zero padded
        if (!JT_CHK((int)(taddr & 0xffff) + 16 * c + 16 <= C::TALLOC)) continue;
        double t[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) t[i] = (c * 8 + i < S) ? v[c * 8 + i] : 0.0;
        tmem_st_d8(taddr + 16 * c, t);
      }
      tmem_wait_st();
    } else {
#pragma unroll
      for (int i = 0; i < S; ++i) sm[i * C::GT + gt] = v[i];
    }
  }
  // TMEM state only: chunk c's loads issued, the caller waits (tmem_wait_ld) before reading o
  __device__ __forceinline__ void chunk_issue(int c, double (&o)[CH]) const {
    static_assert(C::TPRIV, "chunk_issue reads the TMEM state");
    (void)JT_CHK((int)(taddr & 0xffff) + 32 * c + 32 <= C::TALLOC);
    tmem_ld_d8(taddr + 32 * c, &o[0]);
    tmem_ld_d8(taddr + 32 * c + 16, &o[8]);
  }
  __device__ __forceinline__ void chunk(int c, double (&o)[CH]) const {
    if constexpr (!C::PRIV) {
#pragma unroll
      for (int i = 0; i < CH; ++i) o[i] = (c * CH + i < S) ? reg[c * CH + i] : 0.0;
    } else if constexpr (C::TPRIV) {
      (void)JT_CHK((int)(taddr & 0xffff) + 32 * c + 32 <= C::TALLOC);
      tmem_ld_d8(taddr + 32 * c, &o[0]);
      tmem_ld_d8(taddr + 32 * c + 16, &o[8]);
      tmem_wait_ld();
    } else {
#pragma unroll
      for (int i = 0; i < CH; ++i) o[i] = (c * CH + i < S) ? sm[(c * CH + i) * C::GT + gt] : 0.0;
    }
  }
};

template <int MAXR>
__device__ __forceinline__ void load_rows(const double *__restrict__ p, int stride, double (&o)[MAXR]) {
#pragma unroll
  for (int c = 0; c < MAXR; ++c) o[c] = __ldg(p + c * stride);
}

// Addressing of one line's elements.  Lines are (outer, inner) pairs, inner fastest; element j of line
// (o, i) of an axis of length n lives at o n inner + j inner + i (plain C-order), or, in the CHUNK-MAJOR
// layout of the slab all-to-all (cs = n / G chunk length),
//     (j / cs) (outer cs inner) + o cs inner + (j % cs) inner + i,
// which for cs == n is the plain layout.  The layout flag is uniform per launch.
constexpr int MAX_SPLIT = 32;  // chunk-major blocks per axis (in_split / out_split, the ranks of a slab exchange)
struct Layout {
  long long outer, inner;
  int in_cs, out_cs;  // chunk length of the input / output along the axis (== n: plain C-order)
  long long ostride;  // outer extent of the chunk-major blocks (== outer, or the whole slab when a launch
                      // covers only part of its rows: the pipelined all-to-all of the distributed forward)
  long long in_lim, out_lim;  // elements readable / writable from the in / out pointers (JT_CHECKS builds)
  // out_peer != nullptr (chunk-major output only): block g of the output is NOT at g ostride cs inner from `out`
  // but in ANOTHER allocation -- rank g's receive buffer mapped over NVLink (CUDA IPC) -- at element offset
  // out_peer[g] + out_row from `out` (a plan-owned device array), so the pass stores each block straight into the
  // peer that owns it (the fused slab exchange)
  const long long *out_peer;
  long long out_row;
};


// SPLIT is a template flag (a separate kernel instantiation) so that the plain layout costs no registers.
template <bool SPLIT>
struct LineAddr {
  long long b0, cstride, inner;
  int cs;
  const long long *peer;  // Layout::out_peer (output side of a fused-exchange pass), else nullptr
  __device__ __forceinline__ LineAddr(long long L, long long outer, long long inner_, int n, int cs_,
                                      const long long *peer_ = nullptr, long long row = 0) {
    const long long o = L / inner_, i = L - o * inner_;
    inner = inner_;
    cs = SPLIT ? cs_ : n;
    b0 = o * (long long)cs * inner_ + i + (SPLIT && peer_ ? row : 0);
    cstride = SPLIT ? outer * (long long)cs * inner_ : 0;  // outer = Layout::ostride (see the kernels)
    peer = SPLIT ? peer_ : nullptr;
  }
  __device__ __forceinline__ long long at(int j) const {
    if constexpr (SPLIT)
      return b0 + (peer ? __ldg(&peer[j / cs]) : (long long)(j / cs) * cstride) + (long long)(j % cs) * inner;
    else return b0 + (long long)j * inner;
  }
};

// L2 prefetch of the input line the group processes next (the batch-start loads otherwise wait on HBM while the
// whole CTA starts its batch together).  One request per 128-byte segment where the layout makes that cheap to
// pick: the thread with vt % 16 == 0 for contiguous lines, the first of 16 consecutive lines for strided ones.
template <class C, bool SPLIT>
__device__ __forceinline__ void prefetch_line(const double *in, const Layout &lay, long long L, long long nlines, int vt,
                                              int n) {
  {
    if (L >= nlines) return;
    const bool mine = lay.inner == 1 ? (vt % 16 == 0) : (lay.inner % 16 == 0 ? (L % 16 == 0) : true);
    if (!mine) return;
    const LineAddr<SPLIT> ia(L, lay.ostride, lay.inner, n, lay.in_cs);
#pragma unroll
    for (int r = 0; r < C::R; ++r) {
      const int k = vt + r * C::TPL;
      if (k < n) asm volatile("prefetch.global.L2 [%0];" ::"l"(in + ia.at(k)));
    }
  }
}
template <class C, bool SPLIT>
__device__ __forceinline__ void prefetch_next_line(const double *in, const Layout &lay, long long L, long long nlines,
                                                   int vt, int n) {
  if constexpr (JT_PREFETCH && !C::INV && C::N <= JT_PREFETCH_NMAX && C::N >= JT_PREFETCH_NMIN)
    prefetch_line<C, SPLIT>(in, lay, L, nlines, vt, n);
}

// Term split in clusters (TermSplit::cluster): this CTA's partial lines [line in batch][j] in its group areas.
template <class C>
__device__ __forceinline__ double *cluster_part() {
  extern __shared__ __align__(128) char smem_raw[];
  return reinterpret_cast<double *>(smem_raw + C::HDR_BYTES);
}

// Sum of the S CTAs' partial lines of this cluster's batch through distributed shared memory, in slice order (the
// order of ts_reduce: bit-identical results), written in the plain (outer, n, inner) layout.  CTA rank s of the
// cluster sums elements [s E / S, (s + 1) E / S) of the batch's E = lines x n.  The first cluster barrier publishes
// every CTA's partials; the second keeps each CTA's shared memory alive until its peers have read it.
template <class C>
__device__ __forceinline__ void cluster_reduce(double *out, const TermSplit &ts, const Layout &lay, long long nlines,
                                               int n, int r, Phases &phs) {
  jitter();
  __syncwarp();  // (the cluster barrier is .aligned: the warp reconverges after the jitter)
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  phs.mark(8);
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const long long bt = blockIdx.x / ts.S;
  const int GU = ts.gsl == 2 ? C::GPC / 2 : C::GPC;  // line groups per batch
  const long long L0 = bt * GU * C::LG;
  const long long lines = min((long long)GU * C::LG, nlines - L0);
  const long long E = lines * n;
  const uint32_t base = smem_u32(cluster_part<C>());
  const long long e1 = (rank + 1) * E / ts.S;
  // (group term split, Ctx::gsl: CTA t keeps gsl_t partials of the batch's lines, slice group g's at g GU LG lines)
  const bool gs = ts.gsl == 2;
  const uint32_t gstride = (uint32_t)(GU * C::LG * n * 8);
  unsigned two = 0;  // bit t: CTA t holds two partials (Ctx::gsl == 2: at least two terms)
  if (gs)
    for (int t = 0; t < ts.S; ++t)
      if ((t + 1) * r / ts.S - t * r / ts.S >= 2) two |= 1u << t;
  // two elements per thread and iteration, all 2 S remote loads in flight before the first add (one DSMEM round trip
  // per pair instead of S per element: 256^2 forward reduction 4 -> <1 us), each summed in slice order
  constexpr int SM_ = JT_TS_CLUSTER_MAX;
  // element e = lb n + j of the batch: (lb, j) advanced incrementally (no 64-bit division per element), the output
  // offset recomputed only when the line changes
  const int e0 = (int)(rank * E / ts.S) + (int)threadIdx.x;
  int lb = e0 / n, j = e0 - lb * n;
  long long obase = -1;
  int olb = -1;
  for (int e = e0; e < (int)e1; e += 2 * C::NT) {
    double v[2][SM_][2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int t = 0; t < SM_; ++t) {
        v[h][t][0] = v[h][t][1] = 0.0;
        if (t < ts.S && e + h * C::NT < (int)e1) {
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            if (g == 0 || ((two >> t) & 1u)) {
              uint32_t ra;
              asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                           : "=r"(ra)
                           : "r"(base + g * gstride + (uint32_t)((e + h * C::NT) * 8)), "r"(t));
              asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v[h][t][g]) : "r"(ra) : "memory");
            }
          }
        }
      }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (e + h * C::NT >= (int)e1) break;
      double sum = 0.0;
#pragma unroll
      for (int t = 0; t < SM_; ++t)
        if (t < ts.S) {
          sum += v[h][t][0];
          if ((two >> t) & 1u) sum += v[h][t][1];
        }
      if (lb != olb) {
        const long long L = L0 + lb, o = L / lay.inner, i = L - o * lay.inner;
        obase = o * n * lay.inner + i;
        olb = lb;
      }
      const long long idx = obase + (long long)j * lay.inner;
      if (JT_CHK(idx >= 0 && idx < lay.out_lim)) out[idx] = sum;
      j += C::NT;
      while (j >= n) {
        j -= n;
        ++lb;
      }
    }
  }
  phs.mark(9);
  // (only keeps every CTA's shared memory alive until its peers' loads returned -- they have: their values were summed
  // -- so a relaxed arrive: the release form's GPU-scope fence waited ~1-2 us for the output stores to drain)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
  phs.mark(10);
}

// Push form of the cluster reduction (JT_TS_PUSH): instead of every CTA pulling its element range from the S peers
// with 8-byte remote loads (measured ~3.5 us for 8-32 KB per CTA: many small requests over the SM-to-SM network),
// every CTA sends each owner t its partials of t's range with ONE bulk copy (cp.async.bulk shared::cta ->
// shared::cluster, completion on t's mbarrier), into a receive area in t's factor-ring region (free after the term
// loop); the owner sums its S (or S + the CTAs' second-group) slots locally, in slice order -- the order of the pull
// form and of ts_reduce, so results are bit-identical.  Ranges start at even elements (16-byte aligned copies).
// Returns false (nothing done) where the receive area does not fit: the caller then uses cluster_reduce.
template <class C>
__device__ __forceinline__ bool cluster_reduce_push(double *out, const TermSplit &ts, const Layout &lay,
                                                    long long nlines, int n, int r, Phases &phs) {
  extern __shared__ __align__(128) char smem_raw[];
  const int S = ts.S;
  const long long bt = blockIdx.x / S;
  const int GU = ts.gsl == 2 ? C::GPC / 2 : C::GPC;  // line groups per batch
  const long long L0 = bt * GU * C::LG;
  const int lines = (int)min((long long)GU * C::LG, nlines - L0);
  const int E = lines * n;
  const bool gs = ts.gsl == 2;
  unsigned two = 0;
  if (gs)
    for (int t = 0; t < S; ++t)
      if ((t + 1) * r / S - t * r / S >= 2) two |= 1u << t;
  const int slots = gs ? 2 * S : S;
  const int RS = ((E + S - 1) / S + 3) & ~1;  // receive slot stride (doubles, even) >= every range + 1
  const int recv_bytes = slots * RS * 8;
  // (uniform over the cluster: every CTA takes the same branch)
  if (recv_bytes + 16 > C::HDR_BYTES || (gs && (GU * C::LG * n) % 2 != 0)) return false;
  double *recv = reinterpret_cast<double *>(smem_raw);
  uint64_t *mbar = reinterpret_cast<uint64_t *>(smem_raw + ((recv_bytes + 15) & ~15));
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  auto ra = [&](int t) { return t <= 0 ? 0 : (t >= S ? E : ((int)((long long)t * E / S) & ~1)); };
  const int a = ra((int)rank), b = ra((int)rank + 1);
  const uint32_t my_bytes = (uint32_t)(((b - a) * 8 + 15) & ~15);
  if (threadIdx.x == 0) {
    // (the ring's stage barriers live in this region: invalidated before it is reused as data)
    if constexpr (C::STAGED || C::URING || C::SUB)
      for (int st = 0; st < C::NSTAGE; ++st)
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(reinterpret_cast<uint64_t *>(
                         smem_raw + C::NSTAGE * C::STAGE_BYTES) + st))
                     : "memory");
    mbar_init(mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_arrive_expect_tx(mbar, my_bytes * (uint32_t)(S + __popc(two)));
  }
  jitter();
  __syncwarp();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  phs.mark(8);
  if ((int)threadIdx.x < S) {  // thread t: this CTA's partials of owner t's range, one bulk copy per group partial
    const int t = threadIdx.x, at = ra(t), btt = ra(t + 1);
    const uint32_t bytes = (uint32_t)(((btt - at) * 8 + 15) & ~15);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // (the partials were written by generic stores)
    const uint32_t src = smem_u32(cluster_part<C>() + at);
    uint32_t dst, mb;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst) : "r"(smem_u32(recv + rank * RS)), "r"(t));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(mb) : "r"(smem_u32(mbar)), "r"(t));
    if (bytes)
      asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                   "r"(src), "r"(bytes), "r"(mb)
                   : "memory");
    if ((two >> rank) & 1u) {  // the second group's partial (Ctx::gsl == 2) into slot S + rank
      const uint32_t src2 = smem_u32(cluster_part<C>() + GU * C::LG * n + at);
      uint32_t dst2;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst2) : "r"(smem_u32(recv + (S + rank) * RS)), "r"(t));
      if (bytes)
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         dst2),
                     "r"(src2), "r"(bytes), "r"(mb)
                     : "memory");
    }
  }
  mbar_wait(mbar, 0);
  __syncwarp();
  phs.mark(9);
  // owner: elements [a, b) of the batch, summed over the slots in slice order (second-group partial after each slice)
  int lb = (a + (int)threadIdx.x) / n, j = a + (int)threadIdx.x - lb * n, olb = -1;
  long long obase = 0;
  for (int k = threadIdx.x; k < b - a; k += C::NT) {
    double sum = 0.0;
    for (int t = 0; t < S; ++t) {
      sum += recv[t * RS + k];
      if ((two >> t) & 1u) sum += recv[(S + t) * RS + k];
    }
    if (lb != olb) {
      const long long L = L0 + lb, o = L / lay.inner, i = L - o * lay.inner;
      obase = o * n * lay.inner + i;
      olb = lb;
    }
    const long long idx = obase + (long long)j * lay.inner;
    if (JT_CHK(idx >= 0 && idx < lay.out_lim)) out[idx] = sum;
    j += C::NT;
    while (j >= n) {
      j -= n;
      ++lb;
    }
  }
  // every copy out of this CTA's shared memory has completed (its owner waited for it) before anyone exits
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
  phs.mark(10);
  return true;
}

// ------------------------------------------------------------------------------------------------
// Forward axis pass (K4).
// ------------------------------------------------------------------------------------------------
template <class C, bool SPLIT, bool TSPLIT = false>
__global__ void __launch_bounds__(C::NT, C::MINB) fwd_axis_kernel(AxisDev ax, const double *in, double *out,
                                                             long long nlines, Layout lay, TermSplit ts) {
  constexpr int R = C::R, TPL = C::TPL, LG = C::LG, NB = C::NB, MAXR = C::MAXR, NBINS = C::NBINS;
  extern __shared__ __align__(128) char smem_raw[];
  Phases phs;
  pdl_trigger();
  Ctx<C, TSPLIT> cx(smem_raw, ax, nlines, ts);
  cx.start(ax.bstart, ax.tw, [](int vt_, int q) { return q < R / 2 ? out_pos<C>(vt_, fwd_reg_of_bin<C>(q)) : C::N / 2; });
  // (term split, latency-bound: the batch's input lines requested into L2 while the previous kernel finishes -- only a
  // cache hint, so it may precede the dependency wait: L2 is the point of coherence)
  if constexpr (TSPLIT && JT_PDL_PREFETCH)
    prefetch_line<C, SPLIT>(in, lay, cx.batch_line(cx.bt0), nlines, cx.vt, ax.n);
  pdl_wait();  // (the prologue above touches only plan data: the arrays are the previous kernel's)
  phs.mark(1);
  const int n = ax.n, k0 = ax.k0;
  const int vt = cx.vt, line = cx.line;
  // degrees [0, kin) of W V are applied inside the term loop from the ring (KPT per term), the rest here
  const int kin = C::VST ? min(k0, ax.r * C::KPT) : 0;

  int m[NB];
#pragma unroll
  for (int q = 0; q < NB; ++q) m[q] = q < R / 2 ? out_pos<C>(vt, fwd_reg_of_bin<C>(q)) : C::N / 2;

  long long seq = 0;
  for (long long bt = cx.bt0; bt < cx.nbatch; bt += cx.btstep) {
    const long long L = cx.batch_line(bt);
    const bool live = L < nlines && (!TSPLIT || !cx.dead);
    const LineAddr<SPLIT> ia(live ? L : 0, lay.ostride, lay.inner, n, lay.in_cs);
    const LineAddr<SPLIT> oa(live ? L : 0, lay.ostride, lay.inner, n, lay.out_cs, lay.out_peer, lay.out_row);

    // coefficients at the first-pass input positions k = vt + r TPL; degrees < k0 also to alow
    // (all loads issued before any shared-memory store, so that their latencies overlap)
    State<C, R> a(cx.priv, cx.gt, cx.taddr);
    {
      double av[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int k = vt + r * TPL;
        av[r] = (live && k < n && JT_CHK(ia.at(k) >= 0 && ia.at(k) < lay.in_lim)) ? load_in<TSPLIT>(in, ts, ia.at(k)) : 0.0;
      }
      a.store(av);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int k = vt + r * TPL;
        if (r * TPL < K0MAX && k < K0MAX) cx.alow[k * LG + line] = k < k0 ? av[r] : 0.0;  // zero pad: W V pairs
        // (checks: the bins every thread reads are real FFT bins)
        if (r < NB) (void)JT_CHK(m[r] >= 0 && m[r] < NBINS);
      }
    }
    prefetch_next_line<C, SPLIT>(in, lay, ((bt + cx.btstep) * C::GPC + cx.grp) * LG + line, nlines, vt, n);

    // A4: y = W V a_V on the rows of the thread's bins
    double y[NB][MAXR];
#pragma unroll
    for (int q = 0; q < NB; ++q)
#pragma unroll
      for (int c = 0; c < MAXR; ++c) y[q][c] = 0.0;
    group_sync<C>();
    phs.mark(2);
#pragma unroll C::VUN
    for (int k = cx.kv0(kin, k0); k < cx.kv1(kin, k0); ++k) {
      const double ak = cx.alow[k * LG + line];
      const double *pk = ax.phivb + (long long)k * MAXR * NBINS;
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        double pv[MAXR];
        load_rows<MAXR>(pk + m[q], NBINS, pv);
#pragma unroll
        for (int c = 0; c < MAXR; ++c) y[q][c] = fma(pv[c], ak, y[q][c]);
      }
    }
    phs.mark(3);

    for (int l = cx.l0; l < cx.l1; ++l, ++seq) {
      cx.acquire(seq);
      if (!cx.mine(l)) {  // (another group's term, or a dead group: only the ring protocol)
        cx.v_wait(seq);
        cx.v_free(seq);
        cx.acquire_u(seq);
        if constexpr (!C::LATE) group_sync<C>();
        cx.release(seq);
        continue;
      }
      const double2 *vl = cx.vfac(seq, l);
      const double2 *ul = cx.ufac(seq, l);
      if constexpr (C::VST) {  // A4 for degrees l KPT .. l KPT + KPT - 1 (rows of W V staged with the term)
        static_assert(C::KPT % 2 == 0 && K0MAX % C::KPT == 0, "W V chunks are read as double2 pairs");
        constexpr int KP2 = C::KPT / 2;
        const double2 *ph = reinterpret_cast<const double2 *>(cx.ring.ph(seq));
        const int kb = l * C::KPT;
        // stage layout: KPT / 2 consecutive 2-degree chunks [hh][m][c][2] (one bin's rows 32 B apart in every chunk: the
        // broadcast LDS.128s of a warp's 8 bins stay 2 wavefronts; [m][c][4] measured 4); degrees >= k0 are zero-padded
        if (kb < k0) {
          double al[C::KPT];
#pragma unroll
          for (int kk = 0; kk < C::KPT; ++kk) al[kk] = cx.alow[(kb + kk) * LG + line];
#pragma unroll
          for (int q = 0; q < NB; ++q) {
            if (C::PAIR && q == R / 2) continue;  // (no Nyquist slot on the half-integer bin grid)
#pragma unroll
            for (int c = 0; c < MAXR; ++c)
#pragma unroll
              for (int hh = 0; hh < KP2; ++hh) {
                const double2 pp = ph[(hh * NBINS + m[q]) * MAXR + c];
                y[q][c] = fma(pp.x, al[2 * hh], fma(pp.y, al[2 * hh + 1], y[q][c]));
              }
          }
        }
      }
      double xr[R], xi[R];
      if constexpr (C::SUB) {
        // A1 from the ring: sub-stage j holds v_l[1024 j ..], i.e. positions vt + r TPL for r in [8j, 8j + 8)
        static_assert(R == 32 && TPL == 128 && State<C, R>::CH == 16, "SUB layout");
#pragma unroll
        for (int ch = 0; ch < State<C, R>::NCH; ++ch) {
          double ac[State<C, R>::CH];
          a.chunk(ch, ac);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const long long sq = seq * C::NSUB + 2 * ch + hh;
            cx.ring.wait_full(sq);
            const double2 *vs = cx.ring.slot(sq);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const double2 vv = vs[vt + i * TPL];
              xr[16 * ch + 8 * hh + i] = vv.x * ac[8 * hh + i];
              xi[16 * ch + 8 * hh + i] = vv.y * ac[8 * hh + i];
            }
            cx.ring.release_warp(sq);
          }
        }
      } else if constexpr (!C::STAGED && C::TPRIV && (JT_LOADS_FIRST & 1)) {
        // A1, v_l from L1/L2: a chunk's loads issued between its TMEM state load and the wait for it
#pragma unroll
        for (int ch = 0; ch < State<C, R>::NCH; ++ch) {
          double ac[State<C, R>::CH];
          a.chunk_issue(ch, ac);
#pragma unroll
          for (int i = 0; i < State<C, R>::CH; ++i) {
            const int r = ch * State<C, R>::CH + i;
            if (r < R) {
              const double2 vv = vl[vt + r * TPL];
              xr[r] = vv.x;
              xi[r] = vv.y;
            }
          }
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < State<C, R>::CH; ++i) {
            const int r = ch * State<C, R>::CH + i;
            if (r < R) {
              xr[r] *= ac[i];
              xi[r] *= ac[i];
            }
          }
        }
      } else if constexpr (C::VTM) {
        // A1 with v_l from TMEM: 8 positions per step (state chunk of 8 + 8 complex of this warp's v block)
        cx.v_wait(seq);
#pragma unroll
        for (int ch = 0; ch < R / 8; ++ch) {
          double ac[8], vr[16];
          tmem_ld_d8(cx.taddr + 16 * ch, ac);
          tmem_ld_d8(cx.tv + 32 * ch, &vr[0]);
          tmem_ld_d8(cx.tv + 32 * ch + 16, &vr[8]);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            xr[8 * ch + i] = vr[2 * i] * ac[i];
            xi[8 * ch + i] = vr[2 * i + 1] * ac[i];
          }
        }
        cx.v_free(seq);
      } else if constexpr (C::A1FOLD) {
        // A1 folded into the first butterfly layer of the radix-32 DFT: positions r < 16 scaled (state chunk 0), then
        // x_r +- x_{r+16} = fma(+-v_{r+16}, a_{r+16}, v_r a_r) with state chunk 1 (dft<32, true> skips that layer)
        double ac[State<C, R>::CH];
        a.chunk(0, ac);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const double2 vv = vl[vt + r * TPL];
          xr[r] = vv.x * ac[r];
          xi[r] = vv.y * ac[r];
        }
        a.chunk(1, ac);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const double2 vv = vl[vt + (r + 16) * TPL];
          const double tr = xr[r], ti = xi[r];
          xr[r] = fma(vv.x, ac[r], tr);
          xi[r] = fma(vv.y, ac[r], ti);
          xr[r + 16] = fma(-vv.x, ac[r], tr);
          xi[r + 16] = fma(-vv.y, ac[r], ti);
        }
      } else {
#pragma unroll
        for (int ch = 0; ch < State<C, R>::NCH; ++ch) {  // A1
          double ac[State<C, R>::CH];
          a.chunk(ch, ac);
#pragma unroll
          for (int i = 0; i < State<C, R>::CH; ++i) {
            const int r = ch * State<C, R>::CH + i;
            if (r < R) {
              const double2 vv = vl[vt + r * TPL];
              xr[r] = vv.x * ac[i];
              xi[r] = vv.y * ac[i];
            }
          }
        }
      }
      if constexpr (!C::STAGED && !C::URING && !C::SUB && JT_UPF) {
        // (factors from L2: the epilogue's u~_l rows requested into L1 now, the FFT hides the latency)
#pragma unroll
        for (int q = 0; q < NB; ++q)
#pragma unroll
          for (int c = 0; c < MAXR; ++c) asm volatile("prefetch.global.L1 [%0];" ::"l"(ul + c * NBINS + m[q]));
      }
      fft<C, C::A1FOLD>(xr, xi, cx.buf, vt, line, ax.tw + (l >> 30), cx.ttw);  // A2
      cx.acquire_u(seq);
      if constexpr (C::SUB) {
        // A3 from the ring: sub-stage 4 + i holds rows c of bins h 1024 + 256 i + [0, 256), i.e. the thread's bins
        // q in [4i, 4i + 4) (m = vt + (q / 2) TPL + (q % 2) N / 2); the Nyquist bin (q = R / 2) from L2
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const long long sq = seq * C::NSUB + 4 + i;
          cx.ring.wait_full(sq);
          const double2 *us = cx.ring.slot(sq);
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            const int q = 4 * i + qq;
            const int e = fwd_reg_of_bin<C>(q);
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const double2 uu = us[(2 * c + (q & 1)) * 256 + vt + ((q >> 1) - 2 * i) * TPL];
              y[q][c] = fma(uu.x, xr[e], y[q][c]);
              y[q][c] = fma(-uu.y, xi[e], y[q][c]);
            }
          }
          cx.ring.release_warp(sq);
        }
        const int e = fwd_reg_of_bin<C>(R / 2);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const double2 uu = __ldg(&ax.ub[((long long)l * MAXR + c) * NBINS + C::N / 2]);
          y[R / 2][c] = fma(uu.x, xr[e], y[R / 2][c]);
          y[R / 2][c] = fma(-uu.y, xi[e], y[R / 2][c]);
        }
      } else if constexpr (C::PAIR) {
        // A3, paired terms: row c of bin m takes Re(P Z[m]) + Re(conj(Q) Z[N - 1 - m]) (factor rows 2c, 2c + 1)
#pragma unroll
        for (int q = 0; q < R / 2; ++q) {
          const int e = fwd_reg_of_bin<C>(q), em = mirror_reg<C>(e);
#pragma unroll
          for (int c = 0; c < MAXR; ++c) {
            const double2 pp = ul[(2 * c) * NBINS + m[q]];
            const double2 qq = ul[(2 * c + 1) * NBINS + m[q]];
            y[q][c] = fma(pp.x, xr[e], y[q][c]);
            y[q][c] = fma(-pp.y, xi[e], y[q][c]);
            y[q][c] = fma(qq.x, xr[em], y[q][c]);
            y[q][c] = fma(-qq.y, xi[em], y[q][c]);
          }
        }
      } else
#pragma unroll
      for (int q = 0; q < NB; ++q) {  // A3
        const int e = fwd_reg_of_bin<C>(q);
#pragma unroll
        for (int c = 0; c < MAXR; ++c) {
          const double2 uu = ul[c * NBINS + m[q]];
          y[q][c] = fma(uu.x, xr[e], y[q][c]);
          y[q][c] = fma(-uu.y, xi[e], y[q][c]);
        }
      }
      if constexpr (!C::LATE) group_sync<C>();  // exchange buffer and this stage are free again
      cx.release(seq);
    }
    phs.mark(4);

    // (cluster term split: the partial lines go to this CTA's group areas once every group is done with them)
    double *cpart = nullptr;
    if constexpr (TSPLIT && C::CLUSTER_FIT) {
      if (ts.cluster) {
        __syncthreads();  // (one batch per CTA in a term-split launch: every thread is here)
        cpart = cluster_part<C>() + (long long)(cx.grp * LG + line) * n;
      }
    }
    if (live) {
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        if (q < R / 2 || vt == 0) {
          int j0, cnt;
          cx.rows_of(ax.bstart, q, m[q], j0, cnt);
#pragma unroll
          for (int c = 0; c < MAXR; ++c)
            if (c < cnt && JT_CHK(j0 + c >= 0 && j0 + c < n && L < nlines)) {
              if (TSPLIT && cpart) cpart[j0 + c] = y[q][c];
              else if (TSPLIT) ts.part[((long long)cx.slice * nlines + L) * n + j0 + c] = y[q][c];
              else if (JT_CHK(lay.out_peer || (oa.at(j0 + c) >= 0 && oa.at(j0 + c) < lay.out_lim)))
                out[oa.at(j0 + c)] = y[q][c];
            }
        }
      }
    }
    phs.mark(5);
    group_sync<C>();  // alow / PRIV reuse by the next batch
  }
  cx.finish();
  phs.mark(6);
  if constexpr (TSPLIT && C::CLUSTER_FIT)
    if (ts.cluster && !(JT_TS_PUSH && cluster_reduce_push<C>(out, ts, lay, nlines, n, ax.r, phs)))
      cluster_reduce<C>(out, ts, lay, nlines, n, ax.r, phs);
  phs.mark(7);
  phs.print(0, C::N, cx.l1 - cx.l0, lay.inner);
  if constexpr (SPLIT)
    if (lay.out_peer) __threadfence_system();  // (the fused exchange: this thread's peer stores performed system-wide)
}

// ------------------------------------------------------------------------------------------------
// Inverse axis pass (K5).
// ------------------------------------------------------------------------------------------------
template <class C, bool SPLIT, bool TSPLIT = false>
__global__ void __launch_bounds__(C::NT, C::MINB) inv_axis_kernel(AxisDev ax, const double *in, double *out,
                                                             long long nlines, Layout lay, TermSplit ts) {
  // PAIR (the transpose of the paired forward, Cfg::PAIR): a = (W V)^T y + Re(w (.) F_N b) with b[m] = sum of P_j y_j and
  // b[N - 1 - m] = sum of conj(Q)_j y_j over the rows j of bin m.  A thread's first-pass positions vt + r TPL are bins
  // for r < R/2 (slots q = r: its own rows, factor rows P) and mirrors for r >= R/2: position vt + r TPL =
  // N - 1 - m with m = (TPL - 1 - vt) + (R - 1 - r) TPL, so slot q = R/2 + (R - 1 - r) holds the rows of THAT bin
  // (factor rows conj(Q)); NB here = C::NBT = R slots, no Nyquist slot, no empty upper half.
  constexpr int R = C::R, TPL = C::TPL, LG = C::LG, NB = C::NBT, MAXR = C::MAXR, NBINS = C::NBINS;
  constexpr int NBO = C::PAIR ? R / 2 : NB;  // slots of the thread's OWN rows (the dense block sums each row once)
  extern __shared__ __align__(128) char smem_raw[];
  Phases phs;
  pdl_trigger();
  Ctx<C, TSPLIT> cx(smem_raw, ax, nlines, ts);
  cx.start(ax.bstart, ax.tw, [](int vt_, int q) {
    if constexpr (C::PAIR) return q < R / 2 ? vt_ + q * TPL : (TPL - 1 - vt_) + (q - R / 2) * TPL;
    else return q < R / 2 ? vt_ + q * TPL : C::N / 2;
  });
  // (term split, latency-bound: the batch's input lines requested into L2 while the previous kernel finishes -- only a
  // cache hint, so it may precede the dependency wait: L2 is the point of coherence)
  if constexpr (TSPLIT && JT_PDL_PREFETCH)
    prefetch_line<C, SPLIT>(in, lay, cx.batch_line(cx.bt0), nlines, cx.vt, ax.n);
  pdl_wait();  // (the prologue above touches only plan data: the arrays are the previous kernel's)
  phs.mark(1);
  const int n = ax.n, k0 = ax.k0;
  const int vt = cx.vt, line = cx.line;
  // degrees [0, kin) of (W V)^T y are formed inside the term loop from the ring (KPT per term), the rest
  // at batch start
  const int kin = C::VST ? min(k0, ax.r * C::KPT) : 0;

  // input bins: q < R/2 -> first-pass position vt + q TPL; q = R/2 -> position vt + N/2 (Nyquist, vt == 0)
  int m[NB];
#pragma unroll
  for (int q = 0; q < NB; ++q)
    m[q] = q < R / 2 ? vt + q * TPL : (C::PAIR ? (TPL - 1 - vt) + (q - R / 2) * TPL : C::N / 2);

  long long seq = 0;
  for (long long bt = cx.bt0; bt < cx.nbatch; bt += cx.btstep) {
    const long long L = cx.batch_line(bt);
    const bool live = L < nlines && (!TSPLIT || !cx.dead);
    const LineAddr<SPLIT> ia(live ? L : 0, lay.ostride, lay.inner, n, lay.in_cs);
    const LineAddr<SPLIT> oa(live ? L : 0, lay.ostride, lay.inner, n, lay.out_cs, lay.out_peer, lay.out_row);

    State<C, NB * MAXR> yb(cx.priv, cx.gt, cx.taddr);  // element q MAXR + c: row c of input bin q
    {
      // a_V = (W V)^T y: thread partial sums over its rows (held in registers here: nothing else is
      // live yet), reduced over the TPL threads of the line (shuffles within the warp, then SMEM across
      // the GW warps of a multi-warp group)
      double yr[NB * MAXR];
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        const bool own = C::PAIR || q < R / 2 || vt == 0;
        int j0, cnt;
        cx.rows_of(ax.bstart, q, m[q], j0, cnt);
#pragma unroll
        for (int c = 0; c < MAXR; ++c)
          yr[q * MAXR + c] = (live && own && c < cnt && JT_CHK(j0 + c < n && m[q] < NBINS) &&
                              JT_CHK(ia.at(j0 + c) >= 0 && ia.at(j0 + c) < lay.in_lim))
                                 ? load_in<TSPLIT>(in, ts, ia.at(j0 + c))
                                 : 0.0;
      }
      yb.store(yr);
      phs.mark(2);
      prefetch_next_line<C, SPLIT>(in, lay, ((bt + cx.btstep) * C::GPC + cx.grp) * LG + line, nlines, vt, n);
      double *red = static_cast<double *>(cx.buf);  // k0 x GW x LG partials (exchange buffer is free)
      if (TSPLIT) {  // degrees outside this slice's terms contribute 0 (their slices add them)
        for (int i = cx.gt; i < k0 * LG; i += C::GT) cx.alow[i] = 0.0;
        for (int i = cx.gt; i < kin * C::GW * LG; i += C::GT) cx.vred[i] = 0.0;
      }
#pragma unroll C::VUN
      for (int k = cx.kv0(kin, k0); k < cx.kv1(kin, k0); ++k) {
        const double *pk = ax.phivb + (long long)k * MAXR * NBINS;
        double p = 0.0;
#pragma unroll
        for (int q = 0; q < NBO; ++q) {
          double pv[MAXR];
          load_rows<MAXR>(pk + m[q], NBINS, pv);
#pragma unroll
          for (int c = 0; c < MAXR; ++c) p = fma(pv[c], yr[q * MAXR + c], p);
        }
#pragma unroll
        for (int off = LG; off < 32; off *= 2) p += __shfl_xor_sync(0xffffffffu, p, off);
        if constexpr (C::GW == 1) {
          if (vt == 0) cx.alow[k * LG + line] = p;
        } else {
          if ((threadIdx.x & 31) < LG) red[(k * C::GW + (cx.gt >> 5)) * LG + line] = p;
        }
      }
      if constexpr (C::GW > 1) {
        group_sync<C>();
        for (int i = cx.gt + cx.kv0(kin, k0) * LG; i < cx.kv1(kin, k0) * LG; i += C::GT) {
          const int k = i / LG, ln = i % LG;
          double s = 0.0;
#pragma unroll
          for (int w = 0; w < C::GW; ++w) s += red[(k * C::GW + w) * LG + ln];
          cx.alow[k * LG + ln] = s;
        }
      }
      group_sync<C>();
    }
    phs.mark(3);

    double acc[R];
#pragma unroll
    for (int e = 0; e < R; ++e) acc[e] = 0.0;

    for (int l = cx.l0; l < cx.l1; ++l, ++seq) {
      cx.acquire(seq);
      if (!cx.mine(l)) {  // (another group's term, or a dead group: only the ring protocol)
        if constexpr (!C::LATE) group_sync<C>();
        cx.release(seq);
        continue;
      }
      const double2 *vl = cx.vfac(seq, l);
      const double2 *ul = cx.ufac(seq, l);
      double xr[R], xi[R];
      double pv[C::VST ? C::KPT : 1];  // partial (W V)^T y for degrees l KPT + kk (VST)
#pragma unroll
      for (int kk = 0; kk < (C::VST ? C::KPT : 1); ++kk) pv[kk] = 0.0;
      const double2 *ph = reinterpret_cast<const double2 *>(C::VST ? cx.ring.ph(seq) : nullptr);
      const int kb = l * C::KPT;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        xr[r] = 0.0;
        xi[r] = 0.0;
      }
      // bin sums over the rows of the input bins q <= R/2 (positions > N/2 hold no rows), state read in chunks
      using YS = State<C, NB * MAXR>;
      if constexpr (C::SUB) {
        // bin sums from the ring: sub-stage i holds rows c of bins 512 i + [0, 512), i.e. the thread's input bins
        // q in [4i, 4i + 4) (m = vt + q TPL); state chunk ch holds the rows of bins 8 ch .. 8 ch + 7
        static_assert(R == 32 && TPL == 128 && YS::CH == 16 && YS::NCH == 3, "SUB layout");
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          double yc[YS::CH];
          yb.chunk(ch, yc);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const long long sq = seq * C::NSUB + 2 * ch + hh;
            cx.ring.wait_full(sq);
            const double2 *us = cx.ring.slot(sq);
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
              const int q = 8 * ch + 4 * hh + qq;
#pragma unroll
              for (int c = 0; c < 2; ++c) {
                const double2 uu = us[c * 512 + vt + qq * TPL];
                const double yv = yc[(4 * hh + qq) * 2 + c];
                xr[q] = fma(uu.x, yv, xr[q]);
                xi[q] = fma(uu.y, yv, xi[q]);
              }
            }
            cx.ring.release_warp(sq);
          }
        }
        double yc[YS::CH];
        yb.chunk(2, yc);  // the Nyquist bin's rows (nonzero only for vt == 0), u~_l from L2
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const double2 uu = __ldg(&ax.ub[((long long)l * MAXR + c) * NBINS + C::N / 2]);
          xr[R / 2] = fma(uu.x, yc[c], xr[R / 2]);
          xi[R / 2] = fma(uu.y, yc[c], xi[R / 2]);
        }
      } else if constexpr (!C::PAIR && !C::STAGED && !C::VST && MAXR == 2 && (JT_LOADS_FIRST & 2) && C::N >= JT_LF_INV_NMIN) {
        // u~_l from L1/L2: both rows' loads of every bin in flight before the state chunks
        double2 u1[NB];
#pragma unroll
        for (int r = 0; r < NB; ++r) {
          const double2 u0 = ul[m[r]];
          u1[r] = ul[NBINS + m[r]];
          xr[r] = u0.x;
          xi[r] = u0.y;
        }
#pragma unroll
        for (int ch = 0; ch < YS::NCH; ++ch) {
          double yc[YS::CH];
          yb.chunk(ch, yc);
#pragma unroll
          for (int i = 1; i < YS::CH; i += 2) {
            const int r = (ch * YS::CH + i) / 2;
            if (r < NB) {
              xr[r] = fma(u1[r].x, yc[i], xr[r] * yc[i - 1]);
              xi[r] = fma(u1[r].y, yc[i], xi[r] * yc[i - 1]);
            }
          }
        }
      } else
#pragma unroll
      for (int ch = 0; ch < YS::NCH; ++ch) {
        double yc[YS::CH];
        yb.chunk(ch, yc);
#pragma unroll
        for (int i = 0; i < YS::CH; ++i) {
          const int idx = ch * YS::CH + i;
          if (idx < NB * MAXR) {
            const int r = idx / MAXR, c = idx % MAXR;
            // (PAIR: slots >= R/2 are the mirror positions' bins: factor row conj(Q), input register R - 1 - (r - R/2))
            const bool mir = C::PAIR && r >= R / 2;
            const int reg = mir ? R - 1 - (r - R / 2) : r;
            const double2 uu = ul[(C::PAIR ? 2 * c + (mir ? 1 : 0) : c) * NBINS + m[r]];
            const double yv = yc[i];
            xr[reg] = fma(uu.x, yv, xr[reg]);
            xi[reg] = fma(uu.y, yv, xi[reg]);
            if constexpr (C::VST) {
              if (!mir && kb < k0) {
#pragma unroll
                for (int hh = 0; hh < C::KPT / 2; ++hh) {
                  const double2 pp = ph[(hh * NBINS + m[r]) * MAXR + c];
                  pv[2 * hh] = fma(pp.x, yv, pv[2 * hh]);
                  pv[2 * hh + 1] = fma(pp.y, yv, pv[2 * hh + 1]);
                }
              }
            }
          }
        }
      }
      if constexpr (C::VST && JT_PAIRRED && LG < 32 && 2 * LG < 32) {
        // reduce the two degrees' partials over the line's threads of the warp as a pair: the first shuffle level
        // trades halves (lanes with the LG bit keep degree kb + 1, the others kb), so each further level moves one
        // double instead of two (6 shuffles per term instead of 12); then per-warp slots as below
        static_assert(C::KPT == 2, "paired reduction");
        if (kb < k0) {
          const int lane = threadIdx.x & 31;
          const bool hi = (lane & LG) != 0;
          double p = (hi ? pv[1] : pv[0]) + __shfl_xor_sync(0xffffffffu, hi ? pv[0] : pv[1], LG);
#pragma unroll
          for (int off = 2 * LG; off < 32; off *= 2) p += __shfl_xor_sync(0xffffffffu, p, off);
          const int kk = hi ? 1 : 0;
          if (lane < 2 * LG && kb + kk < k0) {
            if constexpr (C::GW == 1) cx.alow[(kb + kk) * LG + line] = p;
            else cx.vred[((kb + kk) * C::GW + (cx.gt >> 5)) * LG + line] = p;
          }
        }
      } else if constexpr (C::VST) {  // reduce over the line's threads: shuffles in the warp, per-warp slots after
#pragma unroll
        for (int kk = 0; kk < C::KPT; ++kk) {
          if (kb + kk < k0) {
            double p = pv[kk];
#pragma unroll
            for (int off = LG; off < 32; off *= 2) p += __shfl_xor_sync(0xffffffffu, p, off);
            if constexpr (C::GW == 1) {
              if (vt == 0) cx.alow[(kb + kk) * LG + line] = p;
            } else {
              if ((threadIdx.x & 31) < LG) cx.vred[((kb + kk) * C::GW + (cx.gt >> 5)) * LG + line] = p;
            }
          }
        }
      }
      if constexpr (!C::STAGED && !C::SUB && JT_UPF) {
        // (factors from L2: the accumulation's v_l entries requested into L1 now, the FFT hides the latency)
#pragma unroll
        for (int e = 0; e < R; ++e) asm volatile("prefetch.global.L1 [%0];" ::"l"(vl + out_pos<C>(vt, e)));
      }
      fft<C, false, !C::PAIR>(xr, xi, cx.buf, vt, line, ax.tw + (l >> 30), cx.ttw);  // (unpaired: inputs above R/2 are empty bins)
      if constexpr (C::SUB) {
        // a[k] += Re(v_l[k] B[k]) from the ring: sub-stage 4 + j holds v_l[1024 h + 256 j + ...], i.e. the outputs
        // e with e / RSL in {2j, 2j + 1} (k = vt + (e / RSL) TPL + (e % RSL) N / RSL, RSL = 4)
        static_assert(C::RSL == 4, "SUB layout");
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const long long sq = seq * C::NSUB + 4 + j;
          cx.ring.wait_full(sq);
          const double2 *vs = cx.ring.slot(sq);
#pragma unroll
          for (int tt = 0; tt < 2; ++tt)
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const int e = 4 * (2 * j + tt) + h;
              const double2 vv = vs[h * 256 + vt + tt * TPL];
              acc[e] = fma(vv.x, xr[e], acc[e]);
              acc[e] = fma(-vv.y, xi[e], acc[e]);
            }
          cx.ring.release_warp(sq);
        }
      } else
#pragma unroll
      for (int e = 0; e < R; ++e) {  // a[k] += Re(v_l[k] B[k])
        const double2 vv = vl[out_pos<C>(vt, e)];
        acc[e] = fma(vv.x, xr[e], acc[e]);
        acc[e] = fma(-vv.y, xi[e], acc[e]);
      }
      if constexpr (!C::LATE) group_sync<C>();
      cx.release(seq);
    }
    phs.mark(4);
    if constexpr (C::VST && C::GW > 1) {  // combine the per-warp partials of degrees < kin
      if constexpr (C::LATE) group_sync<C>();  // (every warp's last partials written)
      for (int i = cx.gt; i < kin * LG; i += C::GT) {
        const int k = i / LG, ln = i % LG;
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < C::GW; ++w) s += cx.vred[(k * C::GW + w) * LG + ln];
        cx.alow[k * LG + ln] = s;
      }
      group_sync<C>();
    }

#pragma unroll
    for (int e = 0; e < R; ++e) {  // the dense block's degrees
      const int k = out_pos<C>(vt, e);
      if (k < k0) acc[e] += cx.alow[k * LG + line];
    }
    double *cpart = nullptr;
    if constexpr (TSPLIT && C::CLUSTER_FIT) {
      if (ts.cluster) {
        __syncthreads();  // (one batch per CTA in a term-split launch: every thread is here)
        cpart = cluster_part<C>() + (long long)(cx.grp * LG + line) * n;
      }
    }
    if (live) {
#pragma unroll
      for (int e = 0; e < R; ++e) {
        const int k = out_pos<C>(vt, e);
        const double val = acc[e];
        if (k < n) {
          if (TSPLIT && cpart) cpart[k] = val;
          else if (TSPLIT) ts.part[((long long)cx.slice * nlines + L) * n + k] = val;
          else if (JT_CHK(lay.out_peer || (oa.at(k) >= 0 && oa.at(k) < lay.out_lim))) out[oa.at(k)] = val;
        }
      }
    }
    phs.mark(5);
    group_sync<C>();
  }
  cx.finish();
  phs.mark(6);
  if constexpr (TSPLIT && C::CLUSTER_FIT)
    if (ts.cluster && !(JT_TS_PUSH && cluster_reduce_push<C>(out, ts, lay, nlines, n, ax.r, phs)))
      cluster_reduce<C>(out, ts, lay, nlines, n, ax.r, phs);
  phs.mark(7);
  phs.print(1, C::N, cx.l1 - cx.l0, lay.inner);
  if constexpr (SPLIT)
    if (lay.out_peer) __threadfence_system();  // (the fused exchange: this thread's peer stores performed system-wide)
}

}  // namespace jtk

namespace jtk {
// Sum of the S term-slice partials of a term-split launch (slice order: deterministic), written in the plain
// (outer, n, inner) layout.  Element (o, j, i), i fastest.
static __global__ void ts_reduce(const double *__restrict__ part, double *__restrict__ out, int S, long long nlines, int n,
                          long long inner) {
  const long long total = nlines * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const long long i = e % inner, oj = e / inner, j = oj % n, o = oj / n;
    const long long L = o * inner + i;
    double sum = 0.0;
    for (int s = 0; s < S; ++s) sum += part[((long long)s * nlines + L) * n + j];
    out[e] = sum;
  }
}
}  // namespace jtk
