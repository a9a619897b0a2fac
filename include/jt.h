/* jt.h — C ABI of the B200-native fast Jacobi polynomial transform library (libjt.so).
 *
 * Implements the hot path of arXiv 1901.07275 (Bremer, Pang, Yang), "Fast Algorithms for the
 * Multi-dimensional Jacobi Polynomial Transform":  the d-dimensional (d = 1, 2, 3) UNIFORM forward
 * and inverse discrete Jacobi transform, applied in the factored form
 *
 *     W J_n = [ W V_n , W Re( B_n (.) F_n ) ],   B_n ~ sum_{l<r} u_l v_l^T     (PAPER.md:576-615,
 *                                                   eq:B, eq:lastJ, eq:permuDFT, eq:approxA, eq:oneJ)
 *
 * axis by axis (eq:TJ PAPER.md:669-674, eq:TJ3 PAPER.md:718-722), each axis pass a hand-written
 * sm_100a CUDA kernel (fp64 FFTs, no cuFFT).  Plans are built on the host (Gauss-Jacobi rule,
 * non-oscillatory P~ + iQ~ = M e^{i psi}; Algorithm 1).
 *
 * Conventions (all calls):
 *   - Arrays are fp64, C-order (row-major), shape n[0] x ... x n[d-1]; axis i uses (a[i], b[i]).
 *   - Coefficient index along an axis = polynomial degree k (0-based, PAPER.md:485 tf:transexp).
 *   - Value index along an axis = quadrature node j, nodes t_j ascending in (0, pi).
 *   - jt_forward computes values = (Phi_0 (x) ... (x) Phi_{d-1}) coeffs with the orthogonal
 *     Phi_i = W_i J_i, Phi_i[j,k] = sqrt(w_j) P~_k(t_j)  (PAPER.md:460-470 tf:transout, 495-509,
 *     663, 706).  These are the paper's WEIGHTED values W f; unweighted f_j = values_j / sqrt(w_j).
 *   - jt_inverse computes coeffs = (Phi_0^T (x) ... (x) Phi_{d-1}^T) values (the uniform inverse,
 *     eq:oneJinv PAPER.md:621-630, eq:invTJ PAPER.md:683-687, eq:invTJ3 PAPER.md:731-735).
 *   - Every call returns a jt_status; no C++ exception crosses the ABI.  On a non-OK status,
 *     jt_last_error() returns a thread-local human-readable message.
 *   - Device-pointer calls enqueue work on `cuda_stream` (a cudaStream_t; NULL = legacy default
 *     stream) and return without synchronising.  Calls on one plan may use different streams: each call's
 *     first work waits (cudaStreamWaitEvent) for the previous call on the plan to finish with the plan-owned
 *     buffers (staging, all-to-all, term-split workspace), so calls on one plan never overlap on the device;
 *     use one plan per concurrent stream for overlap.  Calls on one plan must come from one host thread.
 *   - Sizes: 2 <= n[i] <= 4096.  The upper bound is the kernels' largest FFT length (one register + two
 *     shared-memory Stockham passes per line, tables sized for N <= 4096); 4096^3 (550 GB) is reached with
 *     distributed plans (jt_plan_dist_ex, JT_DIST_LOWMEM on 8 GPUs).
 *   - Aliasing (in the terms of SURVEY.md §8(b)): device calls take input and output pointers that either
 *     coincide exactly (in place, allowed for the single-GPU transforms and plain-layout axis passes) or do
 *     not overlap at all; any partial overlap is JT_ERR_ARG.  Distributed and chunk-major calls must be out
 *     of place.
 */
#ifndef JT_H
#define JT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct jt_plan_s *jt_plan_t; /* opaque plan handle */

typedef enum {
  JT_OK = 0,
  JT_ERR_ARG = 1,     /* bad argument: d not in {1,2,3}, n[i] < 2 or > 4096, eps not in [1e-15, 1e-2],
                         null pointer, aliasing in/out where not allowed, host-only plan on a device call */
  JT_ERR_DOMAIN = 2,  /* a or b outside (-1, 1): the paper's validated range, "not applicable" outside
                          */
  JT_ERR_NUMERIC = 3, /* Newton for the nodes did not converge, or the adaptive rank had to grow beyond its growth
                         cap min(n, n - k0) / 4 (reading R25) */
  JT_ERR_ALLOC = 4,   /* host or device allocation failed */
  JT_ERR_CUDA = 5,    /* a CUDA runtime error (launch, copy, or an asynchronous fault from an earlier call) */
  JT_ERR_NCCL = 6     /* the library-owned NCCL path (distributed plans): libnccl.so.2 missing, a failed call,
                         or an asynchronous communicator error (the communicator is then aborted) */
} jt_status;

/* Plan options.  jt_default_opts() fills the defaults shown. */
typedef struct {
  uint64_t seed;   /* PRNG seed of Algorithm 1's random row/column samples (default 0) */
  int k0;          /* number of low degrees kept in the dense block V, 0..32; default -1 = auto:
                      the paper's 27, or 32 where that lowers the rank (FFT length <= 512), or 20 / 24 where that
                      keeps the rank (FFT length 4096 / 2048; R24) */
  int rmax_init;   /* initial rank cap of Algorithm 1; 0 = max(ceil(2 log2 n), 32) */
  int q;           /* oversampling factor of Algorithm 1 (default 3; "q = O(1)") */
  int sweeps;      /* repetitions of Algorithm 1 steps 2-3 (default 2) */
  int device;      /* CUDA device ordinal for the plan's buffers; -1 = current device;
                      -2 = HOST-ONLY plan (no GPU touched: introspection only, device calls fail) */
} jt_opts;

/* Fill *o with the defaults above.  Returns JT_ERR_ARG if o is NULL. */
jt_status jt_default_opts(jt_opts *o);

/* Build a plan for a d-dimensional uniform transform (d in {1,2,3}).
 *   n[i]   length of axis i, 2 <= n[i] <= 4096;
 *   a[i], b[i]  Jacobi parameters of axis i, in (-1, 1);
 *   eps    relative tolerance of the low-rank factorisation of B (truncation sigma_{r+1} <= eps sigma_1,
 *          PAPER.md:238), in [1e-15, 1e-2];
 *   opts   NULL for defaults.
 * Host work per axis: O(n^2) long-double recurrences (nodes, P~ + iQ~), Algorithm 1 in O(n r^2 q);
 * then one host->device upload of the factors (unless opts->device == -2).
 * On success *out owns all host and device buffers of the plan; free it with jt_destroy. */
jt_status jt_plan(jt_plan_t *out, int d, const int64_t n[], const double a[], const double b[],
                  double eps, const jt_opts *opts);

/* Kinds of modified Jacobi functions (PAPER.md:111-122 eq:modifiedjac, eq:modifiedjac2). */
enum { JT_KIND_P = 0 /* P~ (first kind) */, JT_KIND_Q = 1 /* Q~ (second kind) */ };

/* Extended plan:
 *   points  NULL, or d host pointers; points[i] == NULL selects the UNIFORM transform on axis i (Gauss-Jacobi
 *           nodes, rows weighted by sqrt(w_j), as jt_plan), otherwise points[i] holds n[i] NONUNIFORM points
 *           t_j in (0, pi), non-decreasing, and axis i's matrix is J itself (W = I, "the nonuniform forward
 *           Jacobi transform does not require trigonometric Gauss-Jacobi quadrature nodes and weights",
 *           PAPER.md:491; the same low-rank (.) DFT factorisation applies).  Points
 *           clustered so that more than 4 fall into one FFT bin raise the FFT length (up to 4096), else
 *           JT_ERR_NUMERIC.  The points are copied; the caller keeps ownership.
 *   kind    JT_KIND_P: expansions in P~_k; JT_KIND_Q: in Q~_k ("the transform for Q~ is similar",
 *           PAPER.md:457, 646; Q~ normalised as in DESIGN.md reading R8).
 * Only uniform first-kind plans are orthogonal: jt_inverse / jt_inverse_host refuse the others (JT_ERR_ARG;
 * the nonuniform inverse is an open problem); jt_adjoint applies the transpose for any plan. */
jt_status jt_plan_ex(jt_plan_t *out, int d, const int64_t n[], const double a[], const double b[],
                     const double *const points[], int kind, double eps, const jt_opts *opts);

/* Transpose transform coeffs = (M_0^T (x) ... (x) M_{d-1}^T) values for any plan (M_i axis i's matrix); equal
 * to jt_inverse for uniform first-kind plans.  Device pointers, same rules as jt_forward. */
jt_status jt_adjoint(jt_plan_t p, const double *values, double *coeffs, void *cuda_stream);

/* Whether axis `axis` is uniform (1) or nonuniform (0), and its kind (JT_KIND_P / JT_KIND_Q). */
jt_status jt_plan_kind(jt_plan_t p, int axis, int *uniform, int *kind);

/* Forward transform, device pointers (fp64, C-order, prod(n) elements each, 16-byte aligned).
 * coeffs is read-only; values is written.  coeffs == values is allowed (in place); partial overlap
 * is JT_ERR_ARG.  Runs d fused axis passes. */
jt_status jt_forward(jt_plan_t p, const double *coeffs, double *values, void *cuda_stream);

/* Inverse (transpose) transform, device pointers; same layout/aliasing rules as jt_forward. */
jt_status jt_inverse(jt_plan_t p, const double *values, double *coeffs, void *cuda_stream);

/* End-to-end variants with HOST buffers (pageable or pinned; pinned overlaps): copies host->device,
 * transforms, copies device->host, then synchronises `cuda_stream`.  Uses plan-owned device staging
 * buffers and two plan-owned copy streams: the input arrives in row chunks of axis 0 while the passes of
 * axes d-1..1 run on the chunks already copied; the axis-0 pass runs in column blocks, each copied back
 * while the next one computes.  Results equal jt_forward / jt_inverse up to rounding (the device path may
 * split the rank terms of a few-line launch over several CTAs and sum them in another order). */
jt_status jt_forward_host(jt_plan_t p, const double *coeffs_host, double *values_host, void *cuda_stream);
jt_status jt_inverse_host(jt_plan_t p, const double *values_host, double *coeffs_host, void *cuda_stream);

/* Asynchronous variants: enqueue the same pipelined work and return; results are in host memory after
 * jt_host_wait(p).  Consecutive calls alternate between two plan-owned staging slots, so one call's input copy
 * (host->device engine) overlaps the previous call's output copy (device->host engine) and compute: a stream
 * of transforms runs at the rate of the slower PCIe direction.  The host buffers must stay valid and unmodified
 * until jt_host_wait.  Calls on one plan must come from one host thread. */
jt_status jt_forward_host_async(jt_plan_t p, const double *coeffs_host, double *values_host, void *cuda_stream);
jt_status jt_inverse_host_async(jt_plan_t p, const double *values_host, double *coeffs_host, void *cuda_stream);
jt_status jt_host_wait(jt_plan_t p);

/* One axis pass (the building block of the slab-distributed schedule):
 * applies axis `axis`'s 1D forward (inverse) transform along the middle index of an
 * (outer, n[axis], inner) C-order device array.  in == out allowed (in place). */
jt_status jt_forward_axis(jt_plan_t p, int axis, const double *in, double *out, int64_t outer,
                          int64_t inner, void *cuda_stream);
jt_status jt_inverse_axis(jt_plan_t p, int axis, const double *in, double *out, int64_t outer,
                          int64_t inner, void *cuda_stream);

/* General axis pass, the building block of the slab-distributed schedule (the paper's
 * "n 2D transforms and n^2 1D transforms", with the transpose between them).  Applies axis
 * `axis`'s 1D forward (inverse != 0: inverse) transform to every line of an (outer, n[axis], inner)
 * device array.  in_split / out_split = G >= 1 (G | n[axis]) select the CHUNK-MAJOR layout of the input /
 * output: with c = n[axis] / G, element j of line (o, i) is at
 *     (j / c) * (outer * c * inner) + o * c * inner + (j % c) * inner + i
 * (G = 1: plain C-order).  Chunk g is then the contiguous block an all-to-all sends to / receives from
 * rank g, so no pack or unpack kernel exists.  Chunk-major layouts need in != out (else JT_ERR_ARG); with
 * both splits 1, in == out is allowed. */
jt_status jt_axis_pass(jt_plan_t p, int axis, int inverse, const double *in, double *out, int64_t outer,
                       int64_t inner, int in_split, int out_split, void *cuda_stream);

/* jt_axis_pass over PART of the rows of a chunk-major array: the chunk-major blocks have ostride >= outer
 * rows (element (o, j, i) at (j / c) * (ostride * c * inner) + o * c * inner + (j % c) * inner + i); pass
 * `out` (or `in`) already offset to the first row of the part.  Used to pipeline the distributed forward's
 * all-to-all with its axis-1 pass.  ostride < outer is JT_ERR_ARG. */
jt_status jt_axis_pass_ex(jt_plan_t p, int axis, int inverse, const double *in, double *out, int64_t outer,
                          int64_t inner, int in_split, int out_split, int64_t ostride, void *cuda_stream);

/* ---- slab-distributed plans ----
 * One process per GPU.  Rank 0 calls jt_dist_unique_id and broadcasts the 128-byte id (e.g. over the
 * torch process group); every rank then calls jt_plan_dist with the same n, a, b, eps, opts.  The library
 * creates and owns an NCCL communicator (libnccl.so.2 is loaded on first use; JT_ERR_NCCL if absent or on
 * any NCCL failure).  Rank g of G holds
 *     forward input / inverse output:  the x-slab  [g n0/G, (g+1) n0/G) x n1 (x n2), C-order
 *     forward output / inverse input:  the y-slab  n0 x [g n1/G, (g+1) n1/G) (x n2), C-order
 * (jt_local_box).  jt_forward / jt_inverse / *_host on a distributed plan take and return these local
 * slabs (out of place) and run: the local axis passes, ONE all-to-all (grouped ncclSend/ncclRecv on the
 * caller's stream) of equal contiguous chunks written directly by the preceding axis pass (chunk-major
 * layout, see jt_axis_pass), then the remaining axis pass.  d must be 2 or 3 and G must divide n0 and n1. */
jt_status jt_dist_unique_id(void *nccl_unique_id /* 128 bytes, written */);
jt_status jt_plan_dist(jt_plan_t *out, int d, const int64_t n[], const double a[], const double b[], double eps,
                       const jt_opts *opts, const void *nccl_unique_id, int rank, int nranks);

/* jt_plan_dist with flags (0 = jt_plan_dist):
 *   JT_DIST_LOWMEM  capacity mode (grids larger than one GPU; the paper's memory claim
 *                   O((r_x + r_y + r_z) n^3), is O(n^3) here): the plan allocates NO slab-sized
 *                   buffers.  jt_forward / jt_inverse use the caller's INPUT slab as their workspace and the
 *                   all-to-all runs between the caller's two slabs (not pipelined), so the input's contents are
 *                   DESTROYED (undefined afterwards); per-GPU memory is the caller's two slabs + the plan's factors
 *                   (a few MB per axis) + NCCL's own buffers: 4096^3 on 8 GPUs needs 2 x 68.7 GB per GPU.  The
 *                   *_host variants stage through one plan-owned pair of slabs (copy in, transform, copy out). */
/*   JT_DIST_NCCL_A2A  use the NCCL all-to-all (grouped ncclSend / ncclRecv in row chunks, pipelined with the
 *                   adjacent pass).  Default (flag clear, pipelined mode): the FUSED exchange where peer memory works --
 *                   every rank's receive buffer is mapped into the other ranks (CUDA IPC, peer access over NVLink /
 *                   NVSwitch; ranks of one node), and the axis pass that produces the chunk-major blocks (forward: axis
 *                   1, inverse: axis 0) stores each block straight into the receive buffer of the rank that owns it,
 *                   so the transfer overlaps the pass line by line and no all-to-all runs; two one-element NCCL
 *                   all-reduces bracket it as barriers.  If any rank cannot map a peer, every rank falls back to the
 *                   NCCL all-to-all (the setup is collective). */
enum { JT_DIST_LOWMEM = 1, JT_DIST_NCCL_A2A = 2 };
jt_status jt_plan_dist_ex(jt_plan_t *out, int d, const int64_t n[], const double a[], const double b[], double eps,
                          const jt_opts *opts, const void *nccl_unique_id, int rank, int nranks, int flags);

/* How the plan exchanges its slabs: JT_MODE_SINGLE (not distributed), JT_MODE_FUSED (the fused peer-store exchange),
 * JT_MODE_A2A (the NCCL all-to-all), JT_MODE_LOWMEM (capacity mode: NCCL all-to-all between the caller's slabs). */
enum { JT_MODE_SINGLE = 0, JT_MODE_FUSED = 1, JT_MODE_A2A = 2, JT_MODE_LOWMEM = 3 };
jt_status jt_dist_mode(jt_plan_t p, int *mode);

/* Wait until the work enqueued on `cuda_stream` has finished.  On a distributed plan the communicator is polled
 * meanwhile (ncclCommGetAsyncError): a failed or dead peer returns JT_ERR_NCCL (the communicator is aborted and
 * every later call on the plan returns JT_ERR_NCCL) instead of hanging.  jt_host_wait and the synchronous *_host
 * calls wait the same way. */
jt_status jt_sync(jt_plan_t p, void *cuda_stream);
/* Index box [lo, hi) of this rank's block: which = 0 the forward input (x-slab), 1 the forward output
 * (y-slab).  Non-distributed plans return the whole array. */
jt_status jt_local_box(jt_plan_t p, int which, int64_t lo[], int64_t hi[]);

/* Free a plan (device buffers included).  jt_destroy(NULL) is JT_OK. */
jt_status jt_destroy(jt_plan_t p);

/* ---- introspection (host; valid for host-only plans too) ---- */

/* Rank r of axis `axis`'s factorisation (eq:approxA: Algorithm 1's complex factors).  It is the
 * number of complex FFTs per line of the unpaired kernels; uniform axes of FFT length 256 / 512 / 2048 / 4096 also carry a
 * second factor set with REAL v_l (two terms per complex FFT, about r/2 FFTs per line), which the library uses by
 * itself for launches of >= 2400 lines (DESIGN.md §6 and reading R26; jt_debug_pair_factors in jt_debug.h shows it;
 * JT_PAIR=0 in the environment at plan time disables it).  Results agree to the plan's eps either way. */
jt_status jt_plan_rank(jt_plan_t p, int axis, int *r);

/* Per-axis sizes: n, the FFT length N (power of two >= max(n,16)), effective k0 = min(k0, n), r. */
jt_status jt_plan_info(jt_plan_t p, int axis, int64_t *n, int64_t *nfft, int *k0, int *r);

/* Nodes t_j (ascending, (0, pi)) and trigonometric weights w_j of axis `axis` into host arrays of
 * length n (introduction:modrule; reading R2 of DESIGN.md).  Either may be NULL. */
jt_status jt_plan_nodes(jt_plan_t p, int axis, double *t_host, double *w_host);

/* Factors of axis `axis` into host arrays (any may be NULL):
 *   u_host    n x r complex (interleaved re,im), column l = u~_l = W u_l S^{1/2} (weights folded)
 *   v_host    r x N complex (interleaved), row l = v_l; zero for k < k0 and k >= n
 *   phiv_host n x k0 real, Phi_V[j,k] = sqrt(w_j) P~_k(t_j), k < k0 (the block W V)
 *   bins_host n int32, m_j = nearest integer to t_j N / (2 pi) (ties to even).
 * So that Phi[j,k] ~ phiv[j,k] (k<k0), Re(sum_l u[j,l] v[l,k] e^{2 pi i m_j k / N}) (k>=k0). */
jt_status jt_plan_factors(jt_plan_t p, int axis, double *u_host, double *v_host, double *phiv_host,
                          int32_t *bins_host);

/* Diagnostics of axis `axis`'s factorisation: the singular values sigma_0..sigma_{count-1} of
 * Algorithm 1's middle matrix (descending; count <= rmax; pass sigma=NULL to query count) and the
 * rank cap used. */
jt_status jt_plan_sigma(jt_plan_t p, int axis, double *sigma, int *count, int *rmax_used);

/* Number of kernels the most recent transform call on p enqueued (jt_forward / jt_inverse / jt_adjoint, the
 * *_host variants, jt_forward_axis / jt_inverse_axis / jt_axis_pass*): one fused axis pass per axis, plus one
 * partial-sum reduction per axis whose rank terms were split over CTAs (few lines).  Used by bench.py's
 * gpu_launches.  JT_ERR_ARG for a NULL p or count. */
jt_status jt_last_launches(jt_plan_t p, int *count);

/* Phase timing (bench.py's per-axis and all-to-all split).  jt_profile(p, 1) makes every later jt_forward /
 * jt_inverse / jt_adjoint on p record CUDA timing events around its phases (a few microseconds per call; 0 turns
 * it off).  jt_last_profile waits for the most recent such call and returns, in milliseconds:
 *   ms[0], ms[1], ms[2]  the axis-0 / axis-1 / axis-2 passes (first launch start to last launch end: the
 *                        distributed schedule runs a pass in row chunks overlapped with the exchange), 0 if absent;
 *   ms[3]                the all-to-all (distributed plans; first chunk start to last chunk end on its stream);
 *   ms[4]                the whole call.
 * JT_ERR_ARG if profiling is off or no profiled call was made. */
jt_status jt_profile(jt_plan_t p, int enable);
jt_status jt_last_profile(jt_plan_t p, double ms[5]);

/* Thread-local text of the last non-OK status ("" if none). */
const char *jt_last_error(void);

/* Library version string. */
const char *jt_version(void);

#ifdef __cplusplus
}
#endif
#endif /* JT_H */
