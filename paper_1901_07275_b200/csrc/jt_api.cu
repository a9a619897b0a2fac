// C ABI of libjt.so (include/jt.h): plan lifetime, host->device upload of the per-axis factors,
// and the axis-pass schedule of the d-dimensional transform (eq:TJ PAPER.md:669-674, eq:TJ3
// PAPER.md:718-722): one fused kernel launch per axis, the first reading the input array, the rest in
// place on the output array.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "launch.cuh"
#include "jt_debug.h"
#include "jt_internal.h"

// (JT_HOST_SLOTS, JT_R512, JT_R4096: tuning.h.)  The *_host entry points rotate through JT_HOST_SLOTS staging
// slots, so a call's input copy only waits for the output copy of the call JT_HOST_SLOTS back.

namespace {

using namespace jtl;

struct AxisDevBuf {
  double2 *ub = nullptr, *v = nullptr, *tw = nullptr, *tw_ts = nullptr;  // tw_ts: only if the radixes differ
  double *phivb = nullptr, *phivc = nullptr;
  int *bstart = nullptr;
  int maxr = 0;  // row slots per bin in ub / phivb (template MAXR of the kernels)
};

// Restores the caller's current device on scope exit.
struct DeviceGuard {
  int prev = -1;
  bool changed = false;
  explicit DeviceGuard(int dev) {
    if (dev >= 0 && cudaGetDevice(&prev) == cudaSuccess && prev != dev) {
      changed = cudaSetDevice(dev) == cudaSuccess;
    }
  }
  ~DeviceGuard() {
    if (changed) cudaSetDevice(prev);
  }
};
}  // namespace

// ---- NCCL, loaded on first use (dlopen of libnccl.so.2: the one torch already loaded, else the system's) ----
namespace nccl {
typedef struct { char internal[128]; } UniqueId;
typedef void *Comm;
enum { Success = 0, Float64 = 8, InProgress = 7, Uint8 = 1, Int32 = 2, Sum = 0, Min = 3 };
struct Api {
  bool ok = false;
  std::string why;
  int (*GetUniqueId)(UniqueId *) = nullptr;
  int (*CommInitRank)(Comm *, int, UniqueId, int) = nullptr;
  int (*CommDestroy)(Comm) = nullptr;
  int (*CommAbort)(Comm) = nullptr;
  int (*CommGetAsyncError)(Comm, int *) = nullptr;
  int (*Send)(const void *, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*Recv)(void *, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*AllGather)(const void *, void *, size_t, int, Comm, cudaStream_t) = nullptr;
  int (*AllReduce)(const void *, void *, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(int) = nullptr;
};
Api &api() {
  static Api a = [] {
    Api r;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      r.why = std::string("dlopen libnccl.so.2: ") + dlerror();
      return r;
    }
    r.GetUniqueId = (int (*)(UniqueId *))dlsym(h, "ncclGetUniqueId");
    r.CommInitRank = (int (*)(Comm *, int, UniqueId, int))dlsym(h, "ncclCommInitRank");
    r.CommDestroy = (int (*)(Comm))dlsym(h, "ncclCommDestroy");
    r.CommAbort = (int (*)(Comm))dlsym(h, "ncclCommAbort");
    r.CommGetAsyncError = (int (*)(Comm, int *))dlsym(h, "ncclCommGetAsyncError");
    r.Send = (int (*)(const void *, size_t, int, int, Comm, cudaStream_t))dlsym(h, "ncclSend");
    r.Recv = (int (*)(void *, size_t, int, int, Comm, cudaStream_t))dlsym(h, "ncclRecv");
    r.AllGather = (int (*)(const void *, void *, size_t, int, Comm, cudaStream_t))dlsym(h, "ncclAllGather");
    r.AllReduce = (int (*)(const void *, void *, size_t, int, int, Comm, cudaStream_t))dlsym(h, "ncclAllReduce");
    r.GroupStart = (int (*)())dlsym(h, "ncclGroupStart");
    r.GroupEnd = (int (*)())dlsym(h, "ncclGroupEnd");
    r.GetErrorString = (const char *(*)(int))dlsym(h, "ncclGetErrorString");
    r.ok = r.GetUniqueId && r.CommInitRank && r.CommDestroy && r.CommAbort && r.CommGetAsyncError && r.Send &&
           r.Recv && r.AllGather && r.AllReduce && r.GroupStart && r.GroupEnd && r.GetErrorString;
    if (!r.ok) r.why = "libnccl.so.2 lacks a required symbol";
    return r;
  }();
  return a;
}
}  // namespace nccl

struct jt_plan_s {
  int d = 0;
  int64_t n[3] = {0, 0, 0};
  double a[3] = {0, 0, 0}, b[3] = {0, 0, 0}, eps = 0;
  jt_opts opts{};
  int device = -2;  // -2: host-only
  jt::AxisHost host[3];
  AxisDevBuf dev[3];
  // paired real rank terms (forward kernels with Cfg::PAIR): a second factor set per axis, used by the
  // forward passes only (the inverse / transpose keep the unpaired complex factors)
  bool pair[3] = {false, false, false};
  jt::AxisHost hostp[3];
  AxisDevBuf devp[3];
  int64_t total = 0;
  // *_host entry points: two staging slots (consecutive calls alternate, so one call's input copy overlaps the
  // previous call's output copy), their copy streams and events
  double *stage_in[JT_HOST_SLOTS] = {}, *stage_out[JT_HOST_SLOTS] = {};
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev[2 * 16 + 2] = {};
  cudaEvent_t ev_free[JT_HOST_SLOTS] = {};  // slot's last output copy done
  unsigned host_calls = 0;
  mutable jtl::LaunchState ls;  // kernels enqueued by the latest call (jt_last_launches), term-split workspace
  // slab-distributed plans (jt_plan_dist): this rank's x-slab (forward input) / y-slab
  // (forward output) of the global n[0] x n[1] (x n[2]) array, the all-to-all buffers and the NCCL comm
  bool dist = false;
  int rank = 0, nranks = 1;
  int dist_flags = 0;      // JT_DIST_* (jt_plan_dist_ex)
  nccl::Comm comm = nullptr;
  jt_vgroup_s *vgroup = nullptr;  // test-only in-process exchange (include/jt_debug.h) instead of NCCL
  bool broken = false;     // a failed exchange aborted the communicator: every later call is JT_ERR_NCCL
  double *a2a_send = nullptr, *a2a_recv = nullptr;  // (not allocated with JT_DIST_LOWMEM; no send buffer with p2p)
  // fused slab exchange (the default where peer memory works): every rank's receive buffer mapped into every other
  // rank (CUDA IPC over NVLink; the virtual group: same-process pointers); the pass before the exchange stores each
  // chunk-major block straight into its owner's receive buffer, bracketed by two tiny barriers (dist_barrier)
  bool p2p = false;
  double *peer_recv[jtk::MAX_SPLIT] = {};
  bool peer_ipc[jtk::MAX_SPLIT] = {};  // peer_recv[g] was opened with cudaIpcOpenMemHandle (closed at destroy)
  // element offsets (from this rank's receive buffer) of block `rank` in every rank's receive buffer, on the host
  // and (read by the kernels' chunk-major output addressing) on the device; set by resolve_peers
  long long h_peer_off[jtk::MAX_SPLIT] = {};
  long long *d_peer_off = nullptr;
  bool peers_resolved = false;
  double *bar_buf = nullptr;           // one double for the NCCL barrier (an all-reduce)
  mutable cudaStream_t s_comm = nullptr;  // the pipelined all-to-all's stream (created on first use)
  mutable cudaEvent_t ev_chunk[8] = {}, ev_comm = nullptr;
  // plan-owned buffers (staging, all-to-all, term-split workspace) are reused by every call: a call's first
  // work waits for the previous call's last use (recorded at its end), whatever streams the two calls use
  mutable cudaEvent_t ev_busy = nullptr;
  // phase timing (jt_profile / jt_last_profile): timing events, recorded by transform / transform_dist
  bool prof_on = false;
  mutable cudaEvent_t pev[10] = {};
  mutable bool prec[10] = {};
};

// Test-only virtual exchange group (include/jt_debug.h): G plans on ONE device, each driven by its own host
// thread and stream, exchange their all-to-all blocks by cudaMemcpyAsync between their buffers, ordered by
// cross-stream events and a host barrier (no kernel waits on another: the copies are plain stream work).
struct jt_vgroup_s {
  int G = 0;
  int timeout_ms = 120000;
  std::vector<jt_plan_s *> member;      // by rank
  std::vector<const double *> send;     // each member's send buffer of the exchange in progress
  std::vector<cudaEvent_t> ev_ready, ev_done;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  bool failed = false;
  // all G members arrive (or the group is marked failed after timeout_ms)
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (failed) return false;
    const unsigned long long g = gen;
    if (++arrived == G) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    if (!cv.wait_for(lk, std::chrono::milliseconds(timeout_ms), [&] { return gen != g || failed; }) || failed) {
      failed = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};

namespace {

jtk::AxisDev axis_dev(const jt_plan_s *p, int axis, bool pair = false) {
  const jt::AxisHost &h = pair ? p->hostp[axis] : p->host[axis];
  const AxisDevBuf &dv = pair ? p->devp[axis] : p->dev[axis];
  jtk::AxisDev ax;
  ax.n = (int)h.n;
  ax.N = (int)h.N;
  ax.k0 = h.k0;
  ax.r = h.r;
  ax.nbins = (int)(h.N / 2 + 1);
  ax.v = dv.v;
  ax.ub = dv.ub;
  ax.phivb = dv.phivb;
  ax.phivc = dv.phivc;
  ax.bstart = dv.bstart;
  ax.tw = dv.tw;
  ax.tw_ts = dv.tw_ts ? dv.tw_ts : dv.tw;
  return ax;
}

// One axis pass over the (outer, n[axis], inner) array; in_split / out_split = G > 1 selects the chunk-major
// layout of the slab all-to-all for the input / output.
// in_lim / out_lim: elements of the input / output buffers from the given pointers (bounds of the JT_CHECKS
// build; -1: the extent the geometry addresses).  peer: the fused slab exchange -- the out_split output blocks
// live in the ranks' receive buffers, at the plan's peer offsets (from `out` = this rank's receive buffer) + the
// row offset peer_row; false: one buffer, block g at g ostride (n / out_split) inner.
jt_status launch_axis(const jt_plan_s *p, int axis, bool inverse, const double *in, double *out, long long outer,
                      long long inner, cudaStream_t s, int in_split = 1, int out_split = 1,
                      long long nlines_only = -1, bool allow_ts = true, long long ostride = -1,
                      long long in_lim = -1, long long out_lim = -1, bool peer = false, long long peer_row = 0) {
  // nlines_only >= 0: only the first nlines_only lines (a column block of an outer == 1 pass)
  const long long nlines = nlines_only >= 0 ? nlines_only : outer * inner;
  // paired real terms: forward passes only, and only launches with enough lines to fill the GPU without a term
  // split (the few-line, latency-bound launches keep the unpaired kernels and their one-warp-group / cluster term
  // split: 256^2 forward 27 us unpaired vs 35 us paired, r02zz3)
  const bool pr = p->pair[axis] && nlines >= JT_PAIR_MIN_LINES && (!inverse || JT_PAIR_INV);
  jtk::AxisDev ax = axis_dev(p, axis, pr);
  const int maxr = pr ? -2 : p->dev[axis].maxr;  // (-2: launch_n's tag for the Cfg::PAIR kernels)
  const long long ost = ostride >= 0 ? ostride : outer;
  const long long n = p->n[axis];
  const long long geo_in = (in_split > 1 ? ost : outer) * n * inner, geo_out = (out_split > 1 ? ost : outer) * n * inner;
  if (peer && out_split == 1) {  // one block (a world of one): the plain layout at that block's place
    out += p->h_peer_off[0] + peer_row;
    peer = false;
  }
  const jtk::Layout lay{outer, inner, (int)(n / in_split), (int)(n / out_split), ost,
                        in_lim >= 0 ? in_lim : geo_in, out_lim >= 0 ? out_lim : geo_out,
                        peer ? p->d_peer_off : nullptr, peer ? peer_row : 0};
  switch (ax.N) {
    case 16: return launch_n<16>(p->ls, inverse, maxr, ax, in, out, nlines, lay, s, allow_ts);
    case 32: return launch_n<32>(p->ls, inverse, maxr, ax, in, out, nlines, lay, s, allow_ts);
    case 64: return launch_n<64>(p->ls, inverse, maxr, ax, in, out, nlines, lay, s, allow_ts);
    case 128: return launch_n<128>(p->ls, inverse, maxr, ax, in, out, nlines, lay, s, allow_ts);
    case 256: return launch_n<256>(p->ls, inverse, maxr, ax, in, out, nlines, lay, s, allow_ts);
    case 512: return launch_n<512>(p->ls, inverse, maxr, ax, in, out, nlines, lay, s, allow_ts);
    case 1024: return launch_n<1024>(p->ls, inverse, maxr, ax, in, out, nlines, lay, s, allow_ts);
    case 2048: return launch_n<2048>(p->ls, inverse, maxr, ax, in, out, nlines, lay, s, allow_ts);
    case 4096: return launch_n<4096>(p->ls, inverse, maxr, ax, in, out, nlines, lay, s, allow_ts);
    default: return fail(JT_ERR_ARG, "unsupported FFT length");
  }
}

template <class T>
jt_status upload(T **dst, const T *src, size_t count) {
  if (count == 0) {
    *dst = nullptr;
    return JT_OK;
  }
  cudaError_t e = cudaMalloc((void **)dst, count * sizeof(T));
  if (e != cudaSuccess) return fail(JT_ERR_ALLOC, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  e = cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return fail(JT_ERR_CUDA, std::string("cudaMemcpy: ") + cudaGetErrorString(e));
  return JT_OK;
}

void free_device(jt_plan_s *p) {
  if (p->device < 0) return;
  DeviceGuard g(p->device);
  for (int i = 0; i < 3; ++i)
    for (AxisDevBuf *dv : {&p->dev[i], &p->devp[i]}) {
      cudaFree(dv->ub);
      cudaFree(dv->v);
      cudaFree(dv->tw);
      cudaFree(dv->tw_ts);
      cudaFree(dv->phivb);
      cudaFree(dv->phivc);
      cudaFree(dv->bstart);
      *dv = AxisDevBuf();
    }
  for (int k = 0; k < JT_HOST_SLOTS; ++k) {
    cudaFree(p->stage_in[k]);
    cudaFree(p->stage_out[k]);
    p->stage_in[k] = p->stage_out[k] = nullptr;
    if (p->ev_free[k]) cudaEventDestroy(p->ev_free[k]), p->ev_free[k] = nullptr;
  }
  cudaFree(p->ls.ts_work);
  p->ls.ts_work = nullptr;
  p->ls.ts_elems = 0;
  for (int g = 0; g < jtk::MAX_SPLIT; ++g)
    if (p->peer_ipc[g]) cudaIpcCloseMemHandle(p->peer_recv[g]), p->peer_ipc[g] = false;
  cudaFree(p->bar_buf);
  p->bar_buf = nullptr;
  cudaFree(p->d_peer_off);
  p->d_peer_off = nullptr;
  cudaFree(p->a2a_send);
  cudaFree(p->a2a_recv);
  p->a2a_send = p->a2a_recv = nullptr;
  if (p->comm) (p->broken ? nccl::api().CommAbort(p->comm) : nccl::api().CommDestroy(p->comm)), p->comm = nullptr;
  if (p->vgroup) {
    std::lock_guard<std::mutex> lk(p->vgroup->mu);
    p->vgroup->member[p->rank] = nullptr;
    if (p->vgroup->ev_ready[p->rank]) cudaEventDestroy(p->vgroup->ev_ready[p->rank]), p->vgroup->ev_ready[p->rank] = nullptr;
    if (p->vgroup->ev_done[p->rank]) cudaEventDestroy(p->vgroup->ev_done[p->rank]), p->vgroup->ev_done[p->rank] = nullptr;
    p->vgroup = nullptr;
  }
  if (p->ev_busy) cudaEventDestroy(p->ev_busy), p->ev_busy = nullptr;
  for (auto &e : p->pev)
    if (e) cudaEventDestroy(e), e = nullptr;
  for (auto &e : p->ev_chunk)
    if (e) cudaEventDestroy(e), e = nullptr;
  if (p->ev_comm) cudaEventDestroy(p->ev_comm), p->ev_comm = nullptr;
  if (p->s_comm) cudaStreamDestroy(p->s_comm), p->s_comm = nullptr;
  for (auto &e : p->ev)
    if (e) cudaEventDestroy(e), e = nullptr;
  if (p->s_h2d) cudaStreamDestroy(p->s_h2d), p->s_h2d = nullptr;
  if (p->s_d2h) cudaStreamDestroy(p->s_d2h), p->s_d2h = nullptr;
}

jt_status upload_axis(jt_plan_s *p, int axis, bool pair = false) {
  const jt::AxisHost &h = pair ? p->hostp[axis] : p->host[axis];
  AxisDevBuf &dv = pair ? p->devp[axis] : p->dev[axis];
  const int64_t N = h.N;
  const int r = h.r, k0 = h.k0;
  const int64_t nbins = N / 2 + 1;
  // bin-major layouts (rows of bin m in slots c < MAXR, zero padded) so that a thread owning bin m
  // reads u~ and W V of all its rows with unit-stride vector loads
  int maxr = 0;
  for (int64_t m = 0; m < nbins; ++m) maxr = std::max(maxr, h.bstart[m + 1] - h.bstart[m]);
  if (maxr > 4) return fail(JT_ERR_NUMERIC, "more than 4 nodes share one FFT bin");
  const int MAXR = maxr <= 2 ? 2 : maxr;  // 2 (Gauss-Jacobi nodes), 3 or 4 (clustered nonuniform points)
  if (pair && MAXR != 2) return fail(JT_ERR_NUMERIC, "pair: more than 2 nodes share one FFT bin");
  dv.maxr = MAXR;
  const int UC = pair ? 2 : 1;  // factor columns per term in h.u (pair: P and conj(Q)), rows per bin slot in ub
  std::vector<double2> ub((size_t)r * nbins * MAXR * UC, make_double2(0.0, 0.0)), v((size_t)r * N), tw(N);
  std::vector<double> phivb((size_t)std::max(k0, 1) * nbins * MAXR, 0.0);
  const int KPT = pair ? jtk::VST_KPT_PAIR : jtk::VST_KPT;  // chunk size of the kernels' staged W V (degrees per term)
  const int nchunk = std::max((k0 + KPT - 1) / KPT, 1);
  std::vector<double> phivc((size_t)nchunk * nbins * MAXR * KPT, 0.0);
  for (int64_t m = 0; m < nbins; ++m) {
    for (int c = 0; c < h.bstart[m + 1] - h.bstart[m]; ++c) {
      const int64_t j = h.bstart[m] + c;
      for (int l = 0; l < r; ++l)
        for (int hh = 0; hh < UC; ++hh) {  // (pair: row 2 c of term l = P, row 2 c + 1 = conj(Q))
          const jt::cd z = h.u[(size_t)j * r * UC + l * UC + hh];
          ub[((size_t)l * MAXR * UC + c * UC + hh) * nbins + m] = make_double2(z.real(), z.imag());
        }
      for (int k = 0; k < k0; ++k) {
        phivb[((size_t)k * MAXR + c) * nbins + m] = h.phiv[(size_t)j * k0 + k];
        phivc[(((size_t)(k / 2) * nbins + m) * MAXR + c) * 2 + (k % 2)] = h.phiv[(size_t)j * k0 + k];  // 2-degree chunks
      }
    }
  }
  for (int l = 0; l < r; ++l) {
    for (int64_t k = 0; k < N; ++k) {
      const jt::cd z = h.v[(size_t)l * N + k];
      v[(size_t)l * N + k] = make_double2(z.real(), z.imag());
    }
  }
  // per-pass twiddle tables (jtk::TwOff): for each pass after the first, at sub-size NS with radix RS,
  // entries (r-1) NS + j = e^{+2 pi i j r / (NS RS)}, computed in long double and rounded once
  const long double PI_L = 3.141592653589793238462643383279502884L;
  auto tw_table = [&](int R) {
    std::vector<double2> t;
    int64_t NS = std::min<int64_t>(N, R);
    while (NS < N) {
      const int64_t RS = std::min<int64_t>(N / NS, R);
      for (int64_t r = 1; r < RS; ++r)
        for (int64_t j = 0; j < NS; ++j) {
          const long double ang = 2 * PI_L * (long double)(j * r) / (long double)(NS * RS);
          t.push_back(make_double2((double)cosl(ang), (double)sinl(ang)));
        }
      NS *= RS;
    }
    if (t.empty()) t.push_back(make_double2(1.0, 0.0));
    return t;
  };
  tw = tw_table(pair ? pair_radix(N) : radix_of(N, MAXR));
  jt_status s;
  if ((s = upload(&dv.ub, ub.data(), ub.size())) != JT_OK) return s;
  if ((s = upload(&dv.v, v.data(), v.size())) != JT_OK) return s;
  if ((s = upload(&dv.tw, tw.data(), tw.size())) != JT_OK) return s;
  if (!pair && radix_ts_of(N, MAXR) != radix_of(N, MAXR)) {
    const std::vector<double2> tts = tw_table(radix_ts_of(N, MAXR));
    if ((s = upload(&dv.tw_ts, tts.data(), tts.size())) != JT_OK) return s;
  }
  if ((s = upload(&dv.phivb, phivb.data(), phivb.size())) != JT_OK) return s;
  if ((s = upload(&dv.phivc, phivc.data(), phivc.size())) != JT_OK) return s;
  if ((s = upload(&dv.bstart, h.bstart.data(), h.bstart.size())) != JT_OK) return s;
  return JT_OK;
}

bool overlaps_partially(const double *x, const double *y, int64_t count) {
  if (x == y) return false;
  const double *xe = x + count, *ye = y + count;
  return x < ye && y < xe;
}

// Abort the plan's communicator after a failed or hung exchange (peers blocked on chunks this rank will never
// post get an error from their own communicator instead of hanging), and refuse every later call.
jt_status mark_broken(const jt_plan_s *p, const std::string &msg) {
  jt_plan_s *q = const_cast<jt_plan_s *>(p);
  if (q->comm && !q->broken) nccl::api().CommAbort(q->comm), q->comm = nullptr;
  q->broken = true;
  return fail(JT_ERR_NCCL, msg);
}

// Asynchronous NCCL errors of a distributed plan (a dead or failed peer): JT_ERR_NCCL and abort.
jt_status poll_comm(const jt_plan_s *p) {
  if (p->broken) return fail(JT_ERR_NCCL, "the plan's communicator was aborted after an earlier exchange failure");
  if (!p->comm) return JT_OK;
  int ae = nccl::Success;
  const int e = nccl::api().CommGetAsyncError(p->comm, &ae);
  if (e != nccl::Success) return mark_broken(p, std::string("ncclCommGetAsyncError: ") + nccl::api().GetErrorString(e));
  if (ae != nccl::Success && ae != nccl::InProgress)
    return mark_broken(p, std::string("asynchronous NCCL error: ") + nccl::api().GetErrorString(ae));
  return JT_OK;
}

jt_status check_device_plan(const jt_plan_s *p) {
  if (!p) return fail(JT_ERR_ARG, "null plan");
  if (p->device < 0) return fail(JT_ERR_ARG, "host-only plan (opts.device == -2) cannot run device calls");
  if (p->dist) {
    jt_status st = poll_comm(p);
    if (st != JT_OK) return st;
  }
  // surface an asynchronous fault from an earlier call
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(JT_ERR_CUDA, std::string("pending CUDA error: ") + cudaGetErrorString(e));
  }
  return JT_OK;
}

// Ordering of calls that share the plan-owned buffers: the call's stream waits for the previous call's end.
jt_status begin_call(const jt_plan_s *p, cudaStream_t s) {
  if (capturing(s)) return JT_OK;  // (a graph orders its own nodes; the events are recorded by uncaptured calls)
  if (!p->ev_busy) {
    JT_CUDA_TRY(cudaEventCreateWithFlags(&p->ev_busy, cudaEventDisableTiming));
    JT_CUDA_TRY(cudaEventRecord(p->ev_busy, s));
  }
  JT_CUDA_TRY(cudaStreamWaitEvent(s, p->ev_busy, 0));
  return JT_OK;
}
jt_status end_call(const jt_plan_s *p, cudaStream_t s) {
  if (capturing(s)) return JT_OK;
  JT_CUDA_TRY(cudaEventRecord(p->ev_busy, s));
  return JT_OK;
}

// Phase marks for jt_last_profile: 0 call start, 1 call end, 2 + 2 i / 3 + 2 i axis i pass start / end,
// 8 / 9 exchange start / end (comm stream).
enum { PM_START = 0, PM_END = 1, PM_AX = 2, PM_XS = 8, PM_XE = 9 };
jt_status mark(const jt_plan_s *p, int id, cudaStream_t s) {
  if (!p->prof_on || capturing(s)) return JT_OK;
  if (!p->pev[id]) JT_CUDA_TRY(cudaEventCreate(&p->pev[id]));
  JT_CUDA_TRY(cudaEventRecord(p->pev[id], s));
  p->prec[id] = true;
  return JT_OK;
}
void reset_marks(const jt_plan_s *p) {
  for (auto &r : p->prec) r = false;
}

// Comm stream and events of the pipelined all-to-all (created on first use).
jt_status ensure_comm_stream(const jt_plan_s *p) {
  if (!p->s_comm) {
    JT_CUDA_TRY(cudaStreamCreateWithFlags(&p->s_comm, cudaStreamNonBlocking));
    for (auto &e : p->ev_chunk) JT_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    JT_CUDA_TRY(cudaEventCreateWithFlags(&p->ev_comm, cudaEventDisableTiming));
  }
  return JT_OK;
}

// In-process exchange of a virtual group (test only, include/jt_debug.h): rank `me` copies rows [off, off + cnt)
// of block `me` of every member's send buffer into block g of its own receive buffer.  Barrier 1: every member
// has published its send buffer and recorded "my rows are written" (ev_ready) on its stream; barrier 2: every
// member has enqueued its copies and recorded "I have read my peers' rows" (ev_done); every stream then waits
// for all ev_done, so no member reuses its send buffer before its peers' copies ran (NCCL's completion rule);
// barrier 3: all those waits are enqueued before any member re-records its events in the next exchange.
jt_status vgroup_exchange(const jt_plan_s *p, const double *send, double *recv, size_t chunk, size_t off, size_t cnt,
                          cudaStream_t s) {
  jt_vgroup_s *V = p->vgroup;
  const int me = p->rank;
  {
    std::lock_guard<std::mutex> lk(V->mu);
    V->send[me] = send;
  }
  JT_CUDA_TRY(cudaEventRecord(V->ev_ready[me], s));
  if (!V->barrier()) return mark_broken(p, "virtual exchange: a peer did not arrive (barrier 1 timed out)");
  for (int g = 0; g < V->G; ++g) {
    JT_CUDA_TRY(cudaStreamWaitEvent(s, V->ev_ready[g], 0));
    JT_CUDA_TRY(cudaMemcpyAsync(recv + g * chunk + off, V->send[g] + me * chunk + off, cnt * sizeof(double),
                                cudaMemcpyDeviceToDevice, s));
  }
  JT_CUDA_TRY(cudaEventRecord(V->ev_done[me], s));
  if (!V->barrier()) return mark_broken(p, "virtual exchange: a peer did not arrive (barrier 2 timed out)");
  for (int g = 0; g < V->G; ++g) JT_CUDA_TRY(cudaStreamWaitEvent(s, V->ev_done[g], 0));
  if (!V->barrier()) return mark_broken(p, "virtual exchange: a peer did not arrive (barrier 3 timed out)");
  return JT_OK;
}

// All-to-all of rows [r0, r1) (rowlen elements each) of every contiguous chunk-major block (block g to /
// from rank g) between `send` and `recv` on stream s; the whole exchange is r0 = 0, r1 = rows per block.
// A failure after earlier chunks were posted aborts the communicator (mark_broken), so the peers' pending
// receives fail instead of hanging.
jt_status all_to_all_rows(const jt_plan_s *p, const double *send, double *recv, long long r0, long long r1,
                          long long rowlen, cudaStream_t s) {
  const size_t chunk = (size_t)p->total / p->nranks;
  const size_t off = (size_t)(r0 * rowlen), cnt = (size_t)((r1 - r0) * rowlen);
  if (p->vgroup) return vgroup_exchange(p, send, recv, chunk, off, cnt, s);
  nccl::Api &A = nccl::api();
  int e = A.GroupStart();
  for (int g = 0; g < p->nranks && e == nccl::Success; ++g) {
    e = A.Send(send + g * chunk + off, cnt, nccl::Float64, g, p->comm, s);
    if (e == nccl::Success) e = A.Recv(recv + g * chunk + off, cnt, nccl::Float64, g, p->comm, s);
  }
  const int e2 = A.GroupEnd();
  if (e != nccl::Success || e2 != nccl::Success)
    return mark_broken(p, std::string("all-to-all: ") + A.GetErrorString(e != nccl::Success ? e : e2));
  return poll_comm(p);
}

// Barrier of the fused exchange on stream s: every rank's stream has reached this point before any continues
// (NCCL: a one-double all-reduce; virtual group: cross-stream events + the host barrier).  Before the pass that
// stores into the peers' receive buffers it guarantees the peers are done reading them (their previous call's
// last pass); after it, that every peer's stores into this rank's receive buffer are complete.
jt_status dist_barrier(const jt_plan_s *p, cudaStream_t s) {
  if (p->vgroup) {
    jt_vgroup_s *V = p->vgroup;
    JT_CUDA_TRY(cudaEventRecord(V->ev_ready[p->rank], s));
    if (!V->barrier()) return mark_broken(p, "virtual barrier: a peer did not arrive");
    for (int g = 0; g < V->G; ++g) JT_CUDA_TRY(cudaStreamWaitEvent(s, V->ev_ready[g], 0));
    if (!V->barrier()) return mark_broken(p, "virtual barrier: a peer did not arrive");
    return JT_OK;
  }
  nccl::Api &A = nccl::api();
  const int e = A.AllReduce(p->bar_buf, p->bar_buf, 1, nccl::Float64, nccl::Sum, p->comm, s);
  if (e != nccl::Success) return mark_broken(p, std::string("barrier all-reduce: ") + A.GetErrorString(e));
  return poll_comm(p);
}

// The fused exchange's block offsets (h_peer_off / d_peer_off): block `rank` of rank g's receive buffer, in elements
// from this rank's receive buffer (the launches' `out`).  Computed once; the virtual group resolves its members'
// buffers here (they exist once every member's plan is built), the NCCL plans from the IPC-mapped pointers.
jt_status resolve_peers(const jt_plan_s *p, cudaStream_t s) {
  if (p->peers_resolved) return JT_OK;
  jt_plan_s *q = const_cast<jt_plan_s *>(p);
  const long long chunk = p->total / p->nranks;
  for (int g = 0; g < p->nranks; ++g) {
    const double *base = p->peer_recv[g];
    if (p->vgroup) {
      std::lock_guard<std::mutex> lk(p->vgroup->mu);
      base = p->vgroup->member[g] ? p->vgroup->member[g]->a2a_recv : nullptr;
    }
    if (!base) return fail(JT_ERR_ARG, "fused exchange: rank " + std::to_string(g) + " has no plan yet");
    q->h_peer_off[g] = (long long)(base - p->a2a_recv) + p->rank * chunk;
  }
  if (!q->d_peer_off && cudaMalloc((void **)&q->d_peer_off, jtk::MAX_SPLIT * sizeof(long long)) != cudaSuccess)
    return fail(JT_ERR_ALLOC, "peer offsets");
  JT_CUDA_TRY(cudaMemcpyAsync(q->d_peer_off, q->h_peer_off, jtk::MAX_SPLIT * sizeof(long long), cudaMemcpyHostToDevice, s));
  JT_CUDA_TRY(cudaStreamSynchronize(s));  // (h_peer_off is the source: keep it alive and the copy done)
  q->peers_resolved = true;
  return JT_OK;
}

// Slab schedule of a distributed plan (the C twin of paper_1901_07275_b200/dist.py SlabPlan):
//   forward: axes d-1..1 on the x-slab (axis 1 written chunk-major), all-to-all, axis 0 on the y-slab; the
//            axis-1 pass and the all-to-all are pipelined over KA row chunks of the slab: chunk k's rows are
//            sent (comm stream) while chunk k+1's axis-1 pass computes;
//   inverse: axis d-1 and axis 0 (written chunk-major) on the y-slab, all-to-all, axis 1 read chunk-major; the
//            all-to-all and the axis-1 pass are pipelined over KA row chunks of the x-slab (receiver side).
//
// JT_DIST_LOWMEM (NEXT-2 capacity mode): no plan-owned slab buffers; the caller's INPUT slab is the workspace
// (its contents are destroyed) and the exchange runs between the caller's two slabs, not pipelined:
//   forward: axis d-1 in place on `in`, axis 1 in -> out (chunk-major), all-to-all out -> in, axis 0 in -> out;
//   inverse: axis d-1 in place on `in`, axis 0 in -> out (chunk-major), all-to-all out -> in, axis 1 in -> out.
jt_status transform_dist(const jt_plan_s *p, bool inverse, const double *in, double *out, cudaStream_t s) {
  const int G = p->nranks, d = p->d;
  const long long n0 = p->n[0], n1 = p->n[1], r = d == 3 ? p->n[2] : 1;
  const long long R = n0 / G, c = n1 / G;  // slab rows, chunk length of axis 1
  jt_status st;
  if ((st = ensure_comm_stream(p)) != JT_OK) return st;
  if (p->dist_flags & JT_DIST_LOWMEM) {
    double *work = const_cast<double *>(in);  // documented: the input slab is the workspace
    if (d == 3) {
      if ((st = mark(p, PM_AX + 4, s)) != JT_OK) return st;
      if ((st = launch_axis(p, 2, inverse, work, work, inverse ? n0 * c : R * n1, 1, s)) != JT_OK) return st;
      if ((st = mark(p, PM_AX + 5, s)) != JT_OK) return st;
    }
    const int ax1 = inverse ? 0 : 1;  // the pass before the exchange
    if ((st = mark(p, PM_AX + 2 * ax1, s)) != JT_OK) return st;
    if (inverse) st = launch_axis(p, 0, true, work, out, 1, c * r, s, 1, G);
    else st = launch_axis(p, 1, false, work, out, R, r, s, 1, G);
    if (st != JT_OK) return st;
    if ((st = mark(p, PM_AX + 2 * ax1 + 1, s)) != JT_OK) return st;
    if ((st = mark(p, PM_XS, s)) != JT_OK) return st;
    if ((st = all_to_all_rows(p, out, work, 0, R, c * r, s)) != JT_OK) return st;
    if ((st = mark(p, PM_XE, s)) != JT_OK) return st;
    const int ax2 = inverse ? 1 : 0;
    if ((st = mark(p, PM_AX + 2 * ax2, s)) != JT_OK) return st;
    if (inverse) st = launch_axis(p, 1, true, work, out, R, r, s, G, 1);
    else st = launch_axis(p, 0, false, work, out, 1, c * r, s);
    if (st != JT_OK) return st;
    return mark(p, PM_AX + 2 * ax2 + 1, s);
  }
  if (p->p2p) {
    // fused exchange: the pass before it stores every chunk-major block straight into the receive buffer of the rank
    // that owns it (over NVLink), so the transfer overlaps the pass line by line; two barriers bracket it
    if ((st = resolve_peers(p, s)) != JT_OK) return st;
    if (d == 3) {
      if ((st = mark(p, PM_AX + 4, s)) != JT_OK) return st;
      if ((st = launch_axis(p, 2, inverse, in, out, inverse ? n0 * c : R * n1, 1, s)) != JT_OK) return st;
      if ((st = mark(p, PM_AX + 5, s)) != JT_OK) return st;
    }
    const double *src = d == 3 ? out : in;
    if ((st = dist_barrier(p, s)) != JT_OK) return st;  // the peers are done reading their receive buffers
    const int ax1 = inverse ? 0 : 1, ax2 = inverse ? 1 : 0;
    if ((st = mark(p, PM_AX + 2 * ax1, s)) != JT_OK) return st;
    if (inverse) st = launch_axis(p, 0, true, src, p->a2a_recv, 1, c * r, s, 1, G, -1, true, -1, -1, -1, true, 0);
    else st = launch_axis(p, 1, false, src, p->a2a_recv, R, r, s, 1, G, -1, true, -1, -1, -1, true, 0);
    if (st != JT_OK) return st;
    if ((st = mark(p, PM_AX + 2 * ax1 + 1, s)) != JT_OK) return st;
    if ((st = mark(p, PM_XS, s)) != JT_OK) return st;
    if ((st = dist_barrier(p, s)) != JT_OK) return st;  // every rank's blocks have landed here
    if ((st = mark(p, PM_XE, s)) != JT_OK) return st;
    if ((st = mark(p, PM_AX + 2 * ax2, s)) != JT_OK) return st;
    if (inverse) st = launch_axis(p, 1, true, p->a2a_recv, out, R, r, s, G, 1);
    else st = launch_axis(p, 0, false, p->a2a_recv, out, 1, c * r, s);
    if (st != JT_OK) return st;
    return mark(p, PM_AX + 2 * ax2 + 1, s);
  }
  if (!inverse) {
    const double *src1 = in;
    if (d == 3) {
      if ((st = mark(p, PM_AX + 4, s)) != JT_OK) return st;
      if ((st = launch_axis(p, 2, false, in, out, R * n1, 1, s)) != JT_OK) return st;
      if ((st = mark(p, PM_AX + 5, s)) != JT_OK) return st;
      src1 = out;
    }
    const int KA = (int)std::min<long long>(4, R);  // (also at G = 1: the self-exchange path is exercised)
    if ((st = mark(p, PM_AX + 2, s)) != JT_OK) return st;
    for (int k = 0; k < KA; ++k) {
      const long long r0 = R * k / KA, r1 = R * (k + 1) / KA;
      if (r1 == r0) continue;
      // rows [r0, r1) of the slab: input rows r0.., output rows r0.. of every chunk-major block
      if ((st = launch_axis(p, 1, false, src1 + r0 * n1 * r, p->a2a_send + r0 * c * r, r1 - r0, r, s, 1, G, -1, true,
                            R, p->total - r0 * n1 * r, p->total - r0 * c * r)) != JT_OK)
        return st;
      JT_CUDA_TRY(cudaEventRecord(p->ev_chunk[k], s));
      JT_CUDA_TRY(cudaStreamWaitEvent(p->s_comm, p->ev_chunk[k], 0));
      if (k == 0 && (st = mark(p, PM_XS, p->s_comm)) != JT_OK) return st;
      if ((st = all_to_all_rows(p, p->a2a_send, p->a2a_recv, r0, r1, c * r, p->s_comm)) != JT_OK) return st;
    }
    if ((st = mark(p, PM_AX + 3, s)) != JT_OK) return st;
    if ((st = mark(p, PM_XE, p->s_comm)) != JT_OK) return st;
    JT_CUDA_TRY(cudaEventRecord(p->ev_comm, p->s_comm));
    JT_CUDA_TRY(cudaStreamWaitEvent(s, p->ev_comm, 0));
    if ((st = mark(p, PM_AX + 0, s)) != JT_OK) return st;
    if ((st = launch_axis(p, 0, false, p->a2a_recv, out, 1, c * r, s)) != JT_OK) return st;
    return mark(p, PM_AX + 1, s);
  }
  if (d == 3) {
    if ((st = mark(p, PM_AX + 4, s)) != JT_OK) return st;
    if ((st = launch_axis(p, 2, true, in, out, n0 * c, 1, s)) != JT_OK) return st;
    if ((st = mark(p, PM_AX + 5, s)) != JT_OK) return st;
  }
  if ((st = mark(p, PM_AX + 0, s)) != JT_OK) return st;
  if ((st = launch_axis(p, 0, true, d == 3 ? out : in, p->a2a_send, 1, c * r, s, 1, G)) != JT_OK) return st;
  if ((st = mark(p, PM_AX + 1, s)) != JT_OK) return st;
  JT_CUDA_TRY(cudaEventRecord(p->ev_comm, s));
  JT_CUDA_TRY(cudaStreamWaitEvent(p->s_comm, p->ev_comm, 0));
  // the exchange in KA row chunks of the x-slab on the comm stream; chunk k's axis-1 pass waits for its rows only
  const int KA = (int)std::min<long long>(4, R);
  if ((st = mark(p, PM_XS, p->s_comm)) != JT_OK) return st;
  bool first = true;
  for (int k = 0; k < KA; ++k) {
    const long long r0 = R * k / KA, r1 = R * (k + 1) / KA;
    if (r1 == r0) continue;
    if ((st = all_to_all_rows(p, p->a2a_send, p->a2a_recv, r0, r1, c * r, p->s_comm)) != JT_OK) return st;
    JT_CUDA_TRY(cudaEventRecord(p->ev_chunk[k], p->s_comm));
    JT_CUDA_TRY(cudaStreamWaitEvent(s, p->ev_chunk[k], 0));
    if (first && (st = mark(p, PM_AX + 2, s)) != JT_OK) return st;
    first = false;
    if ((st = launch_axis(p, 1, true, p->a2a_recv + r0 * c * r, out + r0 * n1 * r, r1 - r0, r, s, G, 1, -1, true,
                          R, p->total - r0 * c * r, p->total - r0 * n1 * r)) != JT_OK)
      return st;
  }
  if ((st = mark(p, PM_XE, p->s_comm)) != JT_OK) return st;
  // the comm stream's last use of the plan's buffers is ordered before the call's end (ev_busy on s)
  JT_CUDA_TRY(cudaEventRecord(p->ev_comm, p->s_comm));
  JT_CUDA_TRY(cudaStreamWaitEvent(s, p->ev_comm, 0));
  return mark(p, PM_AX + 3, s);
}

// Axis schedule: axis d-1 (contiguous) first, reading `in`, then axes d-2..0 in place on `out`.
jt_status transform_body(const jt_plan_s *p, bool inverse, const double *in, double *out, cudaStream_t s) {
  jt_status st;
  if (p->dist) return transform_dist(p, inverse, in, out, s);
  const double *src = in;
  auto geo = [&](int axis, long long &outer, long long &inner) {
    outer = inner = 1;
    for (int i = 0; i < axis; ++i) outer *= p->n[i];
    for (int i = axis + 1; i < p->d; ++i) inner *= p->n[i];
  };
  // Fused term-split reduction (latency-bound grids, e.g. 256^2): when the axis d-1 pass and the axis d-2 pass are
  // both term-split and the second reduces in a cluster, the first leaves its S partials in the plan's workspace
  // (plain C order: its lines are rows) and the second sums them while loading its input -- one reduction phase
  // (two cluster barriers + the remote loads, ~4 us) less per call, in the same slice order as ts_reduce.
  bool fuse = false;
  if (JT_TS_FUSE && p->d >= 2) {
    long long o1, i1, o2, i2;
    geo(p->d - 1, o1, i1);
    geo(p->d - 2, o2, i2);
    p->ls.mode = 1;
    p->ls.q_S = 1;
    st = launch_axis(p, p->d - 1, inverse, src, out, o1, i1, s);
    const int S1 = p->ls.q_S;
    p->ls.q_S = 1;
    if (st == JT_OK) st = launch_axis(p, p->d - 2, inverse, out, out, o2, i2, s);
    const bool c2 = p->ls.q_S > 1 && p->ls.q_cluster;
    p->ls.mode = 0;
    if (st != JT_OK) return st;
    fuse = S1 > 1 && c2;
  }
  for (int axis = p->d - 1; axis >= 0; --axis) {
    long long outer, inner;
    geo(axis, outer, inner);
    if ((st = mark(p, PM_AX + 2 * axis, s)) != JT_OK) return st;
    if (fuse && axis == p->d - 1) p->ls.mode = 2;  // partials stay in the workspace
    if (fuse && axis == p->d - 2) {                // ... and are summed by this pass's loads
      p->ls.in_part = p->ls.ts_work;
      p->ls.in_stride = p->total;
      p->ls.in_S = p->ls.q_S;
    }
    st = launch_axis(p, axis, inverse, src, out, outer, inner, s);
    p->ls.mode = 0;
    p->ls.in_part = nullptr;
    p->ls.in_S = 0;
    if (st != JT_OK) return st;
    if ((st = mark(p, PM_AX + 2 * axis + 1, s)) != JT_OK) return st;
    src = out;
  }
  return JT_OK;
}

jt_status transform(const jt_plan_s *p, bool inverse, const double *in, double *out, cudaStream_t s) {
  jt_status st = check_device_plan(p);
  p->ls.launches = 0;
  if (st != JT_OK) return st;
  if (!in || !out) return fail(JT_ERR_ARG, "null data pointer");
  if (overlaps_partially(in, out, p->total)) return fail(JT_ERR_ARG, "input and output partially overlap");
  if (p->dist && in == out)
    return fail(JT_ERR_ARG, "distributed transforms are out of place (x-slab and y-slab differ)");
  DeviceGuard g(p->device);
  reset_marks(p);
  if ((st = begin_call(p, s)) != JT_OK) return st;
  if ((st = mark(p, PM_START, s)) != JT_OK) return st;
  if ((st = transform_body(p, inverse, in, out, s)) != JT_OK) return st;
  if ((st = mark(p, PM_END, s)) != JT_OK) return st;
  return end_call(p, s);
}

// Host-buffer transform, pipelined (DESIGN.md §10 "e2e"): the input is copied in KC row chunks of axis 0
// on a copy stream while the axis passes d-1 .. 1 run on each arrived chunk (their lines lie inside the
// chunk); the axis-0 pass then runs in KC column blocks, each copied back (a pitched 2D copy) on a second
// copy stream while the next block computes.  Every line runs the same kernel code as in jt_forward /
// jt_inverse, so the results equal the device path's up to rounding (term-split launches sum in another order).
// Wait for stream s; on a distributed plan poll the communicator meanwhile, so a failed peer surfaces as
// JT_ERR_NCCL (and aborts the communicator) instead of a hang.
jt_status wait_stream(const jt_plan_s *p, cudaStream_t s) {
  if (!p->dist || !p->comm) {
    JT_CUDA_TRY(cudaStreamSynchronize(s));
    return JT_OK;
  }
  for (;;) {
    const cudaError_t e = cudaStreamQuery(s);
    if (e == cudaSuccess) return JT_OK;
    if (e != cudaErrorNotReady) return fail(JT_ERR_CUDA, std::string("stream: ") + cudaGetErrorString(e));
    jt_status st = poll_comm(p);
    if (st != JT_OK) return st;
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

jt_status host_wait(jt_plan_s *p) {
  if (!p->s_d2h) return JT_OK;
  DeviceGuard g(p->device);
  jt_status st = wait_stream(p, p->s_h2d);
  if (st != JT_OK) return st;
  return wait_stream(p, p->s_d2h);
}

jt_status transform_host(jt_plan_s *p, bool inverse, const double *in_h, double *out_h, cudaStream_t s,
                         bool wait) {
  jt_status st = check_device_plan(p);
  p->ls.launches = 0;
  if (st != JT_OK) return st;
  if (!in_h || !out_h) return fail(JT_ERR_ARG, "null host pointer");
  DeviceGuard g(p->device);
  const size_t bytes = (size_t)p->total * sizeof(double);
  if (!p->s_h2d) {
    JT_CUDA_TRY(cudaStreamCreateWithFlags(&p->s_h2d, cudaStreamNonBlocking));
    JT_CUDA_TRY(cudaStreamCreateWithFlags(&p->s_d2h, cudaStreamNonBlocking));
    for (auto &e : p->ev) JT_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto &e : p->ev_free) JT_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  // (JT_DIST_LOWMEM: one staging slot, i.e. the two slabs of the capacity mode, and no pipelining)
  const bool lowmem = p->dist && (p->dist_flags & JT_DIST_LOWMEM);
  const int slot = lowmem ? 0 : (int)(p->host_calls++ % JT_HOST_SLOTS);
  if (!p->stage_in[slot]) {
    if (cudaMalloc((void **)&p->stage_in[slot], bytes) != cudaSuccess ||
        cudaMalloc((void **)&p->stage_out[slot], bytes) != cudaSuccess)
      return fail(JT_ERR_ALLOC, "staging cudaMalloc");
    JT_CUDA_TRY(cudaEventRecord(p->ev_free[slot], p->s_d2h));
  }
  double *sin = p->stage_in[slot], *sout = p->stage_out[slot];
  cudaEvent_t *ev_in = p->ev, *ev_out = p->ev + 16, ev_start = p->ev[32];
  // ordering: the caller's prior work on s first; the slot's previous use (its output copy) finished; the
  // previous call's use of the plan's other buffers (all-to-all, term-split workspace) finished
  reset_marks(p);
  if ((st = begin_call(p, s)) != JT_OK) return st;
  JT_CUDA_TRY(cudaEventRecord(ev_start, s));
  JT_CUDA_TRY(cudaStreamWaitEvent(p->s_h2d, p->ev_free[slot], 0));
  JT_CUDA_TRY(cudaStreamWaitEvent(s, p->ev_free[slot], 0));
  JT_CUDA_TRY(cudaStreamWaitEvent(p->s_d2h, ev_start, 0));
  const int d = p->d;
  if (p->dist && !inverse && !lowmem) {
    // distributed forward (transform_dist's schedule, pipelined with the copies): the x-slab arrives in KA row
    // chunks; each chunk's axes d-1..1 and its rows of the all-to-all run as soon as it is in; the axis-0 pass on
    // the received y-slab runs in column blocks, each copied back (pitched) while the next computes
    const int G = p->nranks;
    const long long n0 = p->n[0], n1 = p->n[1], r = d == 3 ? p->n[2] : 1;
    const long long R = n0 / G, c = n1 / G, xrow = n1 * r, yrow = c * r;
    if ((st = ensure_comm_stream(p)) != JT_OK) return st;
    const int KA = (int)std::min<long long>(4, R);
    if (p->p2p && (st = dist_barrier(p, s)) != JT_OK) return st;  // (fused exchange: peers done with their buffers)
    for (int k = 0; k < KA; ++k) {
      const long long r0 = R * k / KA, r1 = R * (k + 1) / KA;
      if (r1 == r0) continue;
      const size_t off = (size_t)(r0 * xrow), cnt = (size_t)((r1 - r0) * xrow);
      JT_CUDA_TRY(cudaMemcpyAsync(sin + off, in_h + off, cnt * sizeof(double), cudaMemcpyHostToDevice, p->s_h2d));
      JT_CUDA_TRY(cudaEventRecord(ev_in[k], p->s_h2d));
      JT_CUDA_TRY(cudaStreamWaitEvent(s, ev_in[k], 0));
      const double *src1 = sin + off;
      if (d == 3) {
        if ((st = launch_axis(p, 2, false, sin + off, sout + off, (r1 - r0) * n1, 1, s, 1, 1, -1, true, -1,
                              p->total - (long long)off, p->total - (long long)off)) != JT_OK)
          return st;
        src1 = sout + off;
      }
      if (p->p2p) {  // this chunk's rows of every block straight into their owners' receive buffers
        if ((st = resolve_peers(p, s)) != JT_OK) return st;
        if ((st = launch_axis(p, 1, false, src1, p->a2a_recv, r1 - r0, r, s, 1, G, -1, true, R,
                              p->total - (long long)off, -1, true, r0 * c * r)) != JT_OK)
          return st;
        continue;
      }
      if ((st = launch_axis(p, 1, false, src1, p->a2a_send + r0 * c * r, r1 - r0, r, s, 1, G, -1, true, R,
                            p->total - (long long)off, p->total - r0 * c * r)) != JT_OK)
        return st;
      JT_CUDA_TRY(cudaEventRecord(p->ev_chunk[k], s));
      JT_CUDA_TRY(cudaStreamWaitEvent(p->s_comm, p->ev_chunk[k], 0));
      if ((st = all_to_all_rows(p, p->a2a_send, p->a2a_recv, r0, r1, c * r, p->s_comm)) != JT_OK) return st;
    }
    if (p->p2p) {
      if ((st = dist_barrier(p, s)) != JT_OK) return st;  // every rank's rows have landed here
    } else {
      JT_CUDA_TRY(cudaEventRecord(p->ev_comm, p->s_comm));
      JT_CUDA_TRY(cudaStreamWaitEvent(s, p->ev_comm, 0));
    }
    const int KC = (int)std::min<long long>(8, yrow);
    for (int cb = 0; cb < KC; ++cb) {
      const long long c0 = yrow * cb / KC, c1 = yrow * (cb + 1) / KC;
      if (c1 == c0) continue;
      if ((st = launch_axis(p, 0, false, p->a2a_recv + c0, sout + c0, 1, yrow, s, 1, 1, c1 - c0, true, -1,
                            p->total - c0, p->total - c0)) != JT_OK)
        return st;
      JT_CUDA_TRY(cudaEventRecord(ev_out[cb], s));
      JT_CUDA_TRY(cudaStreamWaitEvent(p->s_d2h, ev_out[cb], 0));
      JT_CUDA_TRY(cudaMemcpy2DAsync(out_h + c0, (size_t)yrow * sizeof(double), sout + c0, (size_t)yrow * sizeof(double),
                                    (size_t)(c1 - c0) * sizeof(double), (size_t)n0, cudaMemcpyDeviceToHost,
                                    p->s_d2h));
    }
  } else if (p->dist && inverse && !lowmem) {
    // distributed inverse (transform_dist's inverse schedule, pipelined with the copies): the y-slab arrives in KC
    // row chunks of axis 0, each chunk's axis-2 lines (d = 3) transformed as it lands; the axis-0 pass (its lines span
    // every row) writes the chunk-major send blocks; the exchange runs in KA row chunks of the x-slab on the comm
    // stream, each chunk's axis-1 pass starts as its rows arrive and its x-slab rows are copied back at once
    const int G = p->nranks;
    const long long n0 = p->n[0], n1 = p->n[1], r = d == 3 ? p->n[2] : 1;
    const long long R = n0 / G, c = n1 / G, yrow = c * r, xrow = n1 * r;
    if ((st = ensure_comm_stream(p)) != JT_OK) return st;
    if (p->p2p && (st = dist_barrier(p, s)) != JT_OK) return st;  // (fused exchange: peers done with their buffers)
    const int KC = (int)std::min<long long>(8, n0);
    for (int k = 0; k < KC; ++k) {
      const long long q0 = n0 * k / KC, q1 = n0 * (k + 1) / KC;
      if (q1 == q0) continue;
      const size_t off = (size_t)(q0 * yrow), cnt = (size_t)((q1 - q0) * yrow);
      JT_CUDA_TRY(cudaMemcpyAsync(sin + off, in_h + off, cnt * sizeof(double), cudaMemcpyHostToDevice, p->s_h2d));
      JT_CUDA_TRY(cudaEventRecord(ev_in[k], p->s_h2d));
      JT_CUDA_TRY(cudaStreamWaitEvent(s, ev_in[k], 0));
      if (d == 3 && (st = launch_axis(p, 2, true, sin + off, sout + off, (q1 - q0) * c, 1, s, 1, 1, -1, true, -1,
                                      p->total - (long long)off, p->total - (long long)off)) != JT_OK)
        return st;
    }
    if (p->p2p) {  // the axis-0 pass stores every block straight into its owner's receive buffer
      if ((st = resolve_peers(p, s)) != JT_OK) return st;
      if ((st = launch_axis(p, 0, true, d == 3 ? sout : sin, p->a2a_recv, 1, yrow, s, 1, G, -1, true, -1, -1, -1,
                            true, 0)) != JT_OK)
        return st;
      if ((st = dist_barrier(p, s)) != JT_OK) return st;  // every rank's blocks have landed here
    } else {
      if ((st = launch_axis(p, 0, true, d == 3 ? sout : sin, p->a2a_send, 1, yrow, s, 1, G)) != JT_OK) return st;
      JT_CUDA_TRY(cudaEventRecord(p->ev_comm, s));
      JT_CUDA_TRY(cudaStreamWaitEvent(p->s_comm, p->ev_comm, 0));
    }
    const int KA = (int)std::min<long long>(4, R);
    for (int k = 0; k < KA; ++k) {
      const long long r0 = R * k / KA, r1 = R * (k + 1) / KA;
      if (r1 == r0) continue;
      if (!p->p2p) {
        if ((st = all_to_all_rows(p, p->a2a_send, p->a2a_recv, r0, r1, yrow, p->s_comm)) != JT_OK) return st;
        JT_CUDA_TRY(cudaEventRecord(p->ev_chunk[k], p->s_comm));
        JT_CUDA_TRY(cudaStreamWaitEvent(s, p->ev_chunk[k], 0));
      }
      if ((st = launch_axis(p, 1, true, p->a2a_recv + r0 * yrow, sout + r0 * xrow, r1 - r0, r, s, G, 1, -1, true, R,
                            p->total - r0 * yrow, p->total - r0 * xrow)) != JT_OK)
        return st;
      JT_CUDA_TRY(cudaEventRecord(ev_out[k], s));
      JT_CUDA_TRY(cudaStreamWaitEvent(p->s_d2h, ev_out[k], 0));
      JT_CUDA_TRY(cudaMemcpyAsync(out_h + r0 * xrow, sout + r0 * xrow, (size_t)((r1 - r0) * xrow) * sizeof(double),
                                  cudaMemcpyDeviceToHost, p->s_d2h));
    }
  } else if (p->dist || d == 1) {  // capacity-mode distributed plans / one line: copy in, transform, copy out
    JT_CUDA_TRY(cudaMemcpyAsync(sin, in_h, bytes, cudaMemcpyHostToDevice, p->s_h2d));
    JT_CUDA_TRY(cudaEventRecord(ev_in[0], p->s_h2d));
    JT_CUDA_TRY(cudaStreamWaitEvent(s, ev_in[0], 0));
    if ((st = transform_body(p, inverse, sin, sout, s)) != JT_OK) return st;
    JT_CUDA_TRY(cudaEventRecord(ev_out[0], s));
    JT_CUDA_TRY(cudaStreamWaitEvent(p->s_d2h, ev_out[0], 0));
    JT_CUDA_TRY(cudaMemcpyAsync(out_h, sout, bytes, cudaMemcpyDeviceToHost, p->s_d2h));
  } else if (JT_HOST_SCHED == 1 || (JT_HOST_SCHED == 2 && d == 2)) {
    // axis 0 first: the input arrives in KC row chunks; the axis-0 pass (every line spans all rows) runs once all are
    // in; then axes d-1..1 run in place on row chunks, each copied back as one contiguous block
    const long long n0 = p->n[0];
    const long long row = p->total / n0;
    const int KC = (int)std::min<long long>(8, n0);
    for (int c = 0; c < KC; ++c) {
      const long long r0 = n0 * c / KC, r1 = n0 * (c + 1) / KC;
      const size_t off = (size_t)(r0 * row), cnt = (size_t)((r1 - r0) * row);
      JT_CUDA_TRY(cudaMemcpyAsync(sin + off, in_h + off, cnt * sizeof(double), cudaMemcpyHostToDevice, p->s_h2d));
    }
    JT_CUDA_TRY(cudaEventRecord(ev_in[0], p->s_h2d));
    JT_CUDA_TRY(cudaStreamWaitEvent(s, ev_in[0], 0));
    if ((st = launch_axis(p, 0, inverse, sin, sout, 1, row, s)) != JT_OK) return st;
    for (int c = 0; c < KC; ++c) {
      const long long r0 = n0 * c / KC, r1 = n0 * (c + 1) / KC;
      const size_t off = (size_t)(r0 * row), cnt = (size_t)((r1 - r0) * row);
      for (int axis = d - 1; axis >= 1; --axis) {
        long long outer = r1 - r0, inner = 1;
        for (int i = 1; i < axis; ++i) outer *= p->n[i];
        for (int i = axis + 1; i < d; ++i) inner *= p->n[i];
        if ((st = launch_axis(p, axis, inverse, sout + off, sout + off, outer, inner, s, 1, 1, -1, true, -1,
                              p->total - (long long)off, p->total - (long long)off)) != JT_OK)
          return st;
      }
      JT_CUDA_TRY(cudaEventRecord(ev_out[c], s));
      JT_CUDA_TRY(cudaStreamWaitEvent(p->s_d2h, ev_out[c], 0));
      JT_CUDA_TRY(cudaMemcpyAsync(out_h + off, sout + off, cnt * sizeof(double), cudaMemcpyDeviceToHost, p->s_d2h));
    }
  } else {
    const long long n0 = p->n[0];
    const long long row = p->total / n0;  // elements per axis-0 index (the axis-0 pass's line count)
    const int KC = (int)std::min<long long>(8, n0);
    // phase 1: row chunks of axis 0 arrive on the copy stream; axes d-1..1 run on each arrived chunk
    for (int c = 0; c < KC; ++c) {
      const long long r0 = n0 * c / KC, r1 = n0 * (c + 1) / KC;
      const size_t off = (size_t)(r0 * row), cnt = (size_t)((r1 - r0) * row);
      JT_CUDA_TRY(cudaMemcpyAsync(sin + off, in_h + off, cnt * sizeof(double), cudaMemcpyHostToDevice, p->s_h2d));
      JT_CUDA_TRY(cudaEventRecord(ev_in[c], p->s_h2d));
      JT_CUDA_TRY(cudaStreamWaitEvent(s, ev_in[c], 0));
      const double *src = sin + off;
      for (int axis = d - 1; axis >= 1; --axis) {
        long long outer = r1 - r0, inner = 1;
        for (int i = 1; i < axis; ++i) outer *= p->n[i];
        for (int i = axis + 1; i < d; ++i) inner *= p->n[i];
        if ((st = launch_axis(p, axis, inverse, src, sout + off, outer, inner, s, 1, 1, -1, true, -1,
                              p->total - (long long)off, p->total - (long long)off)) != JT_OK)
          return st;
        src = sout + off;
      }
    }
    // phase 2: axis-0 pass in column blocks, each copied back (pitched) while the next computes
    for (int c = 0; c < KC; ++c) {
      const long long c0 = row * c / KC, c1 = row * (c + 1) / KC;
      if (c1 == c0) continue;
      if ((st = launch_axis(p, 0, inverse, sout + c0, sout + c0, 1, row, s, 1, 1, c1 - c0, true, -1, p->total - c0,
                            p->total - c0)) != JT_OK)
        return st;
      JT_CUDA_TRY(cudaEventRecord(ev_out[c], s));
      JT_CUDA_TRY(cudaStreamWaitEvent(p->s_d2h, ev_out[c], 0));
      JT_CUDA_TRY(cudaMemcpy2DAsync(out_h + c0, (size_t)row * sizeof(double), sout + c0, (size_t)row * sizeof(double),
                                    (size_t)(c1 - c0) * sizeof(double), (size_t)n0, cudaMemcpyDeviceToHost,
                                    p->s_d2h));
    }
  }
  JT_CUDA_TRY(cudaEventRecord(p->ev_free[slot], p->s_d2h));
  if ((st = end_call(p, s)) != JT_OK) return st;
  return wait ? host_wait(p) : JT_OK;
}

}  // namespace

extern "C" {

const char *jt_last_error(void) { return g_last_error.c_str(); }

const char *jt_version(void) { return "jt 0.1 (sm_100a fused fp64 axis passes)"; }

jt_status jt_last_launches(jt_plan_t p, int *count) {
  if (!p || !count) return fail(JT_ERR_ARG, "null argument");
  *count = p->ls.launches;
  return JT_OK;
}

jt_status jt_default_opts(jt_opts *o) {
  if (!o) return fail(JT_ERR_ARG, "null opts");
  o->seed = 0;
  o->k0 = -1;  // auto: 27 (the paper's) or 32 where that lowers the rank (R24)
  o->rmax_init = 0;
  o->q = 3;
  o->sweeps = 2;
  o->device = -1;
  return JT_OK;
}

jt_status jt_plan(jt_plan_t *out, int d, const int64_t n[], const double a[], const double b[], double eps,
                  const jt_opts *opts) {
  return jt_plan_ex(out, d, n, a, b, nullptr, JT_KIND_P, eps, opts);
}

jt_status jt_plan_ex(jt_plan_t *out, int d, const int64_t n[], const double a[], const double b[],
                     const double *const points[], int kind, double eps, const jt_opts *opts) {
  if (!out) return fail(JT_ERR_ARG, "null out");
  if (kind != JT_KIND_P && kind != JT_KIND_Q) return fail(JT_ERR_ARG, "kind must be JT_KIND_P or JT_KIND_Q");
  *out = nullptr;
  if (d < 1 || d > 3) return fail(JT_ERR_ARG, "d must be 1, 2 or 3");
  if (!n || !a || !b) return fail(JT_ERR_ARG, "null n/a/b");
  if (!(eps >= 1e-15 && eps <= 1e-2)) return fail(JT_ERR_ARG, "eps must be in [1e-15, 1e-2]");
  jt_opts o;
  jt_default_opts(&o);
  if (opts) o = *opts;
  if (o.k0 < -1 || o.k0 > jtk::K0MAX) return fail(JT_ERR_ARG, "k0 must be -1 (auto) or in [0, 32]");
  for (int i = 0; i < d; ++i) {
    if (n[i] < 2 || n[i] > 4096) return fail(JT_ERR_ARG, "n[i] must be in [2, 4096]");
    if (!(a[i] > -1 && a[i] < 1 && b[i] > -1 && b[i] < 1))
      return fail(JT_ERR_DOMAIN, "a, b must lie in (-1, 1) (PAPER.md:1000: not applicable outside)");
  }
  jt_plan_s *p = new (std::nothrow) jt_plan_s();
  if (!p) return fail(JT_ERR_ALLOC, "plan allocation");
  p->d = d;
  p->eps = eps;
  p->opts = o;
  p->total = 1;
  for (int i = 0; i < d; ++i) {
    p->n[i] = n[i];
    p->a[i] = a[i];
    p->b[i] = b[i];
    p->total *= n[i];
  }
  try {
    for (int i = 0; i < d; ++i) {
      // identical axes share the host computation
      const double *pts = points ? points[i] : nullptr;
      int same = -1;
      for (int k = 0; k < i; ++k) {
        const double *pk = points ? points[k] : nullptr;
        const bool same_pts = (pk == nullptr && pts == nullptr) ||
                              (pk && pts && n[k] == n[i] && std::memcmp(pk, pts, n[i] * sizeof(double)) == 0);
        if (n[k] == n[i] && a[k] == a[i] && b[k] == b[i] && same_pts) same = k;
      }
      if (same >= 0) {
        p->host[i] = p->host[same];
        continue;
      }
      std::string err;
      jt_opts oa = o;
      if (o.k0 == -1) oa.k0 = 27;
      jt_status s = jt::build_axis_host(p->host[i], n[i], a[i], b[i], eps, oa, err, pts, kind);
      if (s == JT_OK && o.k0 == -1 && p->host[i].N <= 512 && n[i] > 32) {
        // auto k0 (reading R24): the kernels stage 2 degrees of W V per rank term for N <= 512, so a
        // 32-degree block is free of extra passes; keep it if it saves a rank term
        jt::AxisHost alt;
        std::string err2;
        oa.k0 = 32;
        if (jt::build_axis_host(alt, n[i], a[i], b[i], eps, oa, err2, pts, kind) == JT_OK && alt.r < p->host[i].r)
          p->host[i] = std::move(alt);
      } else if (s == JT_OK && o.k0 == -1 && p->host[i].N >= 2048) {
        // auto k0 (reading R24): for N >= 2048 the batch-start W V loop streams k0 x n doubles per line through L1 (a
        // degree costs ~1/14 of a rank term, r02zt); a narrower block that keeps the rank is strictly cheaper
        // (4096^2: k0 27 -> 20, forward -2.1 %, inverse -2.4 %; 2048^2: 27 -> 24, -1.2 %)
        jt::AxisHost alt;
        std::string err2;
        oa.k0 = p->host[i].N >= 4096 ? 20 : 24;
        if (jt::build_axis_host(alt, n[i], a[i], b[i], eps, oa, err2, pts, kind) == JT_OK && alt.r <= p->host[i].r)
          p->host[i] = std::move(alt);
      }
      if (s != JT_OK) {
        delete p;
        return fail(s, "axis " + std::to_string(i) + ": " + err);
      }
    }
    // Paired real rank terms for the forward passes: uniform axes whose FFT length has Cfg::PAIR
    // kernels; the same k0; kept when it needs fewer FFTs than the complex factorisation (JT_PAIR=0 in the
    // environment turns it off: A/B runs and tests of the unpaired forward kernels)
    const char *pe = std::getenv("JT_PAIR");
    const bool pair_on = JT_PAIR && !(pe && pe[0] == '0');
    for (int i = 0; i < d && pair_on; ++i) {
      const jt::AxisHost &h = p->host[i];
      if (!h.uniform || !jtl::pair_length(h.N) || h.r < 2) continue;
      int same = -1;
      for (int k = 0; k < i; ++k)
        if (p->pair[k] && n[k] == n[i] && a[k] == a[i] && b[k] == b[i] && p->host[k].k0 == h.k0 &&
            p->host[k].kind == h.kind)
          same = k;
      if (same >= 0) {
        p->hostp[i] = p->hostp[same];
        p->pair[i] = true;
        continue;
      }
      std::string err;
      jt_opts oa = o;
      oa.k0 = h.k0;
      if (jt::build_axis_host(p->hostp[i], n[i], a[i], b[i], eps, oa, err, nullptr, h.kind, true) == JT_OK &&
          p->hostp[i].r < h.r)
        p->pair[i] = true;
      else
        p->hostp[i] = jt::AxisHost();
    }
  } catch (const std::bad_alloc &) {
    delete p;
    return fail(JT_ERR_ALLOC, "host allocation during plan");
  } catch (const std::exception &ex) {
    delete p;
    return fail(JT_ERR_NUMERIC, std::string("plan: ") + ex.what());
  }
  if (o.device != -2) {
    int dev = o.device;
    if (dev == -1 && cudaGetDevice(&dev) != cudaSuccess) {
      delete p;
      return fail(JT_ERR_CUDA, "no CUDA device");
    }
    p->device = dev;
    DeviceGuard g(dev);
    for (int i = 0; i < d; ++i) {
      jt_status s = upload_axis(p, i);
      if (s == JT_OK && p->pair[i]) s = upload_axis(p, i, true);
      if (s != JT_OK) {
        std::string msg = g_last_error;
        free_device(p);
        delete p;
        return fail(s, msg);
      }
    }
  }
  *out = p;
  return JT_OK;
}

jt_status jt_forward(jt_plan_t p, const double *coeffs, double *values, void *stream) {
  return transform(p, false, coeffs, values, (cudaStream_t)stream);
}

static jt_status check_orthogonal(jt_plan_t p) {
  if (!p) return fail(JT_ERR_ARG, "null plan");
  for (int i = 0; i < p->d; ++i)
    if (!p->host[i].uniform || p->host[i].kind != JT_KIND_P)
      return fail(JT_ERR_ARG, "jt_inverse needs a uniform first-kind plan (the nonuniform / second-kind matrix is not "
                              "orthogonal, PAPER.md:509; jt_adjoint applies its transpose)");
  return JT_OK;
}

jt_status jt_inverse(jt_plan_t p, const double *values, double *coeffs, void *stream) {
  jt_status st = check_orthogonal(p);
  if (st != JT_OK) return st;
  return transform(p, true, values, coeffs, (cudaStream_t)stream);
}

jt_status jt_adjoint(jt_plan_t p, const double *values, double *coeffs, void *stream) {
  return transform(p, true, values, coeffs, (cudaStream_t)stream);
}

jt_status jt_plan_kind(jt_plan_t p, int axis, int *uniform, int *kind) {
  if (!p || axis < 0 || axis >= p->d) return fail(JT_ERR_ARG, "bad args");
  if (uniform) *uniform = p->host[axis].uniform ? 1 : 0;
  if (kind) *kind = p->host[axis].kind;
  return JT_OK;
}

jt_status jt_forward_host(jt_plan_t p, const double *coeffs_host, double *values_host, void *stream) {
  return transform_host(p, false, coeffs_host, values_host, (cudaStream_t)stream, true);
}

jt_status jt_forward_host_async(jt_plan_t p, const double *coeffs_host, double *values_host, void *stream) {
  return transform_host(p, false, coeffs_host, values_host, (cudaStream_t)stream, false);
}

jt_status jt_inverse_host_async(jt_plan_t p, const double *values_host, double *coeffs_host, void *stream) {
  jt_status st = check_orthogonal(p);
  if (st != JT_OK) return st;
  return transform_host(p, true, values_host, coeffs_host, (cudaStream_t)stream, false);
}

jt_status jt_host_wait(jt_plan_t p) {
  if (!p) return fail(JT_ERR_ARG, "null plan");
  return host_wait(p);
}

jt_status jt_inverse_host(jt_plan_t p, const double *values_host, double *coeffs_host, void *stream) {
  jt_status st = check_orthogonal(p);
  if (st != JT_OK) return st;
  return transform_host(p, true, values_host, coeffs_host, (cudaStream_t)stream, true);
}

static jt_status axis_entry(jt_plan_t p, int axis, bool inverse, const double *in, double *out, int64_t outer,
                            int64_t inner, int in_split, int out_split, void *stream, int64_t ostride = -1) {
  jt_status st = check_device_plan(p);
  if (p) p->ls.launches = 0;
  if (st != JT_OK) return st;
  if (axis < 0 || axis >= p->d) return fail(JT_ERR_ARG, "bad axis");
  if (!in || !out || outer < 0 || inner < 1) return fail(JT_ERR_ARG, "bad pointers / shape");
  if (in_split < 1 || out_split < 1 || p->n[axis] % in_split != 0 || p->n[axis] % out_split != 0)
    return fail(JT_ERR_ARG, "in_split / out_split must be >= 1 and divide n[axis]");
  const int64_t count = outer * inner * p->n[axis];
  if (overlaps_partially(in, out, count)) return fail(JT_ERR_ARG, "partial overlap");
  if (in == out && (in_split != 1 || out_split != 1))
    return fail(JT_ERR_ARG, "chunk-major layouts need out-of-place buffers");
  DeviceGuard g(p->device);
  if (ostride >= 0 && ostride < outer) return fail(JT_ERR_ARG, "ostride must be >= outer");
  const cudaStream_t s = (cudaStream_t)stream;
  if ((st = begin_call(p, s)) != JT_OK) return st;
  if ((st = launch_axis(p, axis, inverse, in, out, outer, inner, s, in_split, out_split, -1, true, ostride)) != JT_OK)
    return st;
  return end_call(p, s);
}

jt_status jt_forward_axis(jt_plan_t p, int axis, const double *in, double *out, int64_t outer, int64_t inner,
                          void *stream) {
  return axis_entry(p, axis, false, in, out, outer, inner, 1, 1, stream);
}

jt_status jt_inverse_axis(jt_plan_t p, int axis, const double *in, double *out, int64_t outer, int64_t inner,
                          void *stream) {
  return axis_entry(p, axis, true, in, out, outer, inner, 1, 1, stream);
}

jt_status jt_axis_pass(jt_plan_t p, int axis, int inverse, const double *in, double *out, int64_t outer,
                       int64_t inner, int in_split, int out_split, void *stream) {
  return axis_entry(p, axis, inverse != 0, in, out, outer, inner, in_split, out_split, stream);
}

jt_status jt_axis_pass_ex(jt_plan_t p, int axis, int inverse, const double *in, double *out, int64_t outer,
                          int64_t inner, int in_split, int out_split, int64_t ostride, void *stream) {
  return axis_entry(p, axis, inverse != 0, in, out, outer, inner, in_split, out_split, stream, ostride);
}

jt_status jt_dist_unique_id(void *nccl_unique_id) {
  if (!nccl_unique_id) return fail(JT_ERR_ARG, "null id");
  nccl::Api &A = nccl::api();
  if (!A.ok) return fail(JT_ERR_NCCL, A.why);
  nccl::UniqueId id;
  const int e = A.GetUniqueId(&id);
  if (e != nccl::Success) return fail(JT_ERR_NCCL, std::string("ncclGetUniqueId: ") + A.GetErrorString(e));
  std::memcpy(nccl_unique_id, &id, sizeof(id));
  return JT_OK;
}

// Fused-exchange setup (collective over the plan's communicator): every rank's receive buffer is exported as a CUDA
// IPC handle, the handles all-gathered, the peers' buffers opened (peer access over NVLink / NVSwitch); an all-reduce
// (min) of the outcome makes every rank use the fused exchange, or every rank fall back to the NCCL all-to-all.
static bool setup_ipc(jt_plan_s *p) {
  nccl::Api &A = nccl::api();
  const int G = p->nranks, me = p->rank;
  const size_t H = sizeof(cudaIpcMemHandle_t);
  int ok = 1;
  cudaIpcMemHandle_t mine;
  std::memset(&mine, 0, H);
  if (cudaIpcGetMemHandle(&mine, p->a2a_recv) != cudaSuccess) ok = 0;
  char *dbuf = nullptr;
  int *dflag = nullptr;
  cudaStream_t st = nullptr;
  if (cudaMalloc((void **)&dbuf, G * H) != cudaSuccess || cudaMalloc((void **)&dflag, sizeof(int)) != cudaSuccess ||
      cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
    ok = 0;  // (still takes part in the collectives below with whatever it has)
  }
  std::vector<cudaIpcMemHandle_t> all(G);
  if (dbuf && dflag && st) {
    cudaMemcpy(dbuf + me * H, &mine, H, cudaMemcpyHostToDevice);
    if (A.AllGather(dbuf + me * H, dbuf, H, nccl::Uint8, p->comm, st) != nccl::Success) ok = 0;
    cudaMemcpyAsync(all.data(), dbuf, G * H, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    for (int g = 0; g < G && ok; ++g) {
      if (g == me) continue;
      void *ptr = nullptr;
      if (cudaIpcOpenMemHandle(&ptr, all[g], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        ok = 0;
        cudaGetLastError();
      } else {
        p->peer_recv[g] = static_cast<double *>(ptr);
        p->peer_ipc[g] = true;
      }
    }
    p->peer_recv[me] = p->a2a_recv;
    cudaMemcpy(dflag, &ok, sizeof(int), cudaMemcpyHostToDevice);
    if (A.AllReduce(dflag, dflag, 1, nccl::Int32, nccl::Min, p->comm, st) != nccl::Success) ok = 0;
    int agreed = 0;
    cudaMemcpyAsync(&agreed, dflag, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    ok = ok && agreed;
  }
  if (!ok) {
    for (int g = 0; g < G; ++g)
      if (p->peer_ipc[g]) cudaIpcCloseMemHandle(p->peer_recv[g]), p->peer_ipc[g] = false;
    for (auto &q : p->peer_recv) q = nullptr;
  }
  cudaFree(dbuf);
  cudaFree(dflag);
  if (st) cudaStreamDestroy(st);
  cudaGetLastError();
  return ok != 0;
}

// Shared by jt_plan_dist_ex (NCCL communicator) and jt_debug_plan_virtual (in-process group).
static jt_status plan_dist_common(jt_plan_t *out, int d, const int64_t n[], const double a[], const double b[],
                                  double eps, const jt_opts *opts, int rank, int nranks, int flags,
                                  const void *nccl_unique_id, jt_vgroup_t group) {
  if (!out) return fail(JT_ERR_ARG, "null out");
  *out = nullptr;
  if (d != 2 && d != 3) return fail(JT_ERR_ARG, "distributed plans need d = 2 or 3");
  if ((!nccl_unique_id && !group) || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(JT_ERR_ARG, "bad rank / nranks / id");
  if (flags & ~(JT_DIST_LOWMEM | JT_DIST_NCCL_A2A)) return fail(JT_ERR_ARG, "unknown JT_DIST_* flag");
  if (nranks > jtk::MAX_SPLIT) return fail(JT_ERR_ARG, "at most 32 ranks");
  if (!n || n[0] % nranks != 0 || n[1] % nranks != 0)
    return fail(JT_ERR_ARG, "n[0] and n[1] must be divisible by nranks");
  if (opts && opts->device == -2) return fail(JT_ERR_ARG, "distributed plans need a device");
  nccl::Api &A = nccl::api();
  if (!group && !A.ok) return fail(JT_ERR_NCCL, A.why);
  jt_plan_t p = nullptr;
  jt_status st = jt_plan(&p, d, n, a, b, eps, opts);
  if (st != JT_OK) return st;
  p->dist = true;
  p->rank = rank;
  p->nranks = nranks;
  p->dist_flags = flags;
  p->total /= nranks;  // local slab elements
  DeviceGuard g(p->device);
  if (group) {
    std::lock_guard<std::mutex> lk(group->mu);
    if (group->member[rank]) {
      jt_destroy(p);
      return fail(JT_ERR_ARG, "virtual group: rank already has a plan");
    }
    if (cudaEventCreateWithFlags(&group->ev_ready[rank], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&group->ev_done[rank], cudaEventDisableTiming) != cudaSuccess) {
      jt_destroy(p);
      return fail(JT_ERR_CUDA, "virtual group events");
    }
    group->member[rank] = p;
    p->vgroup = group;
  } else {
    nccl::UniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof(id));
    const int e = A.CommInitRank(&p->comm, nranks, id, rank);
    if (e != nccl::Success) {
      std::string msg = std::string("ncclCommInitRank: ") + A.GetErrorString(e);
      p->comm = nullptr;
      jt_destroy(p);
      return fail(JT_ERR_NCCL, msg);
    }
  }
  if (!(flags & JT_DIST_LOWMEM)) {
    const size_t bytes = (size_t)p->total * sizeof(double);
    if (cudaMalloc((void **)&p->a2a_recv, bytes) != cudaSuccess ||
        (!group && cudaMalloc((void **)&p->bar_buf, sizeof(double)) != cudaSuccess)) {
      jt_destroy(p);
      return fail(JT_ERR_ALLOC, "all-to-all buffers");
    }
    if (!group) cudaMemset(p->bar_buf, 0, sizeof(double));
    // the fused exchange unless the caller asks for the NCCL all-to-all: peer pointers to every rank's receive
    // buffer (all ranks agree on the outcome: setup_ipc is collective and falls back for everyone)
    if (!(flags & JT_DIST_NCCL_A2A)) p->p2p = group ? true : setup_ipc(p);
    if (!p->p2p && cudaMalloc((void **)&p->a2a_send, bytes) != cudaSuccess) {
      jt_destroy(p);
      return fail(JT_ERR_ALLOC, "all-to-all buffers");
    }
  }
  *out = p;
  return JT_OK;
}

jt_status jt_plan_dist(jt_plan_t *out, int d, const int64_t n[], const double a[], const double b[], double eps,
                       const jt_opts *opts, const void *nccl_unique_id, int rank, int nranks) {
  return plan_dist_common(out, d, n, a, b, eps, opts, rank, nranks, 0, nccl_unique_id, nullptr);
}

jt_status jt_plan_dist_ex(jt_plan_t *out, int d, const int64_t n[], const double a[], const double b[], double eps,
                          const jt_opts *opts, const void *nccl_unique_id, int rank, int nranks, int flags) {
  if (!nccl_unique_id) return fail(JT_ERR_ARG, "null id");
  return plan_dist_common(out, d, n, a, b, eps, opts, rank, nranks, flags, nccl_unique_id, nullptr);
}

jt_status jt_dist_mode(jt_plan_t p, int *mode) {
  if (!p || !mode) return fail(JT_ERR_ARG, "null argument");
  *mode = !p->dist ? JT_MODE_SINGLE
                   : (p->dist_flags & JT_DIST_LOWMEM) ? JT_MODE_LOWMEM : (p->p2p ? JT_MODE_FUSED : JT_MODE_A2A);
  return JT_OK;
}

jt_status jt_sync(jt_plan_t p, void *cuda_stream) {
  if (!p) return fail(JT_ERR_ARG, "null plan");
  if (p->device < 0) return fail(JT_ERR_ARG, "host-only plan");
  DeviceGuard g(p->device);
  jt_status st = p->dist ? poll_comm(p) : JT_OK;
  if (st != JT_OK) return st;
  return wait_stream(p, (cudaStream_t)cuda_stream);
}

jt_status jt_profile(jt_plan_t p, int enable) {
  if (!p) return fail(JT_ERR_ARG, "null plan");
  p->prof_on = enable != 0;
  reset_marks(p);
  return JT_OK;
}

jt_status jt_last_profile(jt_plan_t p, double ms[5]) {
  if (!p || !ms) return fail(JT_ERR_ARG, "null argument");
  if (!p->prof_on || !p->prec[PM_START] || !p->prec[PM_END])
    return fail(JT_ERR_ARG, "no profiled call (jt_profile(p, 1) before a jt_forward / jt_inverse)");
  DeviceGuard g(p->device);
  auto span = [&](int a, int b) -> double {
    if (!p->prec[a] || !p->prec[b]) return 0.0;
    float t = 0;
    if (cudaEventSynchronize(p->pev[b]) != cudaSuccess || cudaEventElapsedTime(&t, p->pev[a], p->pev[b]) != cudaSuccess)
      return -1.0;
    return (double)t;
  };
  for (int i = 0; i < 3; ++i) ms[i] = span(PM_AX + 2 * i, PM_AX + 2 * i + 1);
  ms[3] = span(PM_XS, PM_XE);
  ms[4] = span(PM_START, PM_END);
  for (int i = 0; i < 5; ++i)
    if (ms[i] < 0) return fail(JT_ERR_CUDA, "profile events");
  return JT_OK;
}

// ---- test hooks (include/jt_debug.h) ----
jt_status jt_debug_axis_pass_lim(jt_plan_t p, int axis, int inverse, const double *in, double *out, int64_t outer,
                                 int64_t inner, int64_t in_lim, int64_t out_lim, void *stream) {
  jt_status st = check_device_plan(p);
  if (st != JT_OK) return st;
  if (axis < 0 || axis >= p->d || !in || !out || outer < 1 || inner < 1 || in_lim < 0 || out_lim < 0)
    return fail(JT_ERR_ARG, "bad args");
  p->ls.launches = 0;
  DeviceGuard g(p->device);
  const cudaStream_t s = (cudaStream_t)stream;
  if ((st = begin_call(p, s)) != JT_OK) return st;
  // (no term split: the reduction kernel writes the output without the kernels' checks)
  if ((st = launch_axis(p, axis, inverse != 0, in, out, outer, inner, s, 1, 1, -1, false, -1, in_lim, out_lim)) != JT_OK)
    return st;
  return end_call(p, s);
}

jt_status jt_debug_checks(int *enabled, unsigned long long *count, int *line) {
  if (!enabled || !count || !line) return fail(JT_ERR_ARG, "null argument");
  *enabled = JT_CHECKS;
  unsigned long long c = 0;
  int l = 0;
  JT_CUDA_TRY(cudaDeviceSynchronize());
  jt_status st = JT_OK;
  for (jt_status (*io)(unsigned long long *, int *) :
       {checks_io<16>, checks_io<32>, checks_io<64>, checks_io<128>, checks_io<256>, checks_io<512>, checks_io<1024>,
        checks_io<2048>, checks_io<4096>})
    if ((st = io(&c, &l)) != JT_OK) return st;
  *count = c;
  *line = l;
  return JT_OK;
}

jt_status jt_debug_vgroup_create(jt_vgroup_t *out, int nranks, int timeout_ms) {
  if (!out || nranks < 1 || timeout_ms < 1) return fail(JT_ERR_ARG, "bad args");
  jt_vgroup_s *V = new (std::nothrow) jt_vgroup_s();
  if (!V) return fail(JT_ERR_ALLOC, "group");
  V->G = nranks;
  V->timeout_ms = timeout_ms;
  V->member.assign(nranks, nullptr);
  V->send.assign(nranks, nullptr);
  V->ev_ready.assign(nranks, nullptr);
  V->ev_done.assign(nranks, nullptr);
  *out = V;
  return JT_OK;
}

jt_status jt_debug_vgroup_destroy(jt_vgroup_t g) {
  if (!g) return JT_OK;
  for (jt_plan_s *m : g->member)
    if (m) return fail(JT_ERR_ARG, "virtual group still has plans: destroy them first");
  delete g;
  return JT_OK;
}

jt_status jt_debug_plan_virtual(jt_plan_t *out, int d, const int64_t n[], const double a[], const double b[],
                                double eps, const jt_opts *opts, jt_vgroup_t group, int rank, int flags) {
  if (!group) return fail(JT_ERR_ARG, "null group");
  return plan_dist_common(out, d, n, a, b, eps, opts, rank, group->G, flags, nullptr, group);
}

jt_status jt_local_box(jt_plan_t p, int which, int64_t lo[], int64_t hi[]) {
  if (!p || !lo || !hi || (which != 0 && which != 1)) return fail(JT_ERR_ARG, "bad args");
  for (int i = 0; i < p->d; ++i) {
    lo[i] = 0;
    hi[i] = p->n[i];
  }
  if (p->dist) {
    const int ax = which == 0 ? 0 : 1;
    const int64_t c = p->n[ax] / p->nranks;
    lo[ax] = p->rank * c;
    hi[ax] = (p->rank + 1) * c;
  }
  return JT_OK;
}

jt_status jt_destroy(jt_plan_t p) {
  if (!p) return JT_OK;
  free_device(p);
  delete p;
  return JT_OK;
}

jt_status jt_plan_rank(jt_plan_t p, int axis, int *r) {
  if (!p || !r || axis < 0 || axis >= p->d) return fail(JT_ERR_ARG, "bad args");
  *r = p->host[axis].r;
  return JT_OK;
}

jt_status jt_plan_info(jt_plan_t p, int axis, int64_t *n, int64_t *nfft, int *k0, int *r) {
  if (!p || axis < 0 || axis >= p->d) return fail(JT_ERR_ARG, "bad args");
  const jt::AxisHost &h = p->host[axis];
  if (n) *n = h.n;
  if (nfft) *nfft = h.N;
  if (k0) *k0 = h.k0;
  if (r) *r = h.r;
  return JT_OK;
}

jt_status jt_plan_nodes(jt_plan_t p, int axis, double *t_host, double *w_host) {
  if (!p || axis < 0 || axis >= p->d) return fail(JT_ERR_ARG, "bad args");
  const jt::AxisHost &h = p->host[axis];
  if (t_host) std::memcpy(t_host, h.t.data(), h.n * sizeof(double));
  if (w_host) std::memcpy(w_host, h.w.data(), h.n * sizeof(double));
  return JT_OK;
}

jt_status jt_plan_factors(jt_plan_t p, int axis, double *u_host, double *v_host, double *phiv_host,
                          int32_t *bins_host) {
  if (!p || axis < 0 || axis >= p->d) return fail(JT_ERR_ARG, "bad args");
  const jt::AxisHost &h = p->host[axis];
  if (u_host) std::memcpy(u_host, h.u.data(), h.u.size() * sizeof(jt::cd));
  if (v_host) std::memcpy(v_host, h.v.data(), h.v.size() * sizeof(jt::cd));
  if (phiv_host) std::memcpy(phiv_host, h.phiv.data(), h.phiv.size() * sizeof(double));
  if (bins_host) std::memcpy(bins_host, h.bins.data(), h.bins.size() * sizeof(int32_t));
  return JT_OK;
}

jt_status jt_plan_sigma(jt_plan_t p, int axis, double *sigma, int *count, int *rmax_used) {
  if (!p || axis < 0 || axis >= p->d) return fail(JT_ERR_ARG, "bad args");
  const jt::AxisHost &h = p->host[axis];
  if (count) *count = (int)h.sigma.size();
  if (rmax_used) *rmax_used = h.rmax_used;
  if (sigma) std::memcpy(sigma, h.sigma.data(), h.sigma.size() * sizeof(double));
  return JT_OK;
}

// Test hook (declared in include/jt_debug.h): the paired-real-term factor set of the forward passes.
jt_status jt_debug_pair_factors(jt_plan_t p, int axis, int *r, int *rreal, double *u_host, double *v_host,
                                double *phiv_host, int32_t *bins_host) {
  if (!p || axis < 0 || axis >= p->d) return fail(JT_ERR_ARG, "bad args");
  const jt::AxisHost &h = p->hostp[axis];
  if (r) *r = p->pair[axis] ? h.r : 0;
  if (rreal) *rreal = p->pair[axis] ? h.rreal : 0;
  if (!p->pair[axis]) return JT_OK;
  if (u_host) std::memcpy(u_host, h.u.data(), h.u.size() * sizeof(jt::cd));
  if (v_host) std::memcpy(v_host, h.v.data(), h.v.size() * sizeof(jt::cd));
  if (phiv_host) std::memcpy(phiv_host, h.phiv.data(), h.phiv.size() * sizeof(double));
  if (bins_host) std::memcpy(bins_host, h.bins.data(), h.bins.size() * sizeof(int32_t));
  return JT_OK;
}

// Test hook (declared in include/jt_debug.h): P~_k, Q~_k by the plan's own route.
jt_status jt_debug_modified_pq(double a, double b, int64_t nt, const double *t, int kmax, double *p_out,
                               double *q_out) {
  if (!t || !p_out || !q_out || nt < 0 || kmax < 0) return fail(JT_ERR_ARG, "bad args");
  if (!(a > -1 && a < 1 && b > -1 && b < 1)) return fail(JT_ERR_DOMAIN, "a, b must lie in (-1, 1)");
  jt::modified_pq(a, b, nt, t, kmax, p_out, q_out);
  return JT_OK;
}

}  // extern "C"
