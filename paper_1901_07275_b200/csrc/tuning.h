// Build-time tuning knobs of the axis-pass kernels and the C ABI.  Each default is the
// measured winner of an A/B on one B200 (tools/ab_time.py); override with -DJT_...=v (build.py `defines`) to
// repeat an experiment.  Nothing here changes results beyond rounding order.
#pragma once

// ---- register budgets and per-thread state ----------------------------------------------------------------
#ifndef JT_PRIV16
#define JT_PRIV16 1  // radix-16 kernels (N >= 64) keep their per-batch state out of registers (PRIV)
#endif
#ifndef JT_REGS16
#define JT_REGS16 168  // registers of the radix-16 inverse kernels
#endif
#ifndef JT_REGS16F
#define JT_REGS16F 128  // registers of the radix-16 forward kernels (16 warps/SM: 256^3-class forwards -4.8 %)
#endif
#ifndef JT_REGS16M4
#define JT_REGS16M4 168  // MAXR = 4 radix-16 kernels (128 spilled: nonuniform 256^3 forward 3.85 -> 3.00 ms)
#endif
#ifndef JT_REGS16M3
#define JT_REGS16M3 144  // MAXR = 3 radix-16 kernels (clustered nonuniform points after the cap-3 bin spreading)
#endif
#ifndef JT_TPRIV
#define JT_TPRIV 1  // per-batch state in tensor memory (tcgen05.ld/st) instead of SMEM
#endif
#ifndef JT_TPRIV_NMAX
#define JT_TPRIV_NMAX 4096  // ... for FFT lengths up to this
#endif
#ifndef JT_SPLITX_TPRIV
#define JT_SPLITX_TPRIV 0  // 1: exchange one real plane at a time even with the state in TMEM (3 barriers)
#endif

// ---- twiddles ----------------------------------------------------------------------------------------------
#ifndef JT_TWT
#define JT_TWT 1  // per-thread twiddles in TMEM (N <= 1024: 512^3 forward 17.9 -> 17.3 ms)
#endif
#ifndef JT_A1_FOLD
#define JT_A1_FOLD 1  // radix-32 forwards: column scale folded into the first DFT butterfly layer (FMAs) ...
#endif
#ifndef JT_A1_FOLD_NMIN
#define JT_A1_FOLD_NMIN 2048  // ... for N >= this (4096^2 forward -2.6 %; 512^3 +0.75 %, 1024 +1.2 %)
#endif
#ifndef JT_PAIRRED
#define JT_PAIRRED 0  // inverse (N <= 512): the two staged degrees' (W V)^T y partials reduced over the warp as a pair
                      // (6 shuffles per term instead of 12; measured slower, r02zx: 512^3 inverse 17.73 -> 17.89 ms,
                      // 256^3 2.00 -> 2.03 ms, 128^3 -0.8 %)
#endif
#ifndef JT_PAIR
#define JT_PAIR 1  // forward passes: two REAL rank terms per complex FFT (Cfg::PAIR kernels, N = 256 / 512 / 2048 / 4096; the plan's
                   // second, real-row-space factor set: 9 FFTs instead of 16 per line at 512^3).  JT_PAIR=0 in the
                   // environment turns it off at plan time (A/B)
#endif
#ifndef JT_PAIR_2048
#define JT_PAIR_2048 1  // ... also FFT length 2048 (16 x 16 x 8; its forward then reads u~ from L2 unless the doubled
                        // u-ring stage still fits)
#endif
#ifndef JT_PAIR_INV
#define JT_PAIR_INV 1  // ... also the inverse / transpose passes (the transposed paired operator)
#endif
#ifndef JT_PAIR_MIN_LINES
#define JT_PAIR_MIN_LINES 2400  // ... for launches of at least this many lines (below, the term-split launches of the
                                // unpaired kernels are faster: 256^2 forward 27 vs 35 us)
#endif
#ifndef JT_ZFIRST
#define JT_ZFIRST 1  // inverse: the first DFT layer skips the thread's zero inputs above R/2 (empty bins > N/2)
#endif
#ifndef JT_VTM
#define JT_VTM 0  // N = 512 forward: v_l from tensor memory (tcgen05.cp from the ring stage) instead of LDS broadcasts
                  // (correct, but 512^3 forward 17.1 -> 30.4 ms: TMEM holds one term's v only, so every warp waits
                  // for the slowest warp's previous term at each term start -- the groups lose the phase spread
                  // that overlaps their FP64 and shared-memory work, r02zp)
#endif
#ifndef JT_TW_PREISSUE
#define JT_TW_PREISSUE 0  // TMEM twiddle chunks loaded one chunk ahead (the next butterfly's during the DFT; r02v: no change)
#endif
#ifndef JT_TWT_INV32
#define JT_TWT_INV32 1  // ... also for the radix-32 inverse (round 1: 2 % slower; after the round-2 changes 512^3
                        // inverse 17.84 -> 17.75 ms, 128^3 +0.4 %, r02zn)
#endif
#ifndef JT_TWT_LARGE
#define JT_TWT_LARGE 1  // N > 1024: one TMEM twiddle copy per lane quadrant (4096^2 forward 4.05 -> 3.81 ms)
#endif
#ifndef JT_TWT_LARGE_INV_NMAX
#define JT_TWT_LARGE_INV_NMAX 2048  // ... inverses up to this N (N = 4096 inverse +1..5 % with it, N = 2048 -2 %)
#endif
#ifndef JT_TWT_CH_LARGE_F
#define JT_TWT_CH_LARGE_F 4  // N > 1024 forward: twiddles per TMEM wait (4 vs 8: -5 % at N = 4096)
#endif
#ifndef JT_TWT_CH_LARGE_I
#define JT_TWT_CH_LARGE_I 8  // N > 1024 inverse: twiddles per TMEM wait (8 vs 4: -3 % at N = 2048)
#endif

// ---- factor and input loads --------------------------------------------------------------------------------
#ifndef JT_URING
#define JT_URING 1  // N > 1024 forward: one-stage TMA ring for u~_l in spare SMEM
#endif
#ifndef JT_SUB
#define JT_SUB 0  // N = 4096: v_l and u~_l through a ring of 16 KB sub-stages shared by the CTA's groups (SUB;
                  // measured slower: 5.06 vs 3.54 ms at 4096^2)
#endif
#ifndef JT_SUB_SPLITX
#define JT_SUB_SPLITX 1  // ... with the split exchange (one real plane at a time) to fit a ring deeper than a term
#endif
#ifndef JT_URING_NMAX
#define JT_URING_NMAX 2048  // ... up to this N (2048 forward -5 %; 4096 +8 %: the stage starves L1)
#endif
#ifndef JT_LOADS_FIRST
#define JT_LOADS_FIRST 2  // bit 0: forward A1, bit 1: inverse bin sums issue factor loads before the TMEM state
#endif
#ifndef JT_LF_INV_NMIN
#define JT_LF_INV_NMIN 4096  // ... bit 1 from this N (4096 inverse -7 %, 2048 +1 %; bit 0: 2048 forward +3 %)
#endif
#ifndef JT_VUNROLL
#define JT_VUNROLL 4  // N > 512: batch-start W V loops unrolled (4096 forward -7 %, 2048 inverse -7 %)
#endif
#ifndef JT_PREFETCH
#define JT_PREFETCH 1  // next-line L2 prefetch at batch start ...
#endif
#ifndef JT_PREFETCH_NMIN
#define JT_PREFETCH_NMIN 256  // ... for forwards with N in [NMIN, NMAX] (256^3 -3.4 %; 64^3 +8 %, 512^3 +2.9 %)
#endif
#ifndef JT_PREFETCH_NMAX
#define JT_PREFETCH_NMAX 256
#endif

// ---- radix and host pipeline (jt_api.cu) -------------------------------------------------------------------
#ifndef JT_R64
#define JT_R64 16  // register radix at N = 64 (32: 64^3 inverse +27 %)
#endif
#ifndef JT_R128
#define JT_R128 32  // register radix at N = 128 (32 vs 16: 128^3 forward -7.7 %, inverse -9.5 %)
#endif
#ifndef JT_R128_TS
#define JT_R128_TS 16  // ... in its term-split launches (32 there: 128^2 +30 %)
#endif
#ifndef JT_R256
#define JT_R256 16  // register radix at N = 256 (32: 256^3 inverse -2.3 %, forward +5.6 %, 256^2 +20 %)
#endif
#ifndef JT_R512
#define JT_R512 32  // register radix at N = 512 (16: two exchanges, 26.4 vs 21.7 ms at 512^3 before the TMEM work;
                    // with the current TMEM layouts the radix-16 N = 512 launch configuration is not valid)
#endif
#ifndef JT_R1024
#define JT_R1024 32  // register radix at N = 1024
#endif
#ifndef JT_R2048
#define JT_R2048 16  // register radix at N = 2048 (16 vs 32: 2048^2 inverse -6.4 %, forward -0.8 %)
#endif
#ifndef JT_R4096
#define JT_R4096 32  // register radix at N = 4096 (16: forward +9 %, inverse +12 %)
#endif
#ifndef JT_LG4096
#define JT_LG4096 1  // lines per group of the N = 4096 radix-32 kernels (2: no TMEM twiddles, 4096^2 3.46 -> 3.91 ms)
#endif
#ifndef JT_UPF
#define JT_UPF 0  // factors from L2 (N > 1024): the post-FFT factor entries prefetched into L1 before the FFT
                  // (measured slower: 4096^2 forward 3.46 -> 3.87 ms, inverse 3.70 -> 4.02)
#endif
#ifndef JT_LATE_SYNC
#define JT_LATE_SYNC 1  // end-of-term group barrier moved before the next term's first exchange (Cfg::LATE: only
                        // the ring-less N = 4096 forward, 4096^2 -2.4 %; slower elsewhere)
#endif
#ifndef JT_TS_CLUSTER
#define JT_TS_CLUSTER 1  // term-split launches as thread-block clusters reducing through DSMEM (no ts_reduce launch)
#endif
#ifndef JT_TS_PUSH
#define JT_TS_PUSH 1  // cluster reduction by bulk copies into the owners' shared memory (else 8-byte remote loads)
#endif
#ifndef JT_TS_FUSE
#define JT_TS_FUSE 0  // term-split axis d-1 pass: partials summed by the next (cluster term-split) pass's loads
                      // (measured slower: 256^2 30 -> 40 us, the partial loads take more round trips than the
                      // reduction they replace, r02zk)
#endif
#ifndef JT_TS_CLUSTER_MAX
#define JT_TS_CLUSTER_MAX 16  // largest cluster (non-portable above 8; smaller if the device cannot place it)
#endif
#ifndef JT_WG_LARGE
#define JT_WG_LARGE 0  // N: the one-warp-group configuration (Cfg::WG) for every launch of FFT length N, not only
                       // the term-split ones (0: off)
#endif
#ifndef JT_TS_WG
#define JT_TS_WG 1  // term-split launches of TPL = 16 passes use the one-warp-group configuration (Cfg::WG)
#endif
#ifndef JT_WG_GPC
#define JT_WG_GPC 8  // groups per CTA of the one-warp-group term-split kernels (4: two CTAs per SM)
#endif
#ifndef JT_GSPLIT
#define JT_GSPLIT 2  // group term split (2 or 0 = off): up to this many groups of a term-split CTA share its terms when the batch fits
                     // in one group (1D transforms; 0: off; the cluster reduction reads at most 2 partials per CTA)
#endif
#ifndef JT_PDL
#define JT_PDL 1  // axis-pass kernels launched with programmatic dependent launch (prologue overlaps the previous tail)
#endif
#ifndef JT_PDL_PREFETCH
#define JT_PDL_PREFETCH 1  // term-split launches: L2 prefetch of the batch's input lines before the dependency wait
#endif
#ifndef JT_HOST_SCHED
#define JT_HOST_SCHED 2  // single-GPU *_host pipeline: 0 = axes d-1..1 on arriving row chunks, then axis 0 in column
                         // blocks copied back pitched; 1 = axis 0 first, then row chunks copied back contiguous;
                         // 2 = 1 for 2D, 0 for 3D (e2e streams, tools/e2e_ab.py r02p: 4096^2 4.36 -> 4.20 ms with 1,
                         // but 512^3 24.7 -> 26.9 and 256^3 3.13 -> 3.53 ms)
#endif
#ifndef JT_HOST_SLOTS
#define JT_HOST_SLOTS 2  // staging slots of the *_host entry points (3: no change in the 512^3 e2e stream)
#endif
