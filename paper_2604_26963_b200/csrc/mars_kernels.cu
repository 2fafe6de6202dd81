// B200 (sm_100a) kernels of the MARS scheduling step.
//
// Pipeline: k_scan on the main stream, then the control plane
// on a side stream concurrently with the walk on the main stream:
//   k_scan        persistent cooperative pass over the session table, one CTA
//                 per SM: pin expiry, MLFQ aging (promote_waiting), counters,
//                 per-CTA key histograms and a per-row digit record; grid
//                 barrier; exact global top-k thresholds, window / victim
//                 candidates, S2 retention for BOUNDARY rows, expired pins in
//                 row order; CTA 0 finalises pool/telemetry scalars and
//                 refresh_pressure.
//   k_exp_*       [side] expired pins in session-id (rank) order when the
//                 table is not rank-ordered.
//   k_control     [side] the control plane in one cooperative launch: pack_queue
//                 (one CTA for small queues / first fit, grid-wide stable LSD
//                 sort for big ones), update_window + triple clamp, admit() of
//                 the packed prefix, residual queue; admitted rows that can
//                 join the window become candidates.
//   k_walk        single CTA: window top-k, build_plan decode/prefill passes
//                 with try_fit and reclamation (victim stream or exact
//                 full-table fallback), plan + ordered journal.  Waits for the
//                 admission only when an admitted session can join the window.
//
// Compiled with --fmad=false: every f64 expression keeps CPython's IEEE
// rounding so retention / admission scalars are bit-identical.

#include <cooperative_groups.h>
#include <stdlib.h>
#include <string.h>
#include <cuda_runtime.h>
#include <stdio.h>

namespace cg = cooperative_groups;

#include "mars_internal.cuh"
#include "mars_launch.h"

#define FULL 0xffffffffu

#ifdef MARS_PHASE_TIMING
// Debug builds only (-DMARS_PHASE_TIMING): per-CTA %globaltimer stamps at
// named points of the step, dumped as a timeline after each step.
#define PT_SLOTS 64
__device__ unsigned long long g_ptime[1024][PT_SLOTS];
__device__ __forceinline__ void ptime(int k) {
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_ptime[blockIdx.x][k] = t;
  }
}
__global__ void k_ptime_dump() {
  unsigned long long t0 = ~0ull;
  for (int i = 0; i < 1024; ++i)
    if (g_ptime[i][0]) t0 = min(t0, g_ptime[i][0]);
  if (g_ptime[0][32]) t0 = min(t0, g_ptime[0][32]);  // k_work_init
  printf("t0 %llu\n", t0);
  for (int k = 0; k < PT_SLOTS; ++k) {
    unsigned long long mn = ~0ull, mx = 0;
    int cnt = 0;
    for (int i = 0; i < 1024; ++i) {
      unsigned long long v = g_ptime[i][k];
      if (!v) continue;
      cnt++;
      mn = min(mn, v - t0);
      mx = max(mx, v - t0);
      g_ptime[i][k] = 0;
    }
    if (cnt) printf("stamp %2d: ctas %4d  min %7.2f us  max %7.2f us\n", k, cnt, mn / 1e3, mx / 1e3);
  }
}
#define PTIME(k) ptime(k)
#else
#define PTIME(k)
#endif

// one of a struct's two buffers by a runtime index, as a select: indexing a
// kernel parameter's array with a runtime value makes the compiler copy the
// whole parameter struct into local memory at kernel entry (every thread)
#define PICK2(arr, i) ((i) ? (arr)[1] : (arr)[0])

// ---------------------------------------------------------------------------
// block utilities
// ---------------------------------------------------------------------------

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// block-wide exclusive scan of one i64 per thread (blockDim.x a multiple of
// 32, every thread calls it); *total = the block's sum
__device__ __forceinline__ long long block_excl_scan_i64(long long v, long long* total) {
  __shared__ long long s_ws[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  long long incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long x = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += x;
  }
  __syncthreads();
  if (lane == 31) s_ws[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    long long t = lane < nw ? s_ws[lane] : 0ll;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long x = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += x;
    }
    s_ws[lane] = t;
  }
  __syncthreads();
  *total = s_ws[31];
  return (wid ? s_ws[wid - 1] : 0ll) + incl - v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T x = __shfl_xor_sync(FULL, v, o);
    v = x > v ? x : v;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T x = __shfl_xor_sync(FULL, v, o);
    v = x < v ? x : v;
  }
  return v;
}

// block-wide sum; `sh` needs 32 slots; all threads get the result
template <typename T>
__device__ T block_sum(T v, T* sh) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  T r = (threadIdx.x < nw) ? sh[threadIdx.x] : (T)0;
  if (wid == 0) r = warp_sum(r);
  if (threadIdx.x == 0) sh[0] = r;
  __syncthreads();
  r = sh[0];
  __syncthreads();
  return r;
}

template <typename T>
__device__ T block_max(T v, T* sh, T lowest) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  T r = (threadIdx.x < nw) ? sh[threadIdx.x] : lowest;
  if (wid == 0) r = warp_max(r);
  if (threadIdx.x == 0) sh[0] = r;
  __syncthreads();
  r = sh[0];
  __syncthreads();
  return r;
}

template <typename T>
__device__ T block_min(T v, T* sh, T highest) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_min(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  T r = (threadIdx.x < nw) ? sh[threadIdx.x] : highest;
  if (wid == 0) r = warp_min(r);
  if (threadIdx.x == 0) sh[0] = r;
  __syncthreads();
  r = sh[0];
  __syncthreads();
  return r;
}

// Smallest bin d with cumsum(h[0..d]) >= k over `nb` bins (nb multiple of
// blockDim.x); returns nb-1 if the total is below k.  *below = cumsum(h[0..d-1]),
// *upto = cumsum(h[0..d]).  `sh` needs blockDim.x + 32 u32 slots.
__device__ void block_threshold(const u32* h, int nb, u32 k, u32* sh, int* out_d, u32* below,
                                u32* upto) {
  int per = nb / blockDim.x;
  int base = threadIdx.x * per;
  u32 s = 0;
  for (int i = 0; i < per; ++i) s += h[base + i];
  // inclusive scan of per-thread sums
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int off = 1; off < (int)blockDim.x; off <<= 1) {
    u32 x = (threadIdx.x >= (unsigned)off) ? sh[threadIdx.x - off] : 0u;
    __syncthreads();
    sh[threadIdx.x] += x;
    __syncthreads();
  }
  u32 incl = sh[threadIdx.x];
  u32 excl = incl - s;
  u32 total = sh[blockDim.x - 1];
  __shared__ int s_d;
  __shared__ u32 s_below, s_upto;
  if (threadIdx.x == 0) {
    s_d = nb - 1;
    s_below = total - h[nb - 1];
    s_upto = total;
  }
  __syncthreads();
  if (total >= k && excl < k && incl >= k) {
    u32 c = excl;
    for (int i = 0; i < per; ++i) {
      u32 nc = c + h[base + i];
      if (nc >= k) {
        s_d = base + i;
        s_below = c;
        s_upto = nc;
        break;
      }
      c = nc;
    }
  }
  __syncthreads();
  *out_d = s_d;
  *below = s_below;
  *upto = s_upto;
  __syncthreads();
}

// warp-aggregated append: returns the slot for lanes with pred, -1 otherwise
__device__ __forceinline__ int warp_append(int* counter, bool pred) {
  u32 m = __ballot_sync(__activemask(), pred);
  if (!m) return -1;
  int lane = threadIdx.x & 31;
  int leader = __ffs(m) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(counter, __popc(m));
  base = __shfl_sync(__activemask(), base, leader);
  if (!pred) return -1;
  return base + __popc(m & ((1u << lane) - 1u));
}

// refresh_pressure (telemetry.py:174-208): two-threshold hysteresis on both flags
__device__ void refresh_pressure(const Cfg& c, mars_scalars* sc, int worker_slots, double u) {
  double slots = (double)worker_slots;
  int at = sc->active_tools, qt = sc->queued_tools;
  bool hi = ((double)at >= c.cpu_hi * slots) || qt > 0;
  bool lo = ((double)at < c.cpu_lo * slots) && qt == 0;
  int hs = hi ? sc->cpu_high_streak + 1 : 0;
  int ls = lo ? sc->cpu_low_streak + 1 : 0;
  int on = sc->cpu_overloaded;
  if (!on && hs >= c.hyst) {
    on = 1;
    ls = 0;
  } else if (on && ls >= c.hyst) {
    on = 0;
    hs = 0;
  }
  sc->cpu_overloaded = on;
  sc->cpu_high_streak = hs;
  sc->cpu_low_streak = ls;
  hi = u >= c.kv_hi;
  lo = u < c.kv_lo;
  hs = hi ? sc->kv_high_streak + 1 : 0;
  ls = lo ? sc->kv_low_streak + 1 : 0;
  on = sc->kv_overloaded;
  if (!on && hs >= c.hyst) {
    on = 1;
    ls = 0;
  } else if (on && ls >= c.hyst) {
    on = 0;
    hs = 0;
  }
  sc->kv_overloaded = on;
  sc->kv_high_streak = hs;
  sc->kv_low_streak = ls;
}

// ---------------------------------------------------------------------------
// K_A: scan (expiry, aging, counters, histograms); last CTA finalises
// ---------------------------------------------------------------------------

#define SCAN_TPB 1024
// resident k_scan CTAs per SM (two 512-thread CTAs per SM measured the same
// as one 1024-thread CTA at 1M and 64M rows, r2; the block-level helpers
// take any SCAN_TPB that is a multiple of 32)
#define SCAN_CTAS_PER_SM 1
#define SCAN_TILE (SCAN_TPB * SCAN_RPT)  // rows per tile (4096)

// Per-row digit record written by phase 1 and read by phase 2 of k_scan:
// low half = window digit (DIG_NONE if the row is not ready, DIG_BND set for
// a boundary row), high half = victim digit (DIG_NONE if not a victim,
// DIG_EXP for a pin that expired this step).
#define DIG_NONE 0x8000u
#define DIG_BND 0x4000u
#define DIG_EXP 0x4000u
#define DIG_ABOVE 0x7fffu  // victim digit above every threshold (not computed)

// For two HIST_BINS shared histograms at once: the smallest bin d with
// cumsum(h[0..d]) >= k (HIST_BINS-1 if the total is below k), and
// *upto = cumsum(h[0..d]).  Warp-shuffle scans, three barriers for both.
// blockDim.x == SCAN_TPB, HIST_BINS / SCAN_TPB bins per thread.
__device__ void block_threshold_pair(const u32* ha, u32 ka, const u32* hb, u32 kb, u32* wsum2,
                                     int* da, u32* ua, int* db, u32* ub) {
  constexpr int PER = HIST_BINS / SCAN_TPB;
  constexpr int NW = SCAN_TPB / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int base = threadIdx.x * PER;
  u32 va[PER], vb[PER];
  u32 sa = 0, sb = 0;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    va[i] = ha[base + i];
    vb[i] = hb[base + i];
    sa += va[i];
    sb += vb[i];
  }
  u32 ia = sa, ib = sb;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    u32 xa = __shfl_up_sync(FULL, ia, o), xb = __shfl_up_sync(FULL, ib, o);
    if (lane >= o) {
      ia += xa;
      ib += xb;
    }
  }
  __shared__ int s_d[2];
  __shared__ u32 s_up[2];
  if (lane == 31) {
    wsum2[wid] = ia;
    wsum2[32 + wid] = ib;
  }
  if (threadIdx.x == 0) {
    s_d[0] = s_d[1] = HIST_BINS - 1;
    s_up[0] = s_up[1] = 0xffffffffu;
  }
  __syncthreads();
  if (wid < 2) {
    u32 t = lane < NW ? wsum2[wid * 32 + lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      u32 x = __shfl_up_sync(FULL, t, o);
      if (lane >= o) t += x;
    }
    wsum2[wid * 32 + lane] = t;
  }
  __syncthreads();
  const u32 ta = wsum2[31], tb = wsum2[63];
  ia += wid ? wsum2[wid - 1] : 0u;
  ib += wid ? wsum2[32 + wid - 1] : 0u;
  const u32 ea = ia - sa, eb = ib - sb;
  if (ta >= ka && ea < ka && ia >= ka) {
    u32 cum = ea;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      u32 nc = cum + va[i];
      if (cum < ka && nc >= ka) {
        s_d[0] = base + i;
        s_up[0] = nc;
      }
      cum = nc;
    }
  }
  if (tb >= kb && eb < kb && ib >= kb) {
    u32 cum = eb;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      u32 nc = cum + vb[i];
      if (cum < kb && nc >= kb) {
        s_d[1] = base + i;
        s_up[1] = nc;
      }
      cum = nc;
    }
  }
  __syncthreads();
  *da = s_d[0];
  *ua = (s_up[0] == 0xffffffffu) ? ta : s_up[0];
  *db = s_d[1];
  *ub = (s_up[1] == 0xffffffffu) ? tb : s_up[1];
  __syncthreads();
}

// ---- 1D TMA (cp.async.bulk) + mbarrier helpers -----------------------------
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ u32 smem_u32(const void* p) {
  return (u32)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// bulk copy global -> shared (16-byte aligned, size a multiple of 16)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---- grid radix refinement of the candidate lists ------------------------
typedef unsigned __int128 u128;
__device__ __forceinline__ u128 mk128(u64 h, u64 l) { return ((u128)h << 64) | (u128)l; }
__device__ __forceinline__ int clz128(u128 x) {
  const u64 h = (u64)(x >> 64);
  return h ? __clzll((long long)h) : 64 + __clzll((long long)(u64)x);
}

// Exact radix select over the emitted 128-bit keys of the window list (0)
// and the victim list (1), by the whole cooperative grid: each round
// histograms the next 8 bits of the keys still sharing the prefix (CTA slices
// of the list, shared-memory counts, one global add per bin) and folds their
// AND / OR, one grid barrier, and every CTA derives the bin holding the k-th
// key from the same counts -- or, when every key of the group shared the
// digit, jumps to the group's first differing bit.  It stops once that bin holds <= REF_STOP keys; the refined list is
// every key whose bits above the bin's position are <= the prefix's: the
// exact top k plus fewer than REF_STOP keys, compacted into wr_* / vr_*.
// Called by every thread of every CTA after a grid barrier (the lists are
// complete).  Keys are unique (session rank), so at most 16 rounds.
__device__ void grid_refine(cg::grid_group& grid, Work* w, Bufs& b, bool on_w, bool on_v, int kw,
                            int kv) {
  __shared__ u32 sh[2][256];
  __shared__ u32 s_ws[2][8];
  __shared__ unsigned long long s_ga[2][2], s_go[2][2];
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x, bd = blockDim.x;
  const int lane = tid & 31, wid = tid >> 5;
  const int n[2] = {__ldcg(&w->n_wc), __ldcg(&w->n_vc)};
  const u64* khp[2] = {b.wc_hi, b.vc_key};
  const u64* klp[2] = {b.wc_lo, b.vc_kl};
  const bool on[2] = {on_w, on_v};
  bool act[2];
  u128 P[2];
  int top[2], fin_s[2];
  u32 need[2] = {(u32)kw, (u32)kv};
  // the first round starts at the top byte; a round whose digit is common to
  // the whole group jumps to the group's first differing bit (its AND / OR)
#pragma unroll
  for (int l = 0; l < 2; ++l) {
    act[l] = on[l];
    P[l] = 0;
    top[l] = 127;
    fin_s[l] = 0;
  }
  int it = 0;
  while (act[0] || act[1]) {  // grid-uniform: every CTA holds the same state
    PTIME(48 + (it < 7 ? it : 7));
    const int buf = it % 3;
    for (int i = tid; i < 512; i += bd) (&sh[0][0])[i] = 0u;
    if (tid < 4) {
      (&s_ga[0][0])[tid] = ~0ull;
      (&s_go[0][0])[tid] = 0ull;
    }
    __syncthreads();
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      if (!act[l]) continue;
      const int lo_b = top[l] >= 7 ? top[l] - 7 : 0;
      const u32 msk = (1u << (top[l] - lo_b + 1)) - 1u;
      const int sft = top[l] + 1;
      const u128 pp = sft >= 128 ? (u128)0 : (P[l] >> sft);
      const i64 i0 = (i64)n[l] * g / G, i1 = (i64)n[l] * (g + 1) / G;
      u64 ah = ~0ull, al = ~0ull, oh = 0ull, ol = 0ull;  // the group's AND / OR
      for (i64 i = i0 + tid; i < i1; i += bd) {
        const u64 kh_ = __ldcg(khp[l] + i), kl_ = __ldcg(klp[l] + i);
        const u128 key = mk128(kh_, kl_);
        if (sft < 128 && (key >> sft) != pp) continue;
        atomicAdd(&sh[l][(u32)(key >> lo_b) & msk], 1u);
        ah &= kh_;
        al &= kl_;
        oh |= kh_;
        ol |= kl_;
      }
#pragma unroll
      for (int q = 16; q > 0; q >>= 1) {
        ah &= __shfl_xor_sync(FULL, ah, q);
        al &= __shfl_xor_sync(FULL, al, q);
        oh |= __shfl_xor_sync(FULL, oh, q);
        ol |= __shfl_xor_sync(FULL, ol, q);
      }
      if (lane == 0) {
        if (~ah) atomicAnd(&s_ga[l][0], ah);
        if (~al) atomicAnd(&s_ga[l][1], al);
        if (oh) atomicOr(&s_go[l][0], oh);
        if (ol) atomicOr(&s_go[l][1], ol);
      }
    }
    __syncthreads();
#pragma unroll
    for (int l = 0; l < 2; ++l)
      if (act[l]) {
        for (int d = tid; d < 256; d += bd)
          if (sh[l][d]) atomicAdd(&w->ref_hist[l][buf][d], sh[l][d]);
        if (tid < 2 && ~s_ga[l][tid]) atomicAnd(&w->ref_gand[l][buf][tid], s_ga[l][tid]);
        if (tid < 2 && s_go[l][tid]) atomicOr(&w->ref_gor[l][buf][tid], s_go[l][tid]);
      }
    grid.sync();
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      if (!act[l]) continue;
      // the bin holding the need-th key: a 256-entry scan on 8 warps
      const u32 v = tid < 256 ? __ldcg(&w->ref_hist[l][buf][tid]) : 0u;
      u32 incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 x = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += x;
      }
      __shared__ int s_bin[2];
      __shared__ u32 s_below[2], s_cntb[2];
      if (tid < 256 && lane == 31) s_ws[l][wid] = incl;
      if (tid == 0) {  // (need beyond the total cannot happen: the list holds > k keys)
        s_bin[l] = 255;
        s_below[l] = 0;
        s_cntb[l] = 0;
      }
      __syncthreads();
      u32 wb = 0;
      if (tid < 256)
        for (int q = 0; q < wid; ++q) wb += s_ws[l][q];
      incl += wb;
      if (tid < 256 && incl - v < need[l] && incl >= need[l]) {
        s_bin[l] = tid;
        s_below[l] = incl - v;
        s_cntb[l] = v;
      }
      __syncthreads();
      const int lo_b = top[l] >= 7 ? top[l] - 7 : 0;
      // the group's first differing bit: below this round's digit, every key
      // of the group fell into one bin -- jump straight to that bit (ties in
      // the leading key fields: equal times, equal levels and footprints)
      const u128 ga = mk128(__ldcg(&w->ref_gand[l][buf][0]), __ldcg(&w->ref_gand[l][buf][1]));
      const u128 go = mk128(__ldcg(&w->ref_gor[l][buf][0]), __ldcg(&w->ref_gor[l][buf][1]));
      const u128 gx = ga ^ go;
      const int dtop = gx ? 127 - clz128(gx) : -1;
      if (dtop < lo_b) {
        if (dtop < 0) {  // a single key left
          P[l] = ga;
          act[l] = false;
          fin_s[l] = 0;
        } else {
          P[l] = (ga >> (dtop + 1)) << (dtop + 1);
          top[l] = dtop;
        }
      } else {
        need[l] -= s_below[l];
        P[l] |= (u128)(u32)s_bin[l] << lo_b;
        const u32 cnt = s_cntb[l];
        top[l] = lo_b - 1;
        if (cnt <= (u32)REF_STOP || top[l] < 0) {
          act[l] = false;
          fin_s[l] = lo_b;
        }
      }
      __syncthreads();
    }
    // the buffer two rounds ahead was last read before this round's barrier
    if (g == 0) {
      const int nb = (it + 2) % 3;
      for (int i = tid; i < 512; i += bd) (&w->ref_hist[0][0][0])[((i >> 8) * 3 + nb) * 256 + (i & 255)] = 0u;
      if (tid < 4) {
        w->ref_gand[tid >> 1][nb][tid & 1] = ~0ull;
        w->ref_gor[tid >> 1][nb][tid & 1] = 0ull;
      }
    }
    ++it;
  }
  PTIME(56);
  // compaction: the keys at or below the bound, in any order (the walk sorts)
#pragma unroll
  for (int l = 0; l < 2; ++l) {
    if (!on[l]) continue;
    const int sft = fin_s[l];
    const u128 pp = P[l] >> sft;
    const i64 i0 = (i64)n[l] * g / G, i1 = (i64)n[l] * (g + 1) / G;
    for (i64 base = i0; base < i1; base += bd) {
      const i64 i = base + tid;
      bool pred = false;
      if (i < i1) pred = (mk128(__ldcg(khp[l] + i), __ldcg(klp[l] + i)) >> sft) <= pp;
      int slot = warp_append(l ? &w->n_vr : &w->n_wr, pred);
      if (l == 1 && slot >= VR_CAP) {
        w->status |= ST_WALK_OVERFLOW;
        slot = -1;
      }
      if (slot >= 0) {
        if (l == 0) {
          b.wr_hi[slot] = __ldcg(&b.wc_hi[i]);
          b.wr_lo[slot] = __ldcg(&b.wc_lo[i]);
          b.wr_row[slot] = __ldcg(&b.wc_row[i]);
        } else {
          b.vr_key[slot] = __ldcg(&b.vc_key[i]);
          b.vr_kl[slot] = __ldcg(&b.vc_kl[i]);
          b.vr_whi[slot] = __ldcg(&b.vc_whi[i]);
          b.vr_wlo[slot] = __ldcg(&b.vc_wlo[i]);
          b.vr_row[slot] = __ldcg(&b.vc_row[i]);
          b.vr_blk[slot] = __ldcg(&b.vc_blk[i]);
        }
      }
    }
  }
  if (g == 0 && tid == 0) {
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      w->ref_on[l] = on[l] ? 1 : 0;
      w->ref_p[l][0] = (u64)(P[l] >> 64);
      w->ref_p[l][1] = (u64)P[l];
      w->ref_s[l] = fin_s[l];
    }
    w->ref_iters = it;
  }
}

// The victim list (<= REF_TRIG_V entries, or the refined list) in the
// policy's reclaim order, by rank counting on the whole grid: every CTA
// stages all keys in shared memory, each warp ranks one entry (keys are
// unique) and the entry lands at its rank in the stream arrays (vs_*), the
// first `cap` of them.  Called by every thread after the list is complete.
__device__ void grid_rank_victims(Work* w, Bufs& b, bool ref_v, int cap, u64* sk /* smem */) {
  const int n = ref_v ? __ldcg(&w->n_vr) : __ldcg(&w->n_vc);
  const u64* kh = ref_v ? b.vr_key : b.vc_key;
  const u64* kl = ref_v ? b.vr_kl : b.vc_kl;
  const int m = n < 2 * VSTREAM_CAP ? n : 2 * VSTREAM_CAP;  // (the list never exceeds it)
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    sk[2 * i] = __ldcg(kh + i);
    sk[2 * i + 1] = __ldcg(kl + i);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = gw; i < m; i += nw) {
    const u64 h = sk[2 * i], l = sk[2 * i + 1];
    int cnt = 0;
    for (int j = lane; j < m; j += 32) cnt += key_lt(sk[2 * j], sk[2 * j + 1], h, l) ? 1 : 0;
    const int r = __reduce_add_sync(FULL, cnt);
    if (lane == 0 && r < cap) {
      b.vs_key[r] = h;
      b.vs_kl[r] = l;
      b.vs_whi[r] = __ldcg((ref_v ? b.vr_whi : b.vc_whi) + i);
      b.vs_wlo[r] = __ldcg((ref_v ? b.vr_wlo : b.vc_wlo) + i);
      b.vs_row[r] = __ldcg((ref_v ? b.vr_row : b.vc_row) + i);
      b.vs_blk[r] = __ldcg((ref_v ? b.vr_blk : b.vc_blk) + i);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) w->vs_on = m == n ? 1 : 0;
}

// k_scan staging: one round = SCAN_TPB consecutive rows (one per thread),
// every column k_scan reads arrives by TMA into one of SCAN_NBUF ring buffers.
// (the queued rows' req_blocks come from the admission list itself)
#define SCAN_R SCAN_TPB
#define SCAN_NBUF 3
#define SB_RS 0                       // f64 ready_since (or arrival when coordinator off)
#define SB_WS (SB_RS + 8 * SCAN_R)    // f64 wait_since
#define SB_DL (SB_WS + 8 * SCAN_R)    // f64 pin deadline
#define SB_KV (SB_DL + 8 * SCAN_R)    // i32 kv tokens
#define SB_PB (SB_KV + 4 * SCAN_R)    // i32 pinned blocks
#define SB_FL (SB_PB + 4 * SCAN_R)    // u8 flags
#define SB_PH (SB_FL + SCAN_R)        // u8 phase
#define SB_LV (SB_PH + SCAN_R)        // u8 level
#define SB_PR (SB_LV + SCAN_R)        // u8 promotions
#define SB_PL (SB_PR + SCAN_R)        // u8 pinned level
#define SB_BYTES (SB_PL + SCAN_R)     // 37 bytes per row
#define SCAN_ROW_BYTES 37

static size_t scan_stage_bytes() { return (size_t)SCAN_NBUF * SB_BYTES; }

// Persistent cooperative scan, one CTA per SM; CTA g owns the contiguous rows
// [g * chunk, (g + 1) * chunk), chunk a multiple of 16.
//  phase 1: stream the rows once through a 3-deep TMA ring (bulk copies of
//           every column the scan reads, completion on mbarriers) -- expiry,
//           aging (promote_waiting), counters, local histograms, the per-row
//           digit record, expired pins compacted in row order into the CTA's
//           segment.  After rounds 0 and 2 the CTA's running top-k bins bound
//           the histogram: rows above them cannot be in the CTA's (so not in
//           the global) top-k and skip their shared-memory atomics;
//  grid barrier;
//  phase 2: every CTA derives the global thresholds from the merged histogram
//           prefix and emits its own window / victim candidates from the digit
//           record, the S2 retention of its boundary rows and its expired
//           pins at their place in the row-ordered list; CTA 0 finalises the
//           probe / refresh scalars.
__global__ void __launch_bounds__(SCAN_TPB, SCAN_CTAS_PER_SM) k_scan(Tab t, Cfg c, Work* w, Bufs b,
                                                      mars_scalars* sc, i64 n_rows, i64* xc,
                                                      i64 chunk, Queue Q, const i32* qsel_p,
                                                      int no_stage, Kv kv, int kv_fused) {
  extern __shared__ __align__(128) unsigned char sdyn[];
  __shared__ u32 hw[HIST_BINS];
  __shared__ u32 hv[HIST_BINS];
  __shared__ u32 wsum[64];
  __shared__ u32 s_wc[64];  // per-warp kept-row counts of the current round (x2)
  // S5 with a rank-ordered table (kv_fused): the expired pins' tables go back
  // to the free stack in row order, so this scan also lays out their frees
  // (segment / loose-ID / tail-chunk offsets, as k_kv_exp_scan would) and
  // k_kv_exp_push runs right after it
  __shared__ u32 s_kv[3];  // (per-CTA sums fit 32 bits: < rows x 128 segments)
  __shared__ i64 s_kvb[3];  // the free stack's pre-step tops (segments, arena, chunk pool)
  __shared__ u32 s_bw, s_bv;  // running histogram bounds (digits above are not counted)
  __shared__ __align__(8) u64 bars[SCAN_NBUF];
  cg::grid_group grid = cg::this_grid();

  PTIME(0);
  for (int i = threadIdx.x; i < HIST_BINS; i += blockDim.x) hw[i] = hv[i] = 0;
  if (threadIdx.x < 3) s_kv[threadIdx.x] = 0;
  if (kv_fused && threadIdx.x == 0) {  // read before the grid barrier (CTA 0 moves them after)
    s_kvb[0] = kv.s->seg_top;
    s_kvb[1] = kv.s->arena_top;
    s_kvb[2] = kv.s->cfs_top;
  }
  const int me = blockIdx.x;
  const i64 cs = (i64)me * chunk;
  const i64 ce = (cs + chunk < n_rows) ? cs + chunk : n_rows;
  const int nrounds = ce > cs ? (int)((ce - cs + SCAN_R - 1) / SCAN_R) : 0;
  const double* tcol = c.coord ? t.rs : t.arr;
  // one thread issues a round's bulk copies (rows rounded up to 16: the
  // columns are padded, the extra rows are never used)
  auto issue = [&](int rd) {
    const i64 rb = cs + (i64)rd * SCAN_R;
    const int nr = (int)((ce - rb) < SCAN_R ? (ce - rb) : SCAN_R);
    const u32 n16 = (u32)((nr + 15) & ~15);
    unsigned char* B = sdyn + (size_t)(rd % SCAN_NBUF) * SB_BYTES;
    u64* bar = &bars[rd % SCAN_NBUF];
    mbar_expect_tx(bar, n16 * SCAN_ROW_BYTES);
    bulk_g2s(B + SB_RS, tcol + rb, n16 * 8, bar);
    bulk_g2s(B + SB_WS, t.ws + rb, n16 * 8, bar);
    bulk_g2s(B + SB_DL, t.dl + rb, n16 * 8, bar);
    bulk_g2s(B + SB_KV, t.kv + rb, n16 * 4, bar);
    bulk_g2s(B + SB_PB, t.pb + rb, n16 * 4, bar);
    bulk_g2s(B + SB_FL, t.flags + rb, n16, bar);
    bulk_g2s(B + SB_PH, t.phase + rb, n16, bar);
    bulk_g2s(B + SB_LV, t.level + rb, n16, bar);
    bulk_g2s(B + SB_PR, t.promos + rb, n16, bar);
    bulk_g2s(B + SB_PL, t.plevel + rb, n16, bar);
  };
  if (threadIdx.x == 0) {
    s_bw = s_bv = HIST_BINS - 1;
    for (int q = 0; q < SCAN_NBUF; ++q) mbar_init(&bars[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int rd = 0; rd < nrounds && rd < SCAN_NBUF; ++rd) issue(rd);
  }

  // Launched as k_work_init's programmatic dependent: everything above (the
  // ring's first fill included) overlaps the step head; the work area and
  // the step input are read only past this point
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const double now = w->in.now;
  const int mode = w->in.mode;
  const bool do_exp = !(mode & MARS_MODE_SKIP_EXPIRY) && policy_pins(c);
  // the victim stream is the policy's reclaim order (run_reclaim_key /
  // pin_reclaim_key); pins are victims of the policies that pin
  const bool vic_pin = policy_pins(c);
  const double ascale = (now > 0.0 && now < 1e300) ? 2048.0 / now : 0.0;
  // S2 at tool boundaries: MARS's economics or the TTL rule; fcfs and
  // program_priority never pin (retention_decision None, baselines.py:82-86)
  const bool ret_on = c.policy != POL_FCFS && c.policy != POL_PP;
  const double scale = (now > 0.0 && now < 1e300) ? 1024.0 / now : 0.0;
  // Phase 1 compacts, in row order, every row phase 2 may emit (a digit at
  // or below the CTA's running bound -- the final thresholds are never above
  // it --, a boundary row, an expired pin) with its digit record into the
  // CTA's segment of cand_row / row_dig; phase 2 reads only that list.
  u32* lrow_g = b.cand_row + cs;
  u32* ldig = b.row_dig + cs;
  u32 lbase = 0;  // the list's length (uniform)
  // pre-step scalars: CTA 0 rewrites *sc after the grid barrier
  const i64 sc_total = sc->total_blocks, sc_free = sc->free_blocks;
  const double sc_usage = sc->kv_usage_ratio;
  const double ema = sc->has_ema_tool ? sc->ema_tool : c.tool_prior;
  // The most blocks one plan can allocate: a block per decode slot plus the
  // prefill chunks' blocks (sum of grants <= budget, one partial block per
  // grant).  With that many blocks free before the step (expiry only adds to
  // them) no claim can fail, the reclaimer never runs and the step needs no
  // victim stream: the scan skips the victim digits and candidates.
  const i64 alloc_bound = (i64)c.max_dec + ((i64)c.budget + c.bs - 1) / c.bs + c.window + 1;
  const bool vic_on = sc_free < alloc_bound;

  long long exp_blocks = 0;
  int n_active = 0, n_queued = 0, n_long = 0, n_ready = 0, n_prom = 0, n_vic = 0, n_bnd = 0;
  int n_exp = 0, n_qkv = 0;
  int max_req = 0, min_req = 0x7fffffff;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // pack_queue's key range (control.py:109-122) over the admission list
  // itself: CTA g reduces its slice (coalesced; the loads overlap the first
  // TMA round trip.  Folding a part per round instead -- loads in flight
  // across the row work -- was measured slower: they queue behind the ring)
  {
    const i64 qn = sc->queue_len;
    const i32* qreq = PICK2(Q.req, *qsel_p);
    const i64 q0 = qn * me / gridDim.x, q1 = qn * (me + 1) / gridDim.x;
    for (i64 i = q0 + threadIdx.x; i < q1; i += SCAN_TPB) {
      const i32 q = __ldcg(qreq + i);
      max_req = q > max_req ? q : max_req;
      min_req = q < min_req ? q : min_req;
    }
  }
  __syncthreads();
  PTIME(45);

  // ---- phase 1 ---------------------------------------------------------------
  // Running-victim digits and the window digit's f64 part are skipped once the
  // CTA's running bound already rules the row out: such a row can be neither
  // in the CTA's top-k nor in the global one, and its digit record only has to
  // stay above every threshold (DIG_ABOVE, or the level's largest digit).
  int buf = 0;
  u32 par = 0;
  for (int rd = 0; rd < nrounds; ++rd) {
    const unsigned char* B = sdyn + (size_t)buf * SB_BYTES;
    mbar_wait(&bars[buf], par);
    if (rd == 0) PTIME(46);
    const int lr = threadIdx.x;
    const i64 r = cs + (i64)rd * SCAN_R + lr;
    const bool valid = lr < (int)(ce - (cs + (i64)rd * SCAN_R));
    const u32 bw = s_bw, bv = s_bv;
    u32 rw = DIG_NONE, rv = DIG_NONE;
    bool keep = false;
    if (valid) {
      const u8 f = B[SB_FL + lr];
      const u8 ph = B[SB_PH + lr];
      if (f & MARS_F_ACTIVE) n_active++;
      if (f & MARS_F_QUEUED) {
        n_queued++;
        if (f & MARS_F_LONG) n_long++;
        if (((const i32*)(B + SB_KV))[lr] > 0) n_qkv++;
      }
      if (f & MARS_F_PINNED) {
        const double d = ((const double*)(B + SB_DL))[lr];
        const bool exp_ = d < now;
        const i32 pbk = ((const i32*)(B + SB_PB))[lr];
        if (do_exp && exp_) {
          t.flags[r] = f & ~MARS_F_PINNED;
          t.kv[r] = 0;
          if (kv_fused) {  // (rare rows: shared atomics cost nothing here)
            atomicAdd(&s_kv[0], (u32)(pbk / KV_CH + (pbk % KV_CH ? 1 : 0)));
            if (pbk % KV_CH) {
              atomicAdd(&s_kv[1], (u32)(pbk % KV_CH));
              atomicAdd(&s_kv[2], 1u);
            }
          }
          exp_blocks += pbk;
          n_exp++;
          rv = DIG_EXP;
        } else if (vic_pin && vic_on) {
          rv = pin_reclaim_digit(c.policy, !exp_, B[SB_PL + lr], pbk, d, now);
          if (rv <= bv) atomicAdd(&hv[rv], 1u);
          n_vic++;
        }
      }
      if ((f & MARS_F_ACTIVE) && (ph == MARS_PREFILL || ph == MARS_DECODE)) {
        n_ready++;
        u32 lv = B[SB_LV + lr];
        if (c.coord) {
          const u32 pr = B[SB_PR + lr];
          if (lv != 0 && pr < (u32)c.max_promos &&
              now - ((const double*)(B + SB_WS))[lr] >= c.promo_wait) {
            // promote_waiting (scheduler.py:120-127)
            lv -= 1;
            t.level[r] = (u8)lv;
            t.promos[r] = (u8)(pr + 1);
            t.ws[r] = now;
            n_prom++;
          }
        } else {
          lv = 0;
        }
        i64 sv = 0;
        if (c.policy == POL_PP) {
          sv = t.served[r];
          if (sv > 0xffffffffll) w->status |= ST_BAD_INPUT;  // outside the packed key
          rw = pp_window_digit(sv, ((const double*)(B + SB_RS))[lr], scale);
          if (rw <= bw) atomicAdd(&hw[rw], 1u);
        } else if ((lv << 10) > bw) {
          rw = (lv << 10) | 1023u;  // the level alone is above the bound
        } else {
          rw = window_digit(lv, ((const double*)(B + SB_RS))[lr], scale);
          if (rw <= bw) atomicAdd(&hw[rw], 1u);
        }
        const i32 kvv = ((const i32*)(B + SB_KV))[lr];
        if (kvv > 0 && vic_on) {
          n_vic++;
          if (bv >= (1u << 11)) {  // running digits start at 1 << 11
            rv = run_reclaim_digit(c.policy, lv, held_blocks(c, kvv),
                                   ((const double*)(B + SB_RS))[lr], sv, ascale);
            if (rv <= bv) atomicAdd(&hv[rv], 1u);
          } else {
            rv = DIG_ABOVE;
          }
        }
      }
      if ((f & MARS_F_BOUNDARY) && ret_on) {
        n_bnd++;
        rw |= DIG_BND;
      }
      keep = ((rw & ~DIG_BND) <= bw) || rv <= bv || (rw & DIG_BND) || rv == DIG_EXP;
    }
    const u32 kbal = __ballot_sync(FULL, keep);
    // (per-warp counts double-buffered by round parity: a warp may run one
    // round ahead -- there is no barrier at a round's end -- but not two)
    u32* wc_ = s_wc + (rd & 1) * 32;
    if (lane == 0) wc_[wid] = __popc(kbal);
    if (++buf == SCAN_NBUF) {
      buf = 0;
      par ^= 1u;
    }
    // every thread is done with this round's buffer: refill it
    __syncthreads();
    if (rd == 0) PTIME(47);
    {  // append the kept rows at their row-order positions
      const u32 cw = lane < SCAN_TPB / 32 ? wc_[lane] : 0u;
      const u32 before = __reduce_add_sync(FULL, lane < wid ? cw : 0u);
      const u32 tot = __reduce_add_sync(FULL, cw);
      if (keep) {
        const u32 k = lbase + before + __popc(kbal & ((1u << lane) - 1u));
        lrow_g[k] = (u32)r;
        ldig[k] = rw | (rv << 16);
      }
      lbase += tot;
    }
    if (threadIdx.x == 0 && rd + SCAN_NBUF < nrounds) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(rd + SCAN_NBUF);
    }
    // tighten the histogram bounds to the CTA's running top-k bins (the
    // only rounds that end at a barrier: the next round reads the bounds)
    if (rd == 0) PTIME(59);
    if ((rd == 0 || rd == 2) && rd + 1 < nrounds) {
      int tw, tv;
      u32 up, upv;
      block_threshold_pair(hw, (u32)c.window, hv, (u32)VSEL, wsum, &tw, &up, &tv, &upv);
      if (threadIdx.x == 0) {
        s_bw = (u32)tw;
        s_bv = (u32)tv;
      }
      __syncthreads();
    }
    if (rd < 7) PTIME(25 + rd);
  }
  __syncthreads();

  // local thresholds: only bins at or below them can hold a global top-k key
  {
    int tw, tv;
    u32 up;
    u32 upv;
    block_threshold_pair(hw, (u32)c.window, hv, (u32)VSEL, wsum, &tw, &up, &tv, &upv);
    for (int i = threadIdx.x; i <= tw; i += blockDim.x)
      if (hw[i]) atomicAdd(&w->hist_win[i], hw[i]);
    for (int i = threadIdx.x; i <= tv; i += blockDim.x)
      if (hv[i]) atomicAdd(&w->hist_vic[i], hv[i]);
    if (threadIdx.x == 0) {
      atomicMin(&w->tmin_win, (u32)tw);
      atomicMin(&w->tmin_vic, (u32)tv);
    }
  }

  // counters: warp shuffles, then one shared and one global atomic per warp/CTA
  {
    __shared__ int s_cnt[11];
    __shared__ unsigned long long s_eb;
    if (threadIdx.x < 11) s_cnt[threadIdx.x] = (threadIdx.x == 8) ? 0x7fffffff : 0;
    if (threadIdx.x == 0) s_eb = 0;
    __syncthreads();
    unsigned long long eb = warp_sum<unsigned long long>((unsigned long long)exp_blocks);
    u32 v[9] = {(u32)n_active, (u32)n_queued, (u32)n_long, (u32)n_ready, (u32)n_prom,
                (u32)n_vic,    (u32)n_bnd,    (u32)n_exp,  (u32)n_qkv};
#pragma unroll
    for (int q = 0; q < 9; ++q) v[q] = __reduce_add_sync(FULL, v[q]);
    int mx = __reduce_max_sync(FULL, max_req), mn = __reduce_min_sync(FULL, min_req);
    if (lane == 0) {
      if (eb) atomicAdd(&s_eb, eb);
#pragma unroll
      for (int q = 0; q < 7; ++q)
        if (v[q]) atomicAdd(&s_cnt[q], (int)v[q]);
      if (v[7]) atomicAdd(&s_cnt[9], (int)v[7]);
      if (v[8]) atomicAdd(&s_cnt[10], (int)v[8]);
      atomicMax(&s_cnt[7], mx);
      atomicMin(&s_cnt[8], mn);
    }
    __syncthreads();
    if (threadIdx.x < 3 && kv_fused) b.tile_kv[3 * me + threadIdx.x] = (i64)s_kv[threadIdx.x];
    if (threadIdx.x == 0) {
      b.tile_cnt[me] = s_cnt[9];
      atomicAdd(&w->exp_blocks, s_eb);
      atomicAdd(&w->n_active, s_cnt[0]);
      atomicAdd(&w->n_queued, s_cnt[1]);
      atomicAdd(&w->n_long_q, s_cnt[2]);
      atomicAdd(&w->n_ready, s_cnt[3]);
      atomicAdd(&w->n_promoted, s_cnt[4]);
      atomicAdd(&w->n_victims, s_cnt[5]);
      atomicAdd(&w->n_boundary, s_cnt[6]);
      atomicMax(&w->max_req, s_cnt[7]);
      atomicMin(&w->min_req, s_cnt[8]);
      if (s_cnt[10]) atomicAdd(&w->n_queued_kv, s_cnt[10]);
    }
  }

  PTIME(1);
  grid.sync();
  PTIME(2);
  // the kernel after the scan (S5's expired-table push, launched as a
  // programmatic dependent) may become resident now and wait for this grid
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // ---- phase 2 ---------------------------------------------------------------
  // Every load that does not depend on another is issued at once: the CTA
  // thresholds' minimum, the expiry totals and, speculatively, the low half of
  // both merged histograms (the thresholds almost always fall there: the
  // window top-k sits at level 0, the victim top-k among the pinned rows).
  const u32 tmw = __ldcg(&w->tmin_win), tmv = __ldcg(&w->tmin_vic);
  const int tile_cnt_g = (int)threadIdx.x < (int)gridDim.x ? __ldcg(&b.tile_cnt[threadIdx.x]) : 0;
  long long tkv[3] = {0, 0, 0};  // S5 (kv_fused): CTA t's sums, in flight with the rest
  if (kv_fused && (int)threadIdx.x < (int)gridDim.x)
#pragma unroll
    for (int q = 0; q < 3; ++q) tkv[q] = __ldcg(&b.tile_kv[3 * threadIdx.x + q]);
  const unsigned long long exp_total = __ldcg(&w->exp_blocks);
  {
    constexpr int HALF = HIST_BINS / 2 / SCAN_TPB;
    u32 xw[HALF], xv[HALF];
#pragma unroll
    for (int q = 0; q < HALF; ++q) {
      xw[q] = __ldcg(&w->hist_win[q * SCAN_TPB + threadIdx.x]);
      xv[q] = __ldcg(&w->hist_vic[q * SCAN_TPB + threadIdx.x]);
    }
#pragma unroll
    for (int q = 0; q < HIST_BINS / SCAN_TPB; ++q) {
      const int i = q * SCAN_TPB + threadIdx.x;
      if (q < HALF) {
        hw[i] = (i <= (int)tmw) ? xw[q] : 0u;
        hv[i] = (i <= (int)tmv) ? xv[q] : 0u;
      } else {
        hw[i] = (i <= (int)tmw) ? __ldcg(&w->hist_win[i]) : 0u;
        hv[i] = (i <= (int)tmv) ? __ldcg(&w->hist_vic[i]) : 0u;
      }
    }
  }
  __syncthreads();
  int gw, gv;
  u32 wu, vu;
  block_threshold_pair(hw, (u32)c.window, hv, (u32)VSEL, wsum, &gw, &wu, &gv, &vu);
  if (gw > (int)tmw) gw = (int)tmw;
  if (gv > (int)tmv) gv = (int)tmv;
  // lists the digits cannot cut down to about their target (every CTA derives
  // the same answer from the merged histogram): refined in phase 3
  const bool ref_w = wu > (u32)max(c.ref_trig_w, c.window);
  const bool ref_v = vu > (u32)max(c.ref_trig_v, VSEL);

  // the probe's view after the expiry evictions (telemetry.py:152-158): the
  // usage S2 prices retention with
  const i64 freeb = sc_free + (i64)exp_total;
  const double usage =
      (mode & MARS_MODE_SKIP_PROBE) ? sc_usage : (double)(sc_total - freeb) / (double)sc_total;

  // this CTA's expired pins go after those of the CTAs before it: CTA order
  // is row order, so the list is row-ordered -- already the rank order
  // expired_pins() sorts by when the table is rank-ordered
  // (baselines.py:396-399)
  int n_exp_all, exp_off;
  {
    __shared__ int s_b[32], s_a[32];
    const int cg_ = tile_cnt_g;  // gridDim.x <= SCAN_TPB (host-checked)
    const int bs = __reduce_add_sync(FULL, (int)threadIdx.x < me ? cg_ : 0);
    const int as = __reduce_add_sync(FULL, cg_);
    if (lane == 0) {
      s_b[wid] = bs;
      s_a[wid] = as;
    }
    __syncthreads();
    const int nw = SCAN_TPB / 32;
    exp_off = __reduce_add_sync(FULL, lane < nw ? s_b[lane] : 0);
    n_exp_all = __reduce_add_sync(FULL, lane < nw ? s_a[lane] : 0);
  }
  PTIME(3);

  // candidates at the exact thresholds, S2 retention of boundary rows and the
  // expired pins, from the digit record.  Each thread owns a contiguous run of
  // rows (thread order == row order, as the expired list needs):
  // (A) per-thread counts, one block scan -> CTA-local list offsets; thread 0
  //     issues the global list reservations (their results are first needed
  //     in (D), so the atomics' round trip overlaps (C));
  // (B) the row ids into CTA-local lists (shared memory, the free TMA ring);
  // (C) one thread per entry gathers its row's columns and stages the record;
  // (D) the records and row ids go to the global lists.
  // A CTA with more entries than the staging area holds takes the unstaged
  // path (row ids straight to the global lists, re-read for the gathers).
  {
    __shared__ unsigned long long s_scan[32];
    __shared__ u32 s_escan[32];
    __shared__ int s_base[3], s_tot[4];
    // The compacted list over the warps: warp w owns the entries
    // [w*S, (w+1)*S), read 32 consecutive entries at a time (coalesced), so
    // warp order is row order.
    const i64 len = lbase;
    const i64 per = (len + SCAN_TPB - 1) / SCAN_TPB;
    const i64 r0 = (i64)wid * per * 32 + lane;
    const i64 rlim = (i64)(wid + 1) * per * 32;
    const i64 r1 = rlim < len ? rlim : len;
    const i64 step = 32;
    constexpr int FB = 21;  // count field width (chunk < 2^21 rows)
    constexpr unsigned long long FM = (1ull << FB) - 1;
    unsigned long long cnt = 0;
    u32 ecnt = 0;
    for (i64 i = r0; i < r1; i += step) {
      const u32 rc = ldig[i];
      const u32 rw = rc & 0xffffu, rv = rc >> 16;
      cnt += ((rw & ~DIG_BND) <= (u32)gw ? 1ull : 0ull) + ((rv <= (u32)gv ? 1ull : 0ull) << FB) +
             ((rw & DIG_BND) ? (1ull << (2 * FB)) : 0ull);
      ecnt += rv == DIG_EXP ? 1u : 0u;
    }
    // warp totals (lane 31's inclusive value; fields never carry: each < 2^21)
    unsigned long long incl = cnt;
    u32 eincl = ecnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long x = __shfl_up_sync(FULL, incl, o);
      const u32 y = __shfl_up_sync(FULL, eincl, o);
      if (lane >= o) {
        incl += x;
        eincl += y;
      }
    }
    if (lane == 31) {
      s_scan[wid] = incl;
      s_escan[wid] = eincl;
    }
    __syncthreads();
    if (wid == 0) {
      unsigned long long v = lane < SCAN_TPB / 32 ? s_scan[lane] : 0ull;
      u32 e = lane < SCAN_TPB / 32 ? s_escan[lane] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long x = __shfl_up_sync(FULL, v, o);
        const u32 y = __shfl_up_sync(FULL, e, o);
        if (lane >= o) {
          v += x;
          e += y;
        }
      }
      s_scan[lane] = v;  // inclusive over warps
      s_escan[lane] = e;
      if (lane == 31) {
        s_tot[0] = (int)(v & FM);
        s_tot[1] = (int)((v >> FB) & FM);
        s_tot[2] = (int)(v >> (2 * FB));
        s_tot[3] = (int)e;
      }
    }
    __syncthreads();
    const int nw = s_tot[0], nv = s_tot[1], nb = s_tot[2], ne = s_tot[3];
    const int ntot = nw + nv + nb + ne;
    const bool ro = (mode & MARS_MODE_RANK_ORDERED) != 0;
    u32* exp_rows = ro ? b.exp_row_sorted : b.exp_row;
    // staging: CTA-local row lists (4 B), their digit records (4 B) and one
    // 48-byte record per entry
    constexpr int STAGE_REC = 48;
    const size_t lrow_bytes = ((size_t)ntot * 8 + 15) & ~(size_t)15;
    const bool staged =
        !no_stage && lrow_bytes + (size_t)ntot * STAGE_REC <= (size_t)SCAN_NBUF * SB_BYTES;
    u32* lrow = (u32*)sdyn;                                       // [ntot]
    u32* lrec = lrow + ntot;                                      // [ntot]
    unsigned char* rec = sdyn + lrow_bytes;                       // [ntot][48]
    // (A') global list reservations, issued now, consumed in (D)
    int gb0 = 0, gb1 = 0, gb2 = 0;
    if (threadIdx.x == 0) {
      gb0 = nw ? atomicAdd(&w->n_wc, nw) : 0;
      gb1 = nv ? atomicAdd(&w->n_vc, nv) : 0;
      gb2 = nb ? atomicAdd(&w->n_ret, nb) : 0;
      if (!staged) {
        s_base[0] = gb0;
        s_base[1] = gb1;
        s_base[2] = gb2;
      }
    }
    if (!staged) __syncthreads();
    PTIME(40);
    // (B) row ids: local lists (staged) or the global lists
    const unsigned long long wtot = __shfl_sync(FULL, incl, 31);
    const u32 wetot = __shfl_sync(FULL, eincl, 31);
    if ((wtot | wetot) != 0) {
      const unsigned long long ex = wid ? s_scan[wid - 1] : 0ull;
      int pw = (int)(ex & FM), pv = nw + (int)((ex >> FB) & FM);
      int pr = nw + nv + (int)(ex >> (2 * FB));
      int pe = nw + nv + nb + (int)(wid ? s_escan[wid - 1] : 0u);
      u32* ow = lrow;
      u32* ov = lrow;
      u32* orr = lrow;
      u32* oe = lrow;
      if (!staged) {
        pw += s_base[0];
        pv += s_base[1] - nw;
        pr += s_base[2] - nw - nv;
        pe += exp_off - nw - nv - nb;
        ow = b.wc_row;
        ov = b.vc_row;
        orr = b.ret_row;
        oe = exp_rows;
      }
      {  // 32 consecutive entries per ballot, lane order = row order
        const u32 lt = (1u << lane) - 1u;
        for (i64 c0 = r0 - lane; c0 < r1; c0 += 32) {
          const i64 i = c0 + lane;
          const u32 rc = i < r1 ? ldig[i] : (DIG_NONE | (DIG_NONE << 16));
          const u32 rw = rc & 0xffffu, rv = rc >> 16;
          const u32 r = i < r1 ? lrow_g[i] : 0u;
          const bool qw = (rw & ~DIG_BND) <= (u32)gw, qv = rv <= (u32)gv;
          const bool qb = (rw & DIG_BND) != 0, qe = rv == DIG_EXP;
          const u32 mw = __ballot_sync(FULL, qw), mv = __ballot_sync(FULL, qv);
          const u32 mb = __ballot_sync(FULL, qb), me_ = __ballot_sync(FULL, qe);
          if (qw) {
            ow[pw + __popc(mw & lt)] = r;
            if (staged) lrec[pw + __popc(mw & lt)] = rc;
          }
          if (qv) {
            ov[pv + __popc(mv & lt)] = r;
            if (staged) lrec[pv + __popc(mv & lt)] = rc;
          }
          if (qb) orr[pr + __popc(mb & lt)] = r;
          if (qe) oe[pe + __popc(me_ & lt)] = r;
          pw += __popc(mw);
          pv += __popc(mv);
          pr += __popc(mb);
          pe += __popc(me_);
        }
      }
    }
    __syncthreads();
    PTIME(41);
    // (C) gathers; staged: records in shared memory, else straight to global
    for (int k = threadIdx.x; k < ntot; k += blockDim.x) {
      u32 r;
      if (staged) {
        r = lrow[k];
      } else if (k < nw) {
        r = __ldcg(&b.wc_row[s_base[0] + k]);
      } else if (k < nw + nv) {
        r = __ldcg(&b.vc_row[s_base[1] + k - nw]);
      } else if (k < nw + nv + nb) {
        r = __ldcg(&b.ret_row[s_base[2] + k - nw - nv]);
      } else {
        r = __ldcg(&exp_rows[exp_off + k - nw - nv - nb]);
      }
      unsigned char* R = rec + (size_t)k * STAGE_REC;
      if (k < nw + nv) {
        const bool is_w = k < nw;
        // a ready row (window digit computed) or, for a victim, a pin
        bool ready;
        if (staged) {
          ready = (lrec[k] & DIG_NONE) == 0;
        } else {
          const u8 fl = t.flags[r], ph = t.phase[r];
          ready = (fl & MARS_F_ACTIVE) && (ph == MARS_PREFILL || ph == MARS_DECODE);
        }
        const u32 rk = t.rank[r];
        u64 whi = 0, wlo = 0;
        u32 lv = 0;
        double arr = 0.0;
        i64 sv = 0;
        if (ready) {  // post-aging level
          if (c.policy == POL_PP) {
            sv = t.served[r];
            arr = t.arr[r];
            pp_window_key(sv, arr, rk, whi, wlo);
          } else {
            lv = c.coord ? (u32)t.level[r] : 0u;
            arr = c.coord ? t.rs[r] : t.arr[r];
            window_key(lv, arr, rk, whi, wlo);
          }
        }
        if (is_w) {
          if (staged) {
            ((u64*)R)[0] = whi;
            ((u64*)R)[1] = wlo;
          } else {
            b.wc_hi[s_base[0] + k] = whi;
            b.wc_lo[s_base[0] + k] = wlo;
          }
        } else {
          u64 vk, vkl;
          i32 blk;
          if (ready) {
            const i64 h = held_blocks(c, t.kv[r]);
            run_reclaim_key(c.policy, lv, h, arr, sv, rk, vk, vkl);
            blk = (i32)h;
          } else {  // pinned row
            const double dl = t.dl[r];
            const i32 pbk = t.pb[r];
            pin_reclaim_key(c.policy, !(dl < now), (u32)t.plevel[r], pbk, dl, rk, vk, vkl);
            blk = pbk;
          }
          if (staged) {
            ((u64*)R)[0] = vk;
            ((u64*)R)[1] = vkl;
            ((u64*)R)[2] = whi;
            ((u64*)R)[3] = wlo;
            ((i32*)R)[8] = blk;
          } else {
            const int slot = s_base[1] + k - nw;
            b.vc_key[slot] = vk;
            b.vc_kl[slot] = vkl;
            b.vc_whi[slot] = whi;
            b.vc_wlo[slot] = wlo;
            b.vc_blk[slot] = blk;
          }
        }
      } else if (k < nw + nv + nb) {
        u8 pin;
        double rb_, rc_, rd_;
        decide_retention(c, t.ctx[r], t.kv[r], sc_total, usage, ema, now, pin, rb_, rc_, rd_);
        if (staged) {
          ((double*)R)[0] = rb_;
          ((double*)R)[1] = rc_;
          ((double*)R)[2] = rd_;
          R[24] = pin;
        } else {
          const int slot = s_base[2] + k - nw - nv;
          b.ret_pin[slot] = pin;
          b.ret_b[slot] = rb_;
          b.ret_c[slot] = rc_;
          b.ret_d[slot] = rd_;
        }
      } else {  // expired pin: its blocks (and rank, for the rank sort)
        const int slot = exp_off + k - nw - nv - nb;
        if (ro) {
          b.exp_blk_sorted[slot] = t.pb[r];
        } else {
          b.exp_blk[slot] = t.pb[r];
          b.exp_rank[slot] = t.rank[r];
        }
        if (staged) exp_rows[slot] = r;
      }
    }
    if (staged) {
      if (threadIdx.x == 0) {  // the reservations' results, first use
        s_base[0] = gb0;
        s_base[1] = gb1;
        s_base[2] = gb2;
      }
      __syncthreads();
      PTIME(42);
      // (D) staged records and row ids -> the global lists
      const int bw = s_base[0], bv = s_base[1], bb = s_base[2];
      for (int k = threadIdx.x; k < nw + nv + nb; k += blockDim.x) {
        const u32 r = lrow[k];
        const unsigned char* R = rec + (size_t)k * STAGE_REC;
        if (k < nw) {
          b.wc_row[bw + k] = r;
          b.wc_hi[bw + k] = ((const u64*)R)[0];
          b.wc_lo[bw + k] = ((const u64*)R)[1];
        } else if (k < nw + nv) {
          const int slot = bv + k - nw;
          b.vc_row[slot] = r;
          b.vc_key[slot] = ((const u64*)R)[0];
          b.vc_kl[slot] = ((const u64*)R)[1];
          b.vc_whi[slot] = ((const u64*)R)[2];
          b.vc_wlo[slot] = ((const u64*)R)[3];
          b.vc_blk[slot] = ((const i32*)R)[8];
        } else {
          const int slot = bb + k - nw - nv;
          b.ret_row[slot] = r;
          b.ret_b[slot] = ((const double*)R)[0];
          b.ret_c[slot] = ((const double*)R)[1];
          b.ret_d[slot] = ((const double*)R)[2];
          b.ret_pin[slot] = R[24];
        }
      }
    }
  }

  // S5 (kv_fused): per expired table, in row order (= rank order, the order
  // expired_pins() evicts them, baselines.py:396-399), its segment / loose-ID
  // / tail-chunk positions on the free stack (prefix over the CTAs before it
  // and a block scan): k_kv_exp_push's inputs, no separate scan kernel.  CTA
  // 0 moves the stack scalars.  The lengths are the pinned blocks (a pin
  // moves the whole table) gathered above.
  if (kv_fused) {
    // this CTA's bases (sums over the CTAs before it) and the totals
    __shared__ long long s_kr[6][32];
    __shared__ i64 s_kb[3], s_kt[3];
    {
      long long v[6];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        v[q] = warp_sum<long long>((int)threadIdx.x < me ? tkv[q] : 0ll);
        v[3 + q] = warp_sum<long long>(tkv[q]);
      }
      if (lane == 0)
#pragma unroll
        for (int q = 0; q < 6; ++q) s_kr[q][wid] = v[q];
      __syncthreads();
      if (wid == 0) {
#pragma unroll
        for (int q = 0; q < 6; ++q) {
          const long long x = warp_sum<long long>(lane < SCAN_TPB / 32 ? s_kr[q][lane] : 0ll);
          if (lane == 0) {
            if (q < 3) s_kb[q] = x; else s_kt[q - 3] = x;
          }
        }
      }
      __syncthreads();
    }
    i64 so = s_kb[0], ao = s_kb[1], ro = s_kb[2];
    const bool kv_room = s_kvb[0] + s_kt[0] <= kv.seg_cap;  // (else: status 32, no frees)
    const int ne_cta = kv_room ? __ldcg(&b.tile_cnt[me]) : 0;
    for (int e0 = 0; e0 < ne_cta; e0 += SCAN_TPB) {
      const int e = e0 + (int)threadIdx.x;
      i64 L = 0;
      if (e < ne_cta) L = __ldcg(&b.exp_blk_sorted[exp_off + e]);
      // one scan of the three fields packed 21 bits apart (a 1024-table chunk
      // sums to < 2^21 in each: <= 8K blocks per table)
      constexpr int KB = 21;
      constexpr long long KM = (1ll << KB) - 1;
      const long long pk = (L / KV_CH + (L % KV_CH ? 1 : 0)) | ((L % KV_CH) << KB) |
                           ((long long)(L % KV_CH ? 1 : 0) << (2 * KB));
      long long tot;
      const long long x = block_excl_scan_i64(pk, &tot);
      if (e < ne_cta) {  // absolute positions on the stack / arena / chunk pool
        kv.xoff[exp_off + e] = s_kvb[0] + so + (x & KM);
        kv.xaoff[exp_off + e] = s_kvb[1] + ao + ((x >> KB) & KM);
        kv.xroff[exp_off + e] = s_kvb[2] + ro + (x >> (2 * KB));
      }
      so += tot & KM;
      ao += (tot >> KB) & KM;
      ro += tot >> (2 * KB);
    }
    if (me == 0 && threadIdx.x == 0) {
      kv.xbase[1] = kv_room ? 1 : -1;  // k_kv_exp_push: offsets absolute (or overflow)
      kv.xbase[0] = kv.xbase[2] = kv.xbase[3] = 0;
      if (!kv_room) {
        atomicOr(&kv.s->status, 32);
      } else {
        kv.s->seg_top = s_kvb[0] + s_kt[0];
        kv.s->arena_top = s_kvb[1] + s_kt[1];
        kv.s->cfs_top = s_kvb[2] + s_kt[2];
        kv.s->fs_ids += (i64)exp_total;
      }
    }
  }

  // ---- phase 3: grid radix refinement (only when a candidate list is much
  // longer than its target: coarse digits over tied keys, or huge tables)
  // the victim list (when the step may reclaim) is ranked grid-wide into the
  // walk's stream order, so the single-CTA walk does not sort it
  const bool vsort = vic_on && vu > 0u;
  if (ref_w || ref_v || vsort) {
    grid.sync();
    PTIME(43);
    if (ref_w || ref_v) grid_refine(grid, w, b, ref_w, ref_v, (int)c.window, VSEL);
    PTIME(44);
    if (vsort) {
      if (ref_v) grid.sync();  // the refined list is complete
      grid_rank_victims(w, b, ref_v, c.stream_cap, (u64*)sdyn);
    }
  }

  PTIME(4);
  if (me != 0 || threadIdx.x != 0) return;
  // ---- CTA 0: scalar epilogue on register copies: one burst of independent
  // loads in, plain stores out (no dependent global round trips)
  mars_scalars s;
  {
    const unsigned long long* src = (const unsigned long long*)sc;
    unsigned long long* dst = (unsigned long long*)&s;
#pragma unroll
    for (int q = 0; q < (int)(sizeof(mars_scalars) / 8); ++q) dst[q] = __ldcg(src + q);
  }
  const int n_active_all = __ldcg(&w->n_active), n_queued_all = __ldcg(&w->n_queued);
  const int n_long_all = __ldcg(&w->n_long_q), mx_all = __ldcg(&w->max_req);
  const int mn_all = __ldcg(&w->min_req);
  const mars_step_in in = w->in;
  w->t_win = gw;
  w->t_vic = gv;
  w->vic_on = vic_on ? 1 : 0;
  w->n_win_cand_expected = (i32)wu;
  w->n_vic_cand_expected = (i32)vu;
  w->n_exp = n_exp_all;
  const i64 total = s.total_blocks;
  s.free_blocks = freeb;
  w->free_after_expiry = freeb;
  if (!(mode & MARS_MODE_SKIP_PROBE)) {
    // Telemetry.probe (telemetry.py:152-158) after the expiry evictions
    s.available_kv = freeb;
    s.kv_usage_ratio = usage;
    s.active_sessions = n_active_all;
    s.active_tools = in.active_tools;
    s.queued_tools = in.queued_tools;
  }
  const i64 qlen = s.queue_len;
  w->qlen = qlen;
  if (!(mode & MARS_MODE_NO_ROWS) && (i64)n_queued_all != qlen) w->status |= ST_QUEUE_MISMATCH;
  // what the control plane sees: this replica's probe (pooled in sharded mode,
  // see k_global_control)
  w->adm_avail = s.available_kv;
  w->adm_total = total;
  w->adm_usage = s.kv_usage_ratio;
  w->adm_active = s.active_sessions;
  if (mode & MARS_MODE_SHARDED) {
    xc[0] = s.available_kv;
    xc[1] = total;
    xc[2] = s.active_sessions;
    xc[3] = s.queue_len;
  } else if (in.control_due && !(mode & MARS_MODE_SKIP_REFRESH)) {
    refresh_pressure(c, &s, in.worker_slots, s.kv_usage_ratio);
  }
  {
    const unsigned long long* src = (const unsigned long long*)&s;
    unsigned long long* dst = (unsigned long long*)sc;
#pragma unroll
    for (int q = 0; q < (int)(sizeof(mars_scalars) / 8); ++q) dst[q] = src[q];
  }
  w->xlsd_big = n_exp_all > SORT_CAP ? 1 : 0;
  w->xlsd_n = n_exp_all;
  w->xlsd_maxkey = 0xffffffffull;
  // table-backed queue statistics for pack_queue (control.py:109-122)
  w->tab_long_q = n_long_all;
  w->tab_max_req = mx_all;
  w->tab_min_req = mn_all;
}

// ---------------------------------------------------------------------------
// single-CTA bitonic sort in shared memory: keys (hi, lo) + u32 payload
// ---------------------------------------------------------------------------

__device__ void bitonic_sort(u64* kh, u64* kl, u32* pv, int n2) {
  for (int k = 2; k <= n2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        int p = i ^ j;
        if (p > i) {
          bool up = (i & k) == 0;
          u64 ah = kh[i], al = kl[i], bh = kh[p], bl = kl[p];
          bool gt = key_lt(bh, bl, ah, al);
          if (gt == up) {
            kh[i] = bh;
            kl[i] = bl;
            kh[p] = ah;
            kl[p] = al;
            u32 tv = pv[i];
            pv[i] = pv[p];
            pv[p] = tv;
          }
        }
      }
      __syncthreads();
    }
  }
}

__device__ __forceinline__ int next_pow2(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

// ---------------------------------------------------------------------------
// generic multi-CTA stable LSD radix sort (u64 keys, u32 values, 8-bit digits)
#define LSD_SEG_J (PACK_SEG_ENTRIES / 1024)  // entries per lane of the warp-segment ranking
#define LSD_B 4  // entries per lane per batch of a long chunk's scatter
// control words live in Work (queue: lsd_*, expired: xlsd_*)
// ---------------------------------------------------------------------------

struct LsdView {
  i32* cur;
  i32* skip;
  i32* in;
  u64* maxkey;
  i32* big;
  i32* n;
};

__device__ __forceinline__ LsdView lsd_view(Work* w, int which) {
  LsdView v;
  if (which == 0) {
    v.cur = &w->lsd_cur; v.skip = w->lsd_skip; v.in = w->lsd_in; v.maxkey = &w->lsd_maxkey;
    v.big = &w->lsd_big; v.n = &w->lsd_n;
  } else {
    v.cur = &w->xlsd_cur; v.skip = w->xlsd_skip; v.in = w->xlsd_in; v.maxkey = &w->xlsd_maxkey;
    v.big = &w->xlsd_big; v.n = &w->xlsd_n;
  }
  return v;
}

// One cooperative launch sorts the whole list: per 8-bit pass, chunk
// histograms -> grid barrier -> every CTA derives its own digit offsets from
// all chunk counts (no separate scan launch) -> stable in-order scatter ->
// grid barrier.  Grid <= #SMs, one 1024-thread CTA per SM (co-resident).
// what one grid-wide sort works on (read by every CTA, never from memory
// another CTA may still be writing)
struct LsdArgs {
  int n;
  u64 maxkey;
  const i32* raw;  // the queue's first pass reads req[] straight from the list
  bool asc;        // key = req (ascending pack) or max_req - req (descending)
  i32 mr;
  int cur;
};

__device__ LsdArgs lsd_args_from(Work* w, int which) {
  LsdView v = lsd_view(w, which);
  LsdArgs a;
  a.n = *v.n;
  a.maxkey = *v.maxkey;
  a.raw = (which == 0) ? (const i32*)(uintptr_t)w->lsd_raw_ptr : nullptr;
  a.asc = w->pack_mode == PACK_ASC;
  a.mr = w->max_req;
  a.cur = *v.cur;
  return a;
}

// Returns the buffer holding the sorted values (every CTA; CTA 0 also
// publishes it).  wc: 32 x 256 u32 of (dynamic) shared memory.
// SEG: compile the warp-segment ranking for mid-size chunks (the grids with
// few CTAs: k_pack, the expired-pin sort); k_control's wide grid keeps <= 1K
// entries per CTA and stays lean on registers without it.
template <bool SEG>
__device__ int lsd_grid_sort(Lsd L, LsdView v, LsdArgs a, int npass, u32 (*wc)[256]) {
  PTIME(5);
  cg::grid_group grid = cg::this_grid();
  const int n = a.n;
  const u64 maxkey = a.maxkey;
  const int G = gridDim.x, me = blockIdx.x;
  const int chunk = (n + G - 1) / G;
  const int s = me * chunk, e = min(n, s + chunk);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int d = tid & 255, p = tid >> 8;
  __shared__ u32 h[256], off[256], tt[256];
  __shared__ u32 part[4][256], below[4][256];
  const i32* raw = a.raw;
  const bool asc = a.asc;
  const i32 mr = a.mr;
  // the current buffer is block-uniform: kept in shared memory (a register
  // for it across the passes' grid barriers spilled to local memory)
  __shared__ int s_cur;
  if (tid == 0) s_cur = a.cur;
  __syncthreads();
  for (int pass = 0; pass < npass; ++pass) {
    const int shift = 8 * pass;
    if (pass > 0 && (maxkey >> shift) == 0) {
      if (me == 0 && tid == 0) v.skip[pass] = 1;
      continue;
    }
    // the queue's first pass reads req[] straight from the admission list
    const bool rawp = raw != nullptr && pass == 0;
    const int cur = s_cur;
    const u64* kin = PICK2(L.k, cur);
    const u32* vin = PICK2(L.v, cur);
    u64* kout = PICK2(L.k, 1 - cur);
    u32* vout = PICK2(L.v, 1 - cur);
    // a chunk of <= 1024 entries (the usual case) stays in registers from
    // the histogram to the scatter: one load per entry per pass
    const bool one = e - s <= 1024;
    // chunks up to LSD_SEG_J x 1024 entries: warp w ranks the contiguous
    // segment [s + w*S, s + (w+1)*S) 32 entries at a time with match_any and
    // running per-warp digit counts, all in registers -- one column scan over
    // the warps per pass instead of one per 1024-entry batch, and the CTA
    // histogram falls out of the warp counts
    const bool seg = SEG && !one && e - s <= LSD_SEG_J * 1024;
    u64 k1 = 0;
    u32 v1 = 0;
    const bool has1 = one && s + tid < e;
    if (has1) {
      const int i = s + tid;
      k1 = rawp ? (u64)(asc ? raw[i] : mr - raw[i]) : kin[i];
      v1 = rawp ? (u32)i : vin[i];
    }
    u64 sk[LSD_SEG_J];
    u32 sv[LSD_SEG_J], sr[LSD_SEG_J];  // sr: digit << 16 | rank in the warp (0xffffffff: none)
    if (seg) {
      for (int q = p; q < 32; q += 4) wc[q][d] = 0;
      __syncthreads();
      const int S = (((e - s) + 31) / 32 + 31) & ~31;
      const int ws = s + wid * S, we = min(e, ws + S);
      // every load in flight before the first rank (the ranking's warp
      // syncs would otherwise serialise one memory round trip per batch)
#pragma unroll
      for (int j = 0; j < LSD_SEG_J; ++j) {
        const int i = ws + j * 32 + lane;
        sk[j] = 0;
        sv[j] = 0;
        if (i < we) {
          sk[j] = rawp ? (u64)(asc ? raw[i] : mr - raw[i]) : kin[i];
          sv[j] = rawp ? (u32)i : vin[i];
        }
      }
#pragma unroll
      for (int j = 0; j < LSD_SEG_J; ++j) {
        const int i = ws + j * 32 + lane;
        const bool valid = i < we;
        const u64 k = sk[j];
        const u32 dig = valid ? (u32)((k >> shift) & 255u) : (256u + (u32)lane);
        const u32 peers = __match_any_sync(FULL, dig);
        const int leader = __ffs(peers) - 1;
        u32 base = 0;
        if (valid && lane == leader) {
          base = wc[wid][dig];
          wc[wid][dig] = base + __popc(peers);
        }
        base = __shfl_sync(FULL, base, leader);
        __syncwarp();
        sr[j] = valid ? ((dig << 16) | (base + __popc(peers & ((1u << lane) - 1u)))) : 0xffffffffu;
      }
      __syncthreads();
      if (tid < 256) {  // exclusive scan over the warps; the total is the CTA histogram
        u32 acc = 0;
        for (int q = 0; q < 32; ++q) {
          const u32 x = wc[q][tid];
          wc[q][tid] = acc;
          acc += x;
        }
        h[tid] = acc;
      }
      __syncthreads();
    } else {
      if (tid < 256) h[tid] = 0;
      __syncthreads();
      if (one) {
        if (has1) atomicAdd(&h[(k1 >> shift) & 255u], 1u);
      } else {
        for (int i = s + tid; i < e; i += 1024) {
          u64 k = rawp ? (u64)(asc ? raw[i] : mr - raw[i]) : kin[i];
          atomicAdd(&h[(k >> shift) & 255u], 1u);
        }
      }
      __syncthreads();
    }
    if (tid < 256) L.cnt[me * 256 + tid] = h[tid];
    if (pass == 0) PTIME(6);
    grid.sync();
    if (pass == 0) PTIME(7);
    // digit d's total over all chunks and over the chunks before mine
    const int c0 = (G * p) / 4, c1 = (G * (p + 1)) / 4;
    u32 tot = 0, bel = 0;
    for (int c = c0; c < c1; c += 32) {  // up to 32 independent L2 loads in flight
      u32 x[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) x[q] = c + q < c1 ? __ldcg(&L.cnt[(c + q) * 256 + d]) : 0u;
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        tot += x[q];
        bel += c + q < me ? x[q] : 0u;
      }
    }
    part[p][d] = tot;
    below[p][d] = bel;
    __syncthreads();
    if (tid < 32) {  // exclusive scan of the 256 digit totals, 8 per lane
      u32 x[8], sum = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        int dd = tid * 8 + q;
        x[q] = part[0][dd] + part[1][dd] + part[2][dd] + part[3][dd];
        sum += x[q];
      }
      u32 incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        u32 y = __shfl_up_sync(FULL, incl, o);
        if (tid >= o) incl += y;
      }
      u32 run = incl - sum;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        int dd = tid * 8 + q;
        off[dd] = run + below[0][dd] + below[1][dd] + below[2][dd] + below[3][dd];
        run += x[q];
      }
    }
    if (!seg)
      for (int q = p; q < 32; q += 4) wc[q][d] = 0;
    __syncthreads();
    if (pass == 0) PTIME(8);
    if (seg) {
#pragma unroll
      for (int j = 0; j < LSD_SEG_J; ++j) {
        if (sr[j] == 0xffffffffu) continue;
        const u32 dg = sr[j] >> 16;
        const u32 pos = off[dg] + wc[wid][dg] + (sr[j] & 0xffffu);
        kout[pos] = sk[j];
        vout[pos] = sv[j];
      }
    }
    if (one) {  // the chunk is in registers: one batch
      u32 dig = has1 ? (u32)((k1 >> shift) & 255u) : (256u + (u32)lane);
      u32 peers = __match_any_sync(FULL, dig);
      u32 rk = __popc(peers & ((1u << lane) - 1u));
      if (has1 && rk == 0) wc[wid][dig] = __popc(peers);
      __syncthreads();
      if (tid < 256) {
        u32 acc = 0;
        for (int q = 0; q < 32; ++q) {
          u32 x = wc[q][tid];
          wc[q][tid] = acc;
          acc += x;
        }
      }
      __syncthreads();
      if (has1) {
        u32 pos = off[dig] + wc[wid][dig] + rk;
        kout[pos] = k1;
        vout[pos] = v1;
      }
    }
    // longer chunks: batches of LSD_B x 1024 entries; warp w ranks the LSD_B
    // groups of 32 consecutive entries [base + (w*LSD_B + j)*32, ...) in order
    // with running per-warp digit counts, so one column scan over the warps
    // (and four barriers) serve 4096 entries instead of 1024
    for (int base = s; base < e && !seg && !one; base += LSD_B * 1024) {
      u64 bk[LSD_B];
      u32 bv[LSD_B], br[LSD_B];
#pragma unroll
      for (int j = 0; j < LSD_B; ++j) {  // every load in flight first
        const int i = base + (wid * LSD_B + j) * 32 + lane;
        bk[j] = 0;
        bv[j] = 0;
        if (i < e) {
          bk[j] = rawp ? (u64)(asc ? raw[i] : mr - raw[i]) : kin[i];
          bv[j] = rawp ? (u32)i : vin[i];
        }
      }
#pragma unroll
      for (int j = 0; j < LSD_B; ++j) {
        const int i = base + (wid * LSD_B + j) * 32 + lane;
        const bool valid = i < e;
        const u32 dig = valid ? (u32)((bk[j] >> shift) & 255u) : (256u + (u32)lane);
        const u32 peers = __match_any_sync(FULL, dig);
        const int leader = __ffs(peers) - 1;
        u32 b0 = 0;
        if (valid && lane == leader) {
          b0 = wc[wid][dig];
          wc[wid][dig] = b0 + __popc(peers);
        }
        b0 = __shfl_sync(FULL, b0, leader);
        __syncwarp();
        br[j] = valid ? ((dig << 16) | (b0 + __popc(peers & ((1u << lane) - 1u)))) : 0xffffffffu;
      }
      __syncthreads();
      if (tid < 256) {
        u32 acc = 0;
        for (int q = 0; q < 32; ++q) {
          u32 x = wc[q][tid];
          wc[q][tid] = acc;
          acc += x;
        }
        tt[tid] = acc;
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < LSD_B; ++j) {
        if (br[j] == 0xffffffffu) continue;
        const u32 dg = br[j] >> 16;
        const u32 pos = off[dg] + wc[wid][dg] + (br[j] & 0xffffu);
        kout[pos] = bk[j];
        vout[pos] = bv[j];
      }
      __syncthreads();
      if (tid < 256) off[tid] += tt[tid];
      for (int q = p; q < 32; q += 4) wc[q][d] = 0;
      __syncthreads();
    }
    if (me == 0 && tid == 0) {
      v.skip[pass] = 0;
      v.in[pass] = cur;
    }
    __syncthreads();  // (every thread has read s_cur)
    if (tid == 0) s_cur = 1 - cur;
    __syncthreads();
    if (pass == 0) PTIME(9);
    grid.sync();  // the next pass reads this pass' output and rewrites L.cnt
  }
  PTIME(10);
  const int cur = s_cur;
  if (me == 0 && tid == 0) *v.cur = cur;
  return cur;
}

#define LSD_WC_BYTES (32 * 256 * 4)

__global__ void __launch_bounds__(1024, 1) k_lsd_coop(Lsd L, Work* w, int which, int npass) {
  extern __shared__ __align__(16) u32 lsd_wc[];
  LsdView v = lsd_view(w, which);
  if (!*v.big) return;  // grid-uniform
  lsd_grid_sort<true>(L, v, lsd_args_from(w, which), npass, (u32(*)[256])lsd_wc);
}

static void launch_lsd(Lsd L, Work* w, int which, int npass, int grid, cudaStream_t s) {
  void* args[] = {&L, &w, &which, &npass};
  cudaLaunchCooperativeKernel((const void*)k_lsd_coop, dim3(grid), dim3(1024), args,
                              LSD_WC_BYTES, s);
}

// ---------------------------------------------------------------------------
// expired pins in rank order (side stream)
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(1024) k_exp_small(Work* w, Bufs b, Lsd L) {
  extern __shared__ __align__(16) unsigned char smem[];
  int n = w->n_exp;
  if (n > SORT_CAP) {
    // big: seed the LSD buffers (key = rank, value = index)
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      L.k[0][i] = b.exp_rank[i];
      L.v[0][i] = (u32)i;
    }
    if (threadIdx.x == 0) w->xlsd_cur = 0;
    return;
  }
  int n2 = next_pow2(n > 1 ? n : 1);
  u64* kh = (u64*)smem;
  u64* kl = kh + n2;
  u32* pv = (u32*)(kl + n2);
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    kh[i] = i < n ? (u64)b.exp_rank[i] : ~0ull;
    kl[i] = (u64)i;
    pv[i] = (u32)i;
  }
  __syncthreads();
  bitonic_sort(kh, kl, pv, n2);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    u32 j = pv[i];
    b.exp_row_sorted[i] = b.exp_row[j];
    b.exp_blk_sorted[i] = b.exp_blk[j];
  }
}

__global__ void k_exp_gather(Work* w, Bufs b, Lsd L) {
  if (!w->xlsd_big) return;
  int n = w->xlsd_n;
  int cur = w->xlsd_cur;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    u32 j = PICK2(L.v, cur)[i];
    b.exp_row_sorted[i] = b.exp_row[j];
    b.exp_blk_sorted[i] = b.exp_blk[j];
  }
}

// ---------------------------------------------------------------------------
// K_Q: pack_queue (control.py:101-122) -- small / first-fit part, one CTA
// ---------------------------------------------------------------------------

// k-th smallest (0-based) of a[0..n) by MSD radix select, one CTA
__device__ i32 cta_kth_i32(const i32* a, int n, int k, u32* hist /*256*/, u32* sh) {
  u32 prefix = 0, mask = 0;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      u32 x = (u32)a[i] ^ 0x80000000u;
      if ((x & mask) == prefix) atomicAdd(&hist[(x >> shift) & 255u], 1u);
    }
    __syncthreads();
    __shared__ int s_bin, s_k;
    if (threadIdx.x == 0) {
      u32 cum = 0;
      int bin = 255;
      for (int i = 0; i < 256; ++i) {
        if (cum + hist[i] > (u32)k) {
          bin = i;
          break;
        }
        cum += hist[i];
      }
      s_bin = bin;
      s_k = k - (int)cum;
    }
    __syncthreads();
    prefix |= ((u32)s_bin) << shift;
    mask |= 255u << shift;
    k = s_k;
    __syncthreads();
  }
  return (i32)(prefix ^ 0x80000000u);
}

// pack_queue (control.py:101-122) on one CTA: the mode, and the whole pack for
// small queues (bitonic) and the first-fit mode; big queues only set up the
// grid-wide LSD sort
__device__ void pack_small_cta(Work* w, Queue Q, Lsd L, mars_scalars* sc, i32* qsel_p, Queue G,
                               unsigned char* smem) {
  PTIME(18);
  int qlen = (int)w->qlen;
  if (qlen <= 0) return;
  const bool sharded = (w->in.mode & MARS_MODE_SHARDED) != 0;
  int sel = *qsel_p;
  const i32* req = sharded ? G.req[0] : PICK2(Q.req, sel);
  const u8* lng = sharded ? G.lng[0] : PICK2(Q.lng, sel);
  __shared__ u32 shu[1024 + 32];
  __shared__ u32 hist[256];
  __shared__ int shr[32];
  // pack_queue mode (control.py:109-122): the table scan (or the global-list
  // build) already reduced the queue; only a row-less queue is reduced here
  int all_long, mx, mn;
  if (!(w->in.mode & MARS_MODE_NO_ROWS)) {
    all_long = w->tab_long_q == qlen ? 1 : 0;
    mx = w->tab_max_req;
    mn = w->tab_min_req;
  } else {
    all_long = 1;
    mx = 0;
    mn = 0x7fffffff;
    for (int i = threadIdx.x; i < qlen; i += blockDim.x) {
      all_long &= lng[i] ? 1 : 0;
      i32 rq = req[i];
      mx = rq > mx ? rq : mx;
      mn = rq < mn ? rq : mn;
    }
    all_long = block_min<int>(all_long, shr, 1);
    mx = block_max<int>(mx, shr, 0);
    mn = block_min<int>(mn, shr, 0x7fffffff);
  }
  const int mode = sc->cpu_overloaded ? PACK_DESC : (all_long ? PACK_FF : PACK_ASC);
  if (threadIdx.x == 0) {
    w->pack_mode = mode;
    w->need_seed = (!sc->has_ema_blocks && !sc->has_blocks_seed) ? 1 : 0;
    int big = (qlen > SORT_CAP && mode != PACK_FF) ? 1 : 0;
    w->big_queue = big;
    w->lsd_big = big;
    w->lsd_n = qlen;
    w->max_req = mx;
    w->min_req = mn;
    w->lsd_maxkey = (mode == PACK_ASC) ? (u64)mx : (u64)(mx - mn);
  }
  __syncthreads();
  if (mode == PACK_FF) {
    // first fit against available_kv, in current list order; fits, then deferred
    __shared__ long long s_cap;
    __shared__ int s_cursor, s_nfit;
    if (threadIdx.x == 0) {
      s_cap = w->adm_avail;
      s_nfit = 0;
    }
    u32* fit = L.v[1];  // scratch flags (reuse LSD buffer)
    __syncthreads();
    for (int base = 0; base < qlen; base += blockDim.x) {
      int i = base + threadIdx.x;
      i32 rq = i < qlen ? req[i] : 0;
      if (i < qlen) fit[i] = 0;
      if (threadIdx.x == 0) s_cursor = base;
      __syncthreads();
      while (true) {
        long long cap = s_cap;
        int cand = (i < qlen && i >= s_cursor && (long long)rq <= cap) ? i : 0x7fffffff;
        __shared__ int shmin[32];
        int m = block_min<int>(cand, shmin, 0x7fffffff);
        if (m == 0x7fffffff) break;
        if (threadIdx.x == 0) {
          fit[m] = 1;
          s_cap -= req[m];
          s_cursor = m + 1;
          s_nfit++;
        }
        __syncthreads();
      }
      __syncthreads();
    }
    int nfit = s_nfit;
    // stable partition by block scan over chunks
    __shared__ int s_fit_run, s_def_run;
    if (threadIdx.x == 0) {
      s_fit_run = 0;
      s_def_run = nfit;
    }
    __syncthreads();
    for (int base = 0; base < qlen; base += blockDim.x) {
      int i = base + threadIdx.x;
      u32 isfit = (i < qlen) ? fit[i] : 0;
      // scan of isfit (the deferred count is valid - isfit)
      shu[threadIdx.x] = isfit;
      __syncthreads();
      for (int off = 1; off < (int)blockDim.x; off <<= 1) {
        u32 x = threadIdx.x >= (unsigned)off ? shu[threadIdx.x - off] : 0;
        __syncthreads();
        shu[threadIdx.x] += x;
        __syncthreads();
      }
      u32 incl = shu[threadIdx.x];
      u32 tot = shu[blockDim.x - 1];
      int nvalid = min((int)blockDim.x, qlen - base);
      if (i < qlen) {
        int pos = isfit ? (s_fit_run + (int)incl - 1)
                        : (s_def_run + (int)(threadIdx.x + 1 - incl) - 1);
        L.v[0][pos] = (u32)i;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        s_fit_run += (int)tot;
        s_def_run += nvalid - (int)tot;
      }
      __syncthreads();
    }
    if (w->need_seed) {
      i32 a = cta_kth_i32(req, qlen, (qlen - 1) / 2, hist, shu);
      i32 bq = cta_kth_i32(req, qlen, qlen / 2, hist, shu);
      if (threadIdx.x == 0) w->ff_median = (qlen & 1) ? (double)a : (double)((i64)a + (i64)bq) / 2.0;
    }
    if (threadIdx.x == 0) w->lsd_cur = 0;
    return;
  }
  i32 mr = mx;
  if (qlen > SORT_CAP) {
    // big queue: the multi-CTA LSD sort's first pass reads the list itself
    // (key = req, or max_req - req for the descending pack; value = position)
    (void)mr;
    if (threadIdx.x == 0) {
      w->lsd_raw_ptr = (u64)(uintptr_t)req;
      w->lsd_cur = 0;
    }
    PTIME(19);
    return;
  }
  int n2 = next_pow2(qlen);
  u64* kh = (u64*)smem;
  u64* kl = kh + n2;
  u32* pv = (u32*)(kl + n2);
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    if (i < qlen) {
      i32 rq = req[i];
      kh[i] = (u64)(mode == PACK_ASC ? rq : (mr - rq));
    } else {
      kh[i] = ~0ull;
    }
    kl[i] = (u64)i;  // list position: makes the sort stable
    pv[i] = (u32)i;
  }
  __syncthreads();
  bitonic_sort(kh, kl, pv, n2);
  for (int i = threadIdx.x; i < qlen; i += blockDim.x) L.v[0][i] = pv[i];
  if (threadIdx.x == 0) w->lsd_cur = 0;
}

// ---------------------------------------------------------------------------
// K_AP: update_window + clamp + admit prefix + residual queue
// ---------------------------------------------------------------------------

__device__ __forceinline__ void admit_grid(Tab t, Cfg c, Work* w, Bufs b, Queue Q, const u32* perm,
                           const u64* sorted_keys, u64 keyc, int mode, bool need_seed,
                           mars_scalars* sc, i32* qsel_p, Queue G, Xchg x) {
  PTIME(12);
  __shared__ long long shl[32];
  const double now = w->in.now;
  const i64 qlen = w->qlen;
  const bool sharded = (w->in.mode & MARS_MODE_SHARDED) != 0;
  const int sel = *qsel_p;
  // packed source: the local list, or (sharded) the all-gathered global list
  const u32* src_row = sharded ? G.row[0] : PICK2(Q.row, sel);
  const i32* src_req = sharded ? G.req[0] : PICK2(Q.req, sel);
  const u8* src_lng = sharded ? G.lng[0] : PICK2(Q.lng, sel);
  // balance_and_admit scalars (control.py:181-190), computed redundantly per CTA
  bool has_seed = sc->has_blocks_seed;
  double seed = sc->blocks_seed;
  if (need_seed) {
    has_seed = true;
    if (mode == PACK_FF) {
      seed = w->ff_median;
    } else if (sorted_keys != nullptr) {
      // statistics.median of req (control.py:183-186) straight from the
      // sorted keys (req, or max_req - req descending): one load, no gather
      const u64 ka = sorted_keys[(qlen - 1) / 2], kb = sorted_keys[qlen / 2];
      const i64 mr = keyc ? (i64)keyc : (i64)w->max_req;
      const i64 r1 = mode == PACK_ASC ? (i64)ka : mr - (i64)ka;
      const i64 r2 = mode == PACK_ASC ? (i64)kb : mr - (i64)kb;
      seed = (qlen & 1) ? (double)r1 : (double)(r1 + r2) / 2.0;
    } else {
      i32 r1 = src_req[perm[(qlen - 1) / 2]];
      i32 r2 = src_req[perm[qlen / 2]];
      seed = (qlen & 1) ? (double)r1 : (double)((i64)r1 + (i64)r2) / 2.0;
    }
  }
  double wadm = sc->w_adm, last = sc->last_update;
  if (now - last >= c.ctl_interval) {  // update_window (control.py:154-160)
    if (sc->cpu_overloaded || sc->kv_overloaded) {
      double xm = wadm * c.md;
      wadm = (xm > (double)c.w_min) ? xm : (double)c.w_min;
    } else if (w->adm_usage < c.kv_lo) {
      wadm = wadm + c.ai;
    }
    last = now;
  }
  double raw = (double)w->in.worker_slots * c.oversub - (double)sc->queued_tools;
  double cpu = (raw > (double)c.w_min) ? raw : (double)c.w_min;
  double eff = sc->has_ema_blocks ? sc->ema_blocks : (has_seed ? seed : 1.0);
  double per = (1.0 > eff) ? 1.0 : eff;
  i64 cap = (i64)floor((double)w->adm_avail * (1.0 - c.reserve) / per);
  i64 act = w->adm_active;
  double kvl = ((double)(cap + act) > (double)c.w_min) ? (double)(cap + act) : (double)c.w_min;
  double m = wadm;
  if (cpu < m) m = cpu;
  if (kvl < m) m = kvl;
  i64 limit = (i64)m;
  i64 slots = limit - act;
  i64 take = slots > 0 ? (slots < qlen ? slots : qlen) : 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    w->limit = limit;
    w->slots = slots;
    w->take = take;
  }
  // admit() of the packed prefix (sim.py:148-166 + MarsPolicy.on_admit)
  const double scale = (now > 0.0 && now < 1e300) ? 1024.0 / now : 0.0;
  const u32 tw = (u32)w->t_win;
  const bool ref_w = w->ref_on[0] != 0;
  const int ref_sft = w->ref_s[0];
  const u128 ref_pp = mk128(w->ref_p[0][0], w->ref_p[0][1]) >> ref_sft;
  long long proj = 0;
  const i64 lim = ((take + 31) / 32) * 32;
  // the whole list is admitted: apply admit() in list order (row writes stay
  // sequential for a row-ordered list) -- the admitted set is the same
  const bool in_order = !sharded && !(w->in.mode & MARS_MODE_NO_ROWS) && take == qlen;
  // The packed prefix is handed out in 1024-entry chunks by a counter, not
  // strided over a fixed grid: admit() is a chain of scattered table
  // accesses and CTAs progress unevenly (64M: the last CTA finished 240 us
  // after the first).  The next chunk's grab is in flight during the
  // current one; entries are independent (the candidate appends are atomic
  // and the projected-block sum commutes), so the order does not matter.
  // (CTA g's first chunk is chunk g: no grab before the first entry)
  __shared__ long long s_c0;
  i64 c0 = (i64)blockIdx.x * blockDim.x;
  for (;;) {
    if (c0 >= lim) break;  // (block-uniform)
    u32 nxt = 0;
    if (threadIdx.x == 0) nxt = gridDim.x + atomicAdd(&w->adm_next, 1u);
    const i64 i = c0 + threadIdx.x;
    if (i < lim) {  // (whole warps: lim and c0 are multiples of 32)
      bool valid = i < take;
      bool wc = false, own = false;
      u64 whi = 0, wlo = 0;
      u32 row = 0;
      if (valid && (w->in.mode & MARS_MODE_NO_ROWS)) {
        b.admitted[i] = src_row[perm[i]];
      } else if (valid) {
        // every load is issued before the first table store (the stores may
        // alias them as far as the compiler knows): two dependent round trips
        const u32 pi = perm[i];
        const u32 pos = in_order ? (u32)i : pi;
        row = src_row[pos];
        const u32 adm = in_order ? src_row[pi] : row;
        if (sharded && row == XQ_NONE) {
          // another replica's session: a fresh queued session projects exactly
          // req_blocks (context 0, kv 0: control.py:86-87 vs sim.py:162)
          proj += src_req[pos];
        } else {
          own = sharded;
          const i32 r0p = t.r0p[row];
          const i32 kvv = t.kv[row];
          const i32 ctx0 = t.ctx[row];
          const i32 r0d = t.r0d[row];
          const u8 fl = t.flags[row];
          const double arr = c.coord ? now : t.arr[row];
          const i64 cn = (i64)ctx0 + r0p;
          const u32 lv = initial_level(c, r0p);
          const u32 kl = c.coord ? lv : 0u;
          wc = window_digit(kl, arr, scale) <= tw;
          const u32 rk = wc ? t.rank[row] : 0u;
          t.ctx[row] = (i32)cn;
          t.rem[row] = r0d;
          t.rs[row] = now;
          t.ws[row] = now;
          t.phase[row] = MARS_PREFILL;
          t.flags[row] = (fl | MARS_F_ACTIVE) & ~MARS_F_QUEUED;
          t.level[row] = (u8)lv;
          t.promos[row] = 0;
          t.served[row] = 0;
          proj += blocks_ceil(c, cn) - blocks_ceil(c, kvv);
          if (!sharded) b.admitted[i] = adm;
          if (wc) {
            window_key(kl, arr, rk, whi, wlo);
            // k_scan refined the window list: join it only at or below its bound
            if (ref_w) wc = (mk128(whi, wlo) >> ref_sft) <= ref_pp;
          }
        }
      }
      int s = warp_append(ref_w ? &w->n_wr : &w->n_wc, wc);
      if (s >= 0) {
        (ref_w ? b.wr_hi : b.wc_hi)[s] = whi;
        (ref_w ? b.wr_lo : b.wc_lo)[s] = wlo;
        (ref_w ? b.wr_row : b.wc_row)[s] = row;
      }
      // sharded: this replica's admitted rows, tagged with their packed index
      s = warp_append(&w->n_adm_own, own);
      if (s >= 0) {
        b.admitted[s] = row;
        x.adm_idx[s] = (u32)i;
      }
    }
    if (threadIdx.x == 0) s_c0 = (long long)nxt * blockDim.x;
    __syncthreads();
    c0 = s_c0;
    __syncthreads();  // (every thread has read s_c0 before the next store)
  }
  PTIME(13);
  // residual queue in packed order (control.py:190); sharded: this replica's
  // entries only, each with its new dense global position
  const i64 nres = qlen - take;
  const i64 rlim = ((nres + 31) / 32) * 32;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 j = (i64)blockIdx.x * blockDim.x + threadIdx.x; j < rlim; j += stride) {
    if (!sharded) {
      if (j < nres) {
        u32 pos = perm[take + j];
        PICK2(Q.row, 1 - sel)[j] = PICK2(Q.row, sel)[pos];
        PICK2(Q.req, 1 - sel)[j] = PICK2(Q.req, sel)[pos];
        PICK2(Q.lng, 1 - sel)[j] = PICK2(Q.lng, sel)[pos];
      }
      continue;
    }
    bool mine = false;
    u32 pos = 0;
    if (j < nres) {
      pos = perm[take + j];
      mine = src_row[pos] != XQ_NONE;
    }
    int s = warp_append(&w->n_res_own, mine);
    if (s >= 0) {
      PICK2(Q.row, 1 - sel)[s] = src_row[pos];
      PICK2(Q.req, 1 - sel)[s] = src_req[pos];
      PICK2(Q.lng, 1 - sel)[s] = src_lng[pos];
      PICK2(Q.gpos, 1 - sel)[s] = (u32)j;
    }
  }
  PTIME(14);
  long long ps = block_sum<long long>(proj, shl);
  // the last CTA past admission publishes (no grid barrier: the others exit)
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
    if (ps) atomicAdd((unsigned long long*)&w->projected, (unsigned long long)ps);
    __threadfence();
    s_last = atomicAdd(&w->adm_ctas, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    volatile Work* vw = w;
    sc->w_adm = wadm;
    sc->last_update = last;
    if (need_seed) {
      sc->has_blocks_seed = 1;
      sc->blocks_seed = seed;
    }
    sc->last_w_adm = wadm;  // telemetry.record("window_update") (telemetry.py:326-327)
    sc->has_last_w_adm = 1;
    sc->last_window_update = now;
    // gpu_submit debits (telemetry.py:324-325) on the admission-view counter
    sc->available_kv = w->adm_avail - (i64)vw->projected;
    sc->queue_len = sharded ? (i64)vw->n_res_own : qlen - take;
    w->global_residual = nres;
    *qsel_p = 1 - sel;
    __threadfence();
    atomicExch(&w->admit_done, 1u);  // k_walk may be waiting (admit_async)
    PTIME(15);
  }
}

// refresh_pressure's CPU flag (telemetry.py:174-196) as k_scan's CTA 0 will
// leave it this step, from the pre-step copies: pack_queue's mode
// (control.py:109-110) is known before the table scan ends
__device__ int cpu_overloaded_after_refresh(const Cfg& c, const Work* w) {
  const mars_step_in in = w->in;
  const bool probe = !(in.mode & MARS_MODE_SKIP_PROBE);
  const int at = probe ? in.active_tools : w->pre_active_tools;
  const int qt = probe ? in.queued_tools : w->pre_queued_tools;
  int on = w->pre_cpu_overloaded;
  if (in.control_due && !(in.mode & MARS_MODE_SKIP_REFRESH)) {
    const double slots = (double)in.worker_slots;
    const bool hi = ((double)at >= c.cpu_hi * slots) || qt > 0;
    const bool lo = ((double)at < c.cpu_lo * slots) && qt == 0;
    const int hs = hi ? w->pre_cpu_high_streak + 1 : 0;
    const int ls = lo ? w->pre_cpu_low_streak + 1 : 0;
    if (!on && hs >= c.hyst)
      on = 1;
    else if (on && ls >= c.hyst)
      on = 0;
  }
  return on;
}

// pack_queue's stable sort of a big table-backed admission list
// (control.py:101-122), run on a few SMs concurrently with k_scan on the
// others: it depends only on the list (the previous step's residual plus the
// arrivals) and on the CPU flag, not on the scan.  The descending key is
// C - req with C = 2^(8 npass) - 1 (the same order as max_req - req, with no
// reduction over the list first).  k_control takes the packed permutation
// (and the sorted keys) when the mode it derives from the scan agrees; the
// first-fit mode (every entry long) stays with k_control's CTA 0.
__global__ void __launch_bounds__(1024, 1) k_pack(Cfg c, Work* w, Queue Q, Lsd L,
                                                  const i32* qsel_p, int npass) {
  extern __shared__ __align__(16) unsigned char smem[];
  PTIME(33);
  const int qlen = (int)w->pre_queue_len;
  if (!w->in.control_due || qlen <= SORT_CAP || npass < 1 || npass > 3) return;  // grid-uniform
  const int sel = *qsel_p;
  const i32* req = PICK2(Q.req, sel);
  const int mode = cpu_overloaded_after_refresh(c, w) ? PACK_DESC : PACK_ASC;
  const u64 keyc = (1ull << (8 * npass)) - 1ull;  // > every req (host bound q_maxreq)
  LsdArgs a;
  a.n = qlen;
  a.maxkey = keyc;
  a.raw = req;
  a.asc = mode == PACK_ASC;
  a.mr = (i32)keyc;
  a.cur = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // (before the sort: nothing live across it)
    w->pk_mode = mode;
    w->pk_max_req = (i32)keyc;  // the descending keys' constant
  }
  const int cur = lsd_grid_sort<true>(L, lsd_view(w, 0), a, npass, (u32(*)[256])smem);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    w->pk_cur = cur;
    __threadfence();
    w->pk_done = 1;
  }
  PTIME(34);
}

// The control plane in one cooperative launch (grid <= #SMs - 1, the walk
// keeps an SM): CTA 0 packs small queues / first-fit; big queues are sorted by
// the whole grid (LSD); then update_window + clamp + admit() over the grid.
__global__ void __launch_bounds__(1024, 1) k_control(Tab t, Cfg c, Work* w, Bufs b, Queue Q,
                                                     Lsd L, mars_scalars* sc, i32* qsel_p,
                                                     Queue G, Xchg x, int npass) {
  extern __shared__ __align__(16) unsigned char smem[];
  if (!w->in.control_due) {  // grid-uniform
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicExch(&w->admit_done, 1u);
    return;
  }
  cg::grid_group grid = cg::this_grid();
  const int qlen = (int)w->qlen;
  const bool sharded = (w->in.mode & MARS_MODE_SHARDED) != 0;
  const i32* req = sharded ? G.req[0] : PICK2(Q.req, *qsel_p);
  // pack_queue's mode (control.py:109-122) from the queue statistics the table
  // scan (or the global-list build) reduced: computed by every CTA, so a big
  // queue goes straight into the grid-wide sort without a barrier
  int mode = PACK_ASC;
  bool big = false;
  if (!(w->in.mode & MARS_MODE_NO_ROWS) && qlen > 0) {
    const int all_long = w->tab_long_q == qlen ? 1 : 0;
    mode = sc->cpu_overloaded ? PACK_DESC : (all_long ? PACK_FF : PACK_ASC);
    big = qlen > SORT_CAP && mode != PACK_FF;
  }
  int cur;
  const u64* lsd_keys = nullptr;
  u64 lsd_keyc = 0;  // descending keys are lsd_keyc - req (0: max_req)
  if (big) {
    const int mx = w->tab_max_req, mn = w->tab_min_req;
    LsdArgs a;
    a.n = qlen;
    a.maxkey = (mode == PACK_ASC) ? (u64)mx : (u64)(mx - mn);
    a.raw = req;
    a.asc = mode == PACK_ASC;
    a.mr = mx;
    a.cur = 0;
    // k_pack sorted the list during k_scan (ascending or descending by the
    // CPU flag; a first-fit step never reaches this branch)
    const bool early = w->pk_done != 0 && w->pk_mode == mode;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      w->pack_mode = mode;
      w->need_seed = (!sc->has_ema_blocks && !sc->has_blocks_seed) ? 1 : 0;
      w->big_queue = 1;
      w->lsd_big = 1;
      w->lsd_n = qlen;
      w->max_req = mx;
      w->min_req = mn;
      w->lsd_maxkey = a.maxkey;
      w->sort_path = early ? 3 : 1;
      // the early pack derives the CPU flag from the same pre-step state
      if (w->pk_done && w->pk_mode != mode) atomicOr(&w->status, ST_QUEUE_MISMATCH);
    }
    if (early) {
      // no barrier: admission reads none of block 0's fields above (mode and
      // the seed flag are computed by every CTA; the key bound is k_pack's)
      cur = w->pk_cur;
    } else {
      cur = lsd_grid_sort<false>(L, lsd_view(w, 0), a, npass, (u32(*)[256])smem);
      if (npass == 0) grid.sync();  // (no sort barrier to order the published mode)
    }
    // sorted keys exist when at least one pass ran (pass 0 always does)
    if (npass > 0) lsd_keys = PICK2(L.k, cur);
    if (early) lsd_keyc = (u64)w->pk_max_req;
  } else {
    // small queue, first fit, or a row-less queue: one CTA packs
    if (blockIdx.x == 0 && qlen > 0) pack_small_cta(w, Q, L, sc, qsel_p, G, smem);
    if (blockIdx.x == 0 && threadIdx.x == 0 && qlen > 0) w->sort_path = w->lsd_big ? 1 : 2;
    grid.sync();
    cur = 0;
    if (npass > 0 && w->lsd_big)  // row-less big queue (reduced by pack_small_cta)
      cur = lsd_grid_sort<false>(L, lsd_view(w, 0), lsd_args_from(w, 0), npass, (u32(*)[256])smem);
    mode = w->pack_mode;
  }
  // the median seed is taken only from a non-empty queue (pack_small_cta)
  const bool need_seed = qlen > 0 && !sc->has_ema_blocks && !sc->has_blocks_seed;
  // the grid LSD sort leaves the sorted keys next to the permutation
  admit_grid(t, c, w, b, Q, PICK2(L.v, cur), lsd_keys, lsd_keyc, mode, need_seed, sc, qsel_p, G, x);
}

// ---------------------------------------------------------------------------
// sharded control plane: export / all-gather / pooled telemetry / global list
// ---------------------------------------------------------------------------

// this replica's admission list -> the all-gather send buffer
__global__ void k_export_queue(Queue Q, const i32* qsel_p, mars_scalars* sc, Xchg x, Work* w) {
  const int sel = *qsel_p;
  i64 n = sc->queue_len;
  if (n > x.cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) w->status |= ST_BAD_INPUT;
    n = x.cap;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) x.xsend[0] = (u64)n;
  // one 8-byte word per entry: the row stays home (only the owner needs it;
  // k_build_global_queue takes it from the local list, entry k <-> word k)
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    x.xsend[1 + i] = ((u64)PICK2(Q.gpos, sel)[i] << 32) |
                     ((u64)(u32)PICK2(Q.req, sel)[i] << 1) | (u64)(PICK2(Q.lng, sel)[i] & 1);
}

// all-reduced counters -> pooled telemetry; refresh_pressure on the pooled view
__global__ void k_global_control(Cfg c, Work* w, mars_scalars* sc, Xchg x) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const i64 avail = x.xc[0], total = x.xc[1], active = x.xc[2], qlen = x.xc[3];
  w->adm_avail = avail;
  w->adm_total = total;
  w->adm_usage = (double)(total - avail) / (double)total;
  w->adm_active = active;
  w->qlen = qlen;
  w->tab_long_q = 0;  // recomputed over the union list by k_build_global_queue
  w->tab_max_req = 0;
  w->tab_min_req = 0x7fffffff;
  if (w->in.control_due && !(w->in.mode & MARS_MODE_SKIP_REFRESH))
    refresh_pressure(c, sc, w->in.worker_slots, w->adm_usage);
}

// all-gathered entries -> the global list indexed by global position (this
// replica's own entries with their rows from the local list)
__global__ void k_build_global_queue(Work* w, Xchg x, Queue Q, const i32* qsel_p) {
  const i64 stride1 = 1 + x.cap;
  const u32* own_row = PICK2(Q.row, *qsel_p);
  const i64 total = (i64)x.world * x.cap;
  const i64 qlen = w->qlen;
  for (i64 f = (i64)blockIdx.x * blockDim.x + threadIdx.x; f < total;
       f += (i64)gridDim.x * blockDim.x) {
    i64 g = f / x.cap, k = f % x.cap;
    i64 cnt = (i64)x.xrecv[g * stride1];
    if (k >= cnt) continue;
    u64 key = x.xrecv[g * stride1 + 1 + k];
    u32 gp = (u32)(key >> 32);
    if ((i64)gp >= qlen) {
      w->status |= ST_BAD_INPUT;
      continue;
    }
    i32 rq = (i32)((key >> 1) & 0x7fffffffu);
    x.gq_req[gp] = rq;
    x.gq_lng[gp] = (u8)(key & 1);
    x.gq_row[gp] = (g == x.rank) ? own_row[k] : XQ_NONE;
    // statistics of the union list for pack_queue's mode (pack_small_cta)
    if (key & 1) atomicAdd(&w->tab_long_q, 1);
    atomicMax(&w->tab_max_req, rq);
    atomicMin(&w->tab_min_req, rq);
  }
}

// ---------------------------------------------------------------------------
// K_D: the window walk (scheduler.py:283-371 with baselines.py:406-438)
// ---------------------------------------------------------------------------

#define WALK_TPB 1024

// victim stream entry (prefix of the reclaim order, scheduler.py:259)
struct VEnt {
  u64 key, kl, whi, wlo;
  u32 row;
  i32 blk;
  int16_t wi;   // window index or -1
  u8 pinned, dead;
  u8 phase, flags;  // the row's phase and flags when the stream was built
  i32 pre;          // and its preemption count
};

enum { REQ_NONE = 0, REQ_DONE = 1, REQ_SORT = 2, REQ_FULLSCAN = 3 };
enum { CL_TRUE = 1, CL_FALSE = 0, CL_NEED_SORT = 2, CL_NEED_FULL = 3 };

#define FS_CAP 4096  // victims one full-scan claim may return

struct WalkShared {
  // window
  u64 whi[WIN_MAX], wlo[WIN_MAX];
  u32 wrow[WIN_MAX];
  i32 wkv[WIN_MAX], wctx[WIN_MAX], wrem[WIN_MAX];
  u8 wph[WIN_MAX], wplanned[WIN_MAX];
  int nwin;
  // walk state
  int pass, idx, sub, request, ndec, npre, nev, nj;
  long long total, freeb;
  int stream_ready, stream_len, stream_complete, stream_first;
  int fs_ready, fs_need_i, fs_b, fs_n;
  long long fs_need;
  int status;
  // fast path results
  int fast_ok;
};

struct WalkReg {
  int pass, idx, sub, ndec, npre, nev, nj, status, nwin;
  int stream_first, stream_len, stream_ready, stream_complete;
  long long total, freeb;
};

__device__ __forceinline__ void jpush(Bufs& b, WalkReg& R, u8 op, u32 row, i32 n) {
  int j = R.nj++;
  if (j < b.j_cap) {
    b.j_op[j] = op;
    b.j_row[j] = row;
    b.j_n[j] = n;
  } else {
    R.status |= ST_WALK_OVERFLOW;
  }
}

// evict one victim (sim.py:168-188) -- thread 0 only.  Stream entries carry
// the row's phase, flags and window index (gathered by the whole CTA when the
// stream is built), so their eviction is stores only; the full-table
// fallback's victims pass ph < 0 and are read here.
__device__ void walk_evict(Tab& t, Bufs& b, WalkShared& S, WalkReg& R, u32 row, bool pinned, i32 blk,
                           int ph = -1, int fl = 0, int wi = -2, int pre = 0) {
  if (ph < 0) {
    ph = t.phase[row];
    fl = t.flags[row];
    wi = t.winpos[row];
    pre = t.pre[row];
  }
  if (pinned) {
    t.flags[row] = (u8)(fl & ~MARS_F_PINNED);
  } else {
    t.pre[row] = pre + 1;  // (an atomic here would be a blocking round trip)
    if (ph == MARS_DECODE) t.phase[row] = MARS_PREFILL;
  }
  t.kv[row] = 0;
  R.freeb += blk;
  int e = R.nev++;
  if (e < b.ev_cap) {
    b.ev_row[e] = row;
    b.ev_kind[e] = pinned ? 1 : 0;
    b.ev_blk[e] = blk;
  } else {
    R.status |= ST_WALK_OVERFLOW;
  }
  jpush(b, R, pinned ? MARS_J_EVICT_PINNED : MARS_J_EVICT_RUNNING, row, blk);
  if (wi >= 0) {
    S.wkv[wi] = 0;
    if (S.wph[wi] == MARS_DECODE) S.wph[wi] = MARS_PREFILL;
  }
}

// is running row `e` (stream entry) an eligible victim for beneficiary bi
__device__ __forceinline__ bool run_eligible(const Cfg& c, const WalkShared& S, u32 row, u64 ehi,
                                             u64 elo, int ewi, int bi) {
  if (row == S.wrow[bi]) return false;
  if (ewi >= 0 && S.wplanned[ewi]) return false;
  // program_priority: strictly more service (baselines.py:180-186); the
  // key's top 32 bits are served_tokens
  if (c.policy == POL_PP) return (ehi >> 32) > (S.whi[bi] >> 32);
  if (c.coord) return key_lt(S.whi[bi], S.wlo[bi], ehi, elo);
  // coordinator off: arrival_time strictly greater (baselines.py:431); the
  // key's time part is ord(arrival)
  u64 ev = (ehi << 2) | (elo >> 62), bv = (S.whi[bi] << 2) | (S.wlo[bi] >> 62);
  return ev > bv;
}

// claim_blocks (scheduler.py:313-324) via the MARS reclaimer -- thread 0
__device__ int walk_claim(const Cfg& c, Tab& t, Bufs& b, WalkShared& S, WalkReg& R, VEnt* st, u32* fs_row,
                          u8* fs_pin, i32* fs_blk, long long need, int bi) {
  if (R.freeb >= need) return CL_TRUE;
  if (S.fs_ready && S.fs_need == need && S.fs_b == bi) {
    S.fs_ready = 0;
    if (S.fs_n == 0) return CL_FALSE;
    for (int k = 0; k < S.fs_n; ++k) {
      walk_evict(t, b, S, R, fs_row[k], fs_pin[k] != 0, fs_blk[k]);
      for (int q = 0; q < R.stream_len; ++q)
        if (st[q].row == fs_row[k]) st[q].dead = 1;
    }
    return R.freeb >= need ? CL_TRUE : CL_FALSE;
  }
  if (!R.stream_ready) return CL_NEED_SORT;
  // scan the stream prefix for the shortest sufficient eligible prefix
  long long freed = 0;
  int nch = 0;
  bool found = false;
  for (int q = R.stream_first; q < R.stream_len; ++q) {
    VEnt& e = st[q];
    if (e.dead) continue;
    if (!e.pinned) {
      if (e.blk <= 0) continue;
      if (!run_eligible(c, S, e.row, e.whi, e.wlo, e.wi, bi)) continue;
    }
    fs_row[nch] = (u32)q;  // temporarily stream indices
    nch++;
    freed += e.blk;
    if (R.freeb + freed >= need) {
      found = true;
      break;
    }
  }
  if (found) {
    for (int k = 0; k < nch; ++k) {
      VEnt& e = st[fs_row[k]];
      e.dead = 1;
      walk_evict(t, b, S, R, e.row, e.pinned != 0, e.blk, e.phase, e.flags, e.wi, e.pre);
    }
    while (R.stream_first < R.stream_len && st[R.stream_first].dead) R.stream_first++;
    return CL_TRUE;
  }
  if (R.stream_complete) return CL_FALSE;  // reclaim_for returns [] (scheduler.py:267)
  S.fs_need = need;
  S.fs_b = bi;
  return CL_NEED_FULL;
}

// try_fit (scheduler.py:136-157) -- thread 0; allocates on success
__device__ long long walk_try_fit(const Cfg& c, Bufs& b, WalkShared& S, WalkReg& R, int wi, long long desired) {
  long long kvv = S.wkv[wi];
  long long held = blocks_ceil(c, kvv);
  long long room = (held + R.freeb) * c.bs - kvv;
  long long g = desired <= room ? desired : blocks_floor_tokens(c, room);
  if (g < 1) return 0;
  long long need = blocks_ceil(c, kvv + g) - held;
  if (need > 0) {
    R.freeb -= need;
    jpush(b, R, MARS_J_ALLOC, S.wrow[wi], (i32)need);
  }
  return g;
}

// the sequential walk; returns a request code when it needs the whole CTA
__device__ int walk_run_r(const Cfg& c, Tab& t, Bufs& b, WalkShared& S, WalkReg& R, VEnt* st,
                          u32* fs_row, u8* fs_pin, i32* fs_blk) {
  const long long budget = c.budget;
  while (true) {
    if (R.pass == 0) {
      if (R.idx >= R.nwin) {
        R.pass = 1;
        R.idx = 0;
        R.sub = 0;
        continue;
      }
      int i = R.idx;
      if (S.wph[i] != MARS_DECODE || S.wrem[i] < 1) {
        R.idx++;
        continue;
      }
      if (R.total >= budget || R.ndec >= c.max_dec) {
        R.idx++;
        continue;
      }
      long long need = block_aligned(c, S.wkv[i]) ? 1 : 0;
      if (need > 0) {
        int r = walk_claim(c, t, b, S, R, st, fs_row, fs_pin, fs_blk, need, i);
        if (r == CL_NEED_SORT) return REQ_SORT;
        if (r == CL_NEED_FULL) return REQ_FULLSCAN;
        if (r == CL_FALSE) {
          R.idx++;
          continue;
        }
        R.freeb -= need;
        jpush(b, R, MARS_J_ALLOC, S.wrow[i], (i32)need);
      }
      b.dec_rows[R.ndec] = S.wrow[i];
      R.ndec++;
      S.wplanned[i] = 1;
      R.total += 1;
      R.idx++;
    } else {
      if (R.idx >= R.nwin) return REQ_DONE;
      int i = R.idx;
      if (S.wph[i] != MARS_PREFILL) {
        R.idx++;
        continue;
      }
      long long left = budget - R.total;
      if (left < 1) return REQ_DONE;
      long long rp = (long long)S.wctx[i] - S.wkv[i];
      long long desired = rp < left ? rp : left;
      if (desired < 1) {
        R.idx++;
        continue;
      }
      long long g = 0;
      long long kvv = S.wkv[i];
      long long incr = blocks_ceil(c, kvv + desired) - blocks_ceil(c, kvv);
      if (c.cosched) {
        if (R.sub == 0) {
          g = walk_try_fit(c, b, S, R, i, desired);
          if (g == 0) R.sub = 1;
        }
        if (R.sub == 1) {
          int r = walk_claim(c, t, b, S, R, st, fs_row, fs_pin, fs_blk, incr, i);
          if (r == CL_NEED_SORT) return REQ_SORT;
          if (r == CL_NEED_FULL) return REQ_FULLSCAN;
          R.sub = 0;
          g = (r == CL_TRUE) ? walk_try_fit(c, b, S, R, i, desired) : 0;
        }
      } else {
        if (incr == 0) {
          g = desired;
        } else {
          int r = walk_claim(c, t, b, S, R, st, fs_row, fs_pin, fs_blk, incr, i);
          if (r == CL_NEED_SORT) return REQ_SORT;
          if (r == CL_NEED_FULL) return REQ_FULLSCAN;
          if (r == CL_TRUE) {
            R.freeb -= incr;
            jpush(b, R, MARS_J_ALLOC, S.wrow[i], (i32)incr);
            g = desired;
          }
        }
      }
      if (g > 0) {
        b.pre_rows[R.npre] = S.wrow[i];
        b.pre_grant[R.npre] = (i32)g;
        R.npre++;
        S.wplanned[i] = 1;
        R.total += g;
      } else if (c.strict) {
        return REQ_DONE;  // head-of-line blocking (scheduler.py:369-370)
      }
      R.idx++;
    }
  }
}


// The walk's scalar state lives in thread 0's registers while it runs (every
// field of WalkShared is a shared-memory round trip, and the claim / evict /
// journal chain is strictly sequential); it is written back whenever the walk
// hands control to the whole CTA (stream sort, full-table search) or ends.
__device__ __forceinline__ void wreg_load(WalkReg& R, const WalkShared& S) {
  R.pass = S.pass;
  R.idx = S.idx;
  R.sub = S.sub;
  R.ndec = S.ndec;
  R.npre = S.npre;
  R.nev = S.nev;
  R.nj = S.nj;
  R.status = S.status;
  R.nwin = S.nwin;
  R.stream_first = S.stream_first;
  R.stream_len = S.stream_len;
  R.stream_ready = S.stream_ready;
  R.stream_complete = S.stream_complete;
  R.total = S.total;
  R.freeb = S.freeb;
}
__device__ __forceinline__ void wreg_store(WalkShared& S, const WalkReg& R) {
  S.pass = R.pass;
  S.idx = R.idx;
  S.sub = R.sub;
  S.ndec = R.ndec;
  S.npre = R.npre;
  S.nev = R.nev;
  S.nj = R.nj;
  S.status = R.status;
  S.nwin = R.nwin;
  S.stream_first = R.stream_first;
  S.stream_len = R.stream_len;
  S.stream_ready = R.stream_ready;
  S.stream_complete = R.stream_complete;
  S.total = R.total;
  S.freeb = R.freeb;
}

__device__ int walk_run(const Cfg& c, Tab& t, Bufs& b, WalkShared& S, VEnt* st, u32* fs_row,
                        u8* fs_pin, i32* fs_blk) {
  WalkReg R;
  wreg_load(R, S);
  const int rq = walk_run_r(c, t, b, S, R, st, fs_row, fs_pin, fs_blk);
  wreg_store(S, R);
  return rq;
}

// Row r's place in the policy's reclaim order, if it is an eligible victim
// for beneficiary bi: a unique 128-bit key (kh, kl), pinned rows first.
//  mars     pinned (expired first, -level, -blocks, sid), then running
//           (-level, -blocks, sid) ranked after the beneficiary
//           (scheduler.py:249-259, baselines.py:406-438);
//  fcfs     running later arrivals, latest first (baselines.py:120-130);
//  program_priority  running with more service, most first (:176-186);
//  ttl      pinned (expired first, deadline, -blocks, sid), then running like
//           fcfs (:268-298).
__device__ __forceinline__ bool fs_key(const Cfg& c, Tab& t, const WalkShared& S, i64 r,
                                       double now, int bi, u64& kh, u64& kl) {
  const u8 f = t.flags[r];
  if (f & MARS_F_PINNED) {
    if (!policy_pins(c)) return false;
    const bool nonexp = !(t.dl[r] < now);
    if (c.policy == POL_MARS) {
      kh = victim_key(false, nonexp, t.plevel[r], t.pb[r], t.rank[r]);
      kl = 0;
    } else {
      const u64 o = ord_f64(t.dl[r]);
      const i64 pb = t.pb[r];
      const u64 bb = pb > (i64)MAXH ? MAXH : (u64)(pb < 0 ? 0 : pb);
      kh = ((u64)(nonexp ? 1 : 0) << 62) | (o >> 2);
      kl = ((o & 3ull) << 62) | ((MAXH - bb) << 32) | (u64)t.rank[r];
    }
    return true;
  }
  if (!((f & MARS_F_ACTIVE) && (t.phase[r] == MARS_PREFILL || t.phase[r] == MARS_DECODE)))
    return false;
  const i32 kvv = t.kv[r];
  if (kvv <= 0) return false;
  const u32 rk = t.rank[r];
  const u32 lv = c.coord ? t.level[r] : 0u;
  u64 hi, lo;
  row_window_key(c, lv, t.rs[r], t.arr[r], t.served[r], rk, hi, lo);
  if (!run_eligible(c, S, (u32)r, hi, lo, t.winpos[r], bi)) return false;
  if (c.policy == POL_MARS) {
    kh = victim_key(true, false, lv, blocks_ceil(c, kvv), rk);
    kl = 0;
  } else if (c.policy == POL_PP) {
    const i64 sv = t.served[r];
    const u64 su = sv <= 0 ? 0ull : (u64)sv;
    kh = (1ull << 63) | (0x3fffffffffffffffull - (su & 0x3fffffffffffffffull));
    kl = rk;
  } else {
    const u64 o = ~ord_f64(t.arr[r]);  // latest arrival first
    kh = (1ull << 63) | (o >> 1);
    kl = ((o & 1ull) << 63) | (u64)rk;
  }
  return true;
}

// exact reclaimer over the whole table (the comparison policies, and MARS
// when the stream prefix is not enough) -- all threads: the shortest prefix
// of the policy's reclaim order that covers the shortfall, by repeated block
// argmin, or nothing when even every eligible victim would not cover it
__device__ void walk_fullscan(const Cfg& c, Tab& t, WalkShared& S, i64 n_rows, double now,
                              u32* fs_row, u8* fs_pin, i32* fs_blk) {
  __shared__ long long shl[32];
  __shared__ unsigned long long shk[32], shk2[32];
  __shared__ u32 shr[32];
  const int bi = S.fs_b;
  const long long need = S.fs_need;
  // eligibility + total available
  long long tot = 0;
  for (i64 r = threadIdx.x; r < n_rows; r += blockDim.x) {
    u64 kh, kl;
    if (!fs_key(c, t, S, r, now, bi, kh, kl)) continue;
    tot += (kh >> 63) == 0 ? (long long)t.pb[r] : blocks_ceil(c, t.kv[r]);
  }
  tot = block_sum<long long>(tot, shl);
  __shared__ int s_n;
  __shared__ long long s_freed;
  if (threadIdx.x == 0) {
    s_n = 0;
    s_freed = 0;
  }
  __syncthreads();
  if (S.freeb + tot < need) {
    if (threadIdx.x == 0) {
      S.fs_n = 0;
      S.fs_ready = 1;
    }
    __syncthreads();
    return;
  }
  u64 lasth = 0, lastl = 0;
  bool first = true;
  while (true) {
    u64 bh = ~0ull, bl = ~0ull;
    u32 brow = 0xffffffffu;
    for (i64 r = threadIdx.x; r < n_rows; r += blockDim.x) {
      u64 kh, kl;
      if (!fs_key(c, t, S, r, now, bi, kh, kl)) continue;
      if (!first && !key_lt(lasth, lastl, kh, kl)) continue;
      if (key_lt(kh, kl, bh, bl)) {
        bh = kh;
        bl = kl;
        brow = (u32)r;
      }
    }
    // block argmin (keys unique through the rank field)
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) {
      const u64 oh = __shfl_xor_sync(FULL, bh, o);
      const u64 ol = __shfl_xor_sync(FULL, bl, o);
      const u32 orow = __shfl_xor_sync(FULL, brow, o);
      if (key_lt(oh, ol, bh, bl)) {
        bh = oh;
        bl = ol;
        brow = orow;
      }
    }
    if (lane == 0) {
      shk[wid] = bh;
      shk2[wid] = bl;
      shr[wid] = brow;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      u64 kh = ~0ull, kl = ~0ull;
      u32 br = 0xffffffffu;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q)
        if (key_lt(shk[q], shk2[q], kh, kl)) {
          kh = shk[q];
          kl = shk2[q];
          br = shr[q];
        }
      shk[0] = kh;
      shk2[0] = kl;
      shr[0] = br;
      if (br != 0xffffffffu && s_n < FS_CAP) {
        const bool pinned = (kh >> 63) == 0;
        const i32 blk = pinned ? t.pb[br] : (i32)blocks_ceil(c, t.kv[br]);
        fs_row[s_n] = br;
        fs_pin[s_n] = pinned;
        fs_blk[s_n] = blk;
        s_n++;
        s_freed += blk;
      }
    }
    __syncthreads();
    const u64 kh = shk[0], kl = shk2[0];
    const u32 br = shr[0];
    __syncthreads();
    if (br == 0xffffffffu || S.freeb + s_freed >= need || s_n >= FS_CAP) break;
    lasth = kh;
    lastl = kl;
    first = false;
  }
  if (threadIdx.x == 0) {
    if (S.freeb + s_freed < need) S.status |= ST_WALK_OVERFLOW;
    S.fs_n = s_n;
    S.fs_ready = 1;
  }
  __syncthreads();
}

// optional: the walk's window columns, gathered for the survivors while the
// ranking runs (the payload is a table row)
struct WinGather {
  const i32 *kv, *ctx, *rem;
  const u8* phase;
  i32 *okv, *octx, *orem;
  u8* oph;
  int done;  // set when the selection filled the outputs
};

// select the `k` smallest (hi, lo) keys of a global candidate list into smem,
// sorted.  Bitonic when n <= SORT_CAP, else MSD radix refinement first.
#define GPAY(i) (gpay != nullptr ? gpay[i] : (u32)(i))
__device__ int cta_select_sorted(const u64* ghi, const u64* glo, const u32* gpay, int n, int k,
                                 u64* kh, u64* kl, u32* pv, u32* hist /*256*/,
                                 WinGather* wg = nullptr) {
  if (n > k && n <= (int)blockDim.x && n <= SORT_CAP / 2) {
    // more candidates than wanted: a 256-bucket linear histogram over the
    // candidates' hi range (monotone in the key) keeps the buckets up to the
    // k-th key's; the survivors are ranked by counting, 1024 threads sharing
    // the comparisons (keys are unique through the session rank)
    __shared__ u64 s_mm[32];
    __shared__ int s_B, s_ns;
    __shared__ u32 s_rank[512];
    u64* th = kh + SORT_CAP / 2;
    u64* tl = kl + SORT_CAP / 2;
    u32* tp = pv + SORT_CAP / 2;
    const int i = threadIdx.x;
    u64 h = ~0ull, l = ~0ull;
    u32 p = 0;
    if (i < n) {
      h = ghi[i];
      l = glo[i];
      p = GPAY(i);
    }
    // the candidates' hi range: one barrier, every warp folds the 32 partials
    __shared__ u64 s_mx[32];
    {
      const u64 wmn = warp_min(h), wmx = warp_max(i < n ? h : 0ull);
      if ((i & 31) == 0) {
        s_mm[i >> 5] = wmn;
        s_mx[i >> 5] = wmx;
      }
    }
    __syncthreads();
    const int nwarp = (int)(blockDim.x >> 5);
    const u64 mn = warp_min((i & 31) < nwarp ? s_mm[i & 31] : ~0ull);
    const u64 mx = warp_max((i & 31) < nwarp ? s_mx[i & 31] : 0ull);
    PTIME(36);
    const double span = (double)(mx - mn);
    const double inv = span > 0.0 ? 255.0 / span : 0.0;
    u32 bk = 0;
    if (i < n) {
      const double f = (double)(h - mn) * inv;
      bk = f >= 255.0 ? 255u : (u32)f;
    }
    for (int q = i; q < 256; q += blockDim.x) hist[q] = 0;
    if (i == 0) s_ns = 0;
    __syncthreads();
    if (i < n) atomicAdd(&hist[bk], 1u);
    __syncthreads();
    if (i < 32) {  // first bucket whose cumulative count reaches k
      u32 v[8], sum = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        v[q] = hist[i * 8 + q];
        sum += v[q];
      }
      u32 incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 x = __shfl_up_sync(FULL, incl, o);
        if (i >= o) incl += x;
      }
      u32 cum = incl - sum;
      int B = 0x7fffffff;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (cum < (u32)k && cum + v[q] >= (u32)k) B = i * 8 + q;
        cum += v[q];
      }
      B = __reduce_min_sync(FULL, B);
      if (i == 0) s_B = B;
    }
    __syncthreads();
    if (i < n && (int)bk <= s_B) {
      const int sl = atomicAdd(&s_ns, 1);
      th[sl] = h;
      tl[sl] = l;
      tp[sl] = p;
    }
    __syncthreads();
    PTIME(37);
    const int ns = s_ns;
    if (ns <= 512) {
      // the survivors' window columns: loads in flight during the ranking
      i32 gkv = 0, gctx = 0, grem = 0;
      u8 gph = 0;
      if (wg != nullptr && i < ns) {
        const u32 r = tp[i];
        gkv = wg->kv[r];
        gctx = wg->ctx[r];
        grem = wg->rem[r];
        gph = wg->phase[r];
      }
      // parts threads per survivor, each counting a slice of the others
      const int parts = ns <= 128 ? 8 : ns <= 170 ? 6 : ns <= 256 ? 4 : 2;
      const int q = i / parts, part = i % parts;
      if (i < 512) s_rank[i] = 0;
      __syncthreads();
      if (q < ns) {
        const u64 qh = th[q], ql = tl[q];
        int cnt = 0;
        for (int j = part; j < ns; j += parts) cnt += key_lt(th[j], tl[j], qh, ql) ? 1 : 0;
        if (cnt) atomicAdd(&s_rank[q], (u32)cnt);
      }
      __syncthreads();
      if (i < ns) {
        const int rnk = (int)s_rank[i];
        if (rnk < k) {
          kh[rnk] = th[i];
          kl[rnk] = tl[i];
          pv[rnk] = tp[i];
          if (wg != nullptr) {
            wg->okv[rnk] = gkv;
            wg->octx[rnk] = gctx;
            wg->orem[rnk] = grem;
            wg->oph[rnk] = gph;
          }
        }
      }
      if (wg != nullptr && i == 0) wg->done = 1;
      __syncthreads();
      return k;
    }
    // clustered keys: fall through to the full sort
  }
  if (n <= (int)blockDim.x && n <= SORT_CAP / 2) {
    // small candidate sets: bitonic network with one key per thread held in
    // registers -- partners exchange by warp shuffle for strides < 32 and
    // through shared memory (two barriers) only for the wider strides
    u64* xh = kh + SORT_CAP / 2;
    u64* xl = kl + SORT_CAP / 2;
    u32* xp = pv + SORT_CAP / 2;
    const int i = threadIdx.x;
    const int n2 = next_pow2(n > 1 ? n : 1);
    u64 h = ~0ull, l = ~0ull;
    u32 p = 0xffffffffu;
    if (i < n) {
      h = ghi[i];
      l = glo[i];
      p = GPAY(i);
    }
    for (int kk = 2; kk <= n2; kk <<= 1) {
      for (int j = kk >> 1; j > 0; j >>= 1) {
        u64 oh, ol;
        u32 op;
        if (j >= 32) {
          __syncthreads();
          if (i < n2) {
            xh[i] = h;
            xl[i] = l;
            xp[i] = p;
          }
          __syncthreads();
          const int q = (i ^ j) < n2 ? (i ^ j) : i;
          oh = xh[q];
          ol = xl[q];
          op = xp[q];
        } else if ((i & ~31) < n2) {  // warps without elements skip the shuffles
          oh = __shfl_xor_sync(FULL, h, j);
          ol = __shfl_xor_sync(FULL, l, j);
          op = __shfl_xor_sync(FULL, p, j);
        } else {
          continue;
        }
        // the lower position of an ascending pair keeps the minimum
        const bool want_min = ((i & j) == 0) == ((i & kk) == 0);
        const bool other_less = key_lt(oh, ol, h, l);
        if (i < n2 && (want_min ? other_less : key_lt(h, l, oh, ol))) {
          h = oh;
          l = ol;
          p = op;
        }
      }
    }
    __syncthreads();
    if (i < n && i < k) {
      kh[i] = h;
      kl[i] = l;
      pv[i] = p;
    }
    __syncthreads();
    return n < k ? n : k;
  }
  if (n <= SORT_CAP) {
    int n2 = next_pow2(n > 1 ? n : 1);
    for (int i = threadIdx.x; i < n2; i += blockDim.x) {
      kh[i] = i < n ? ghi[i] : ~0ull;
      kl[i] = i < n ? glo[i] : ~0ull;
      pv[i] = i < n ? GPAY(i) : 0xffffffffu;
    }
    __syncthreads();
    bitonic_sort(kh, kl, pv, n2);
    return n < k ? n : k;
  }
  // MSD refinement over the 128-bit key: find the k-th smallest key exactly
  __shared__ u64 s_ph, s_pl, s_mh, s_ml;
  __shared__ int s_need;
  if (threadIdx.x == 0) {
    s_ph = s_pl = s_mh = s_ml = 0;
    s_need = k;
  }
  __syncthreads();
  for (int d = 0; d < 16; ++d) {
    int shift = 56 - 8 * (d & 7);
    bool hiword = d < 8;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    u64 ph = s_ph, pl = s_pl, mh = s_mh, ml = s_ml;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      u64 h = ghi[i], l = glo[i];
      if ((h & mh) == ph && (l & ml) == pl) {
        u32 dg = (u32)(((hiword ? h : l) >> shift) & 255u);
        atomicAdd(&hist[dg], 1u);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int need = s_need;
      u32 cum = 0;
      int bin = 255;
      for (int q = 0; q < 256; ++q) {
        if (cum + hist[q] >= (u32)need) {
          bin = q;
          break;
        }
        cum += hist[q];
      }
      s_need = need - (int)cum;
      if (hiword) {
        s_ph |= ((u64)bin) << shift;
        s_mh |= 255ull << shift;
      } else {
        s_pl |= ((u64)bin) << shift;
        s_ml |= 255ull << shift;
      }
    }
    __syncthreads();
  }
  // s_ph/s_pl is now the exact k-th smallest key; gather keys <= it
  __shared__ int s_cnt;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  u64 th = s_ph, tl = s_pl;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    u64 h = ghi[i], l = glo[i];
    if (!key_lt(th, tl, h, l)) {
      int s = atomicAdd(&s_cnt, 1);
      if (s < SORT_CAP) {
        kh[s] = h;
        kl[s] = l;
        pv[s] = GPAY(i);
      }
    }
  }
  __syncthreads();
  int m = s_cnt < SORT_CAP ? s_cnt : SORT_CAP;
  int n2 = next_pow2(m > 1 ? m : 1);
  for (int i = m + threadIdx.x; i < n2; i += blockDim.x) {
    kh[i] = ~0ull;
    kl[i] = ~0ull;
    pv[i] = 0xffffffffu;
  }
  __syncthreads();
  bitonic_sort(kh, kl, pv, n2);
  return m < k ? m : k;
}

// The victim stream (whole CTA): the policy's reclaim-order prefix k_scan
// selected (refined: the exact top VSEL plus < REF_STOP), sorted by the
// 128-bit key, with each entry's row state gathered once (phase, flags,
// window index) so that evicting it is stores only.
__device__ void walk_build_stream(const Cfg& c, Tab& t, Work* w, Bufs& b, WalkShared& S, VEnt* st,
                                  u64* kh, u64* kl, u32* pv, u32* hist) {
  PTIME(38);
  const bool ref_v = w->ref_on[1] != 0;
  const int nvc = ref_v ? w->n_vr : w->n_vc;
  const bool presorted = w->vs_on != 0;  // k_scan ranked the candidates (grid-wide)
  const u64* vkh = presorted ? b.vs_key : (ref_v ? b.vr_key : b.vc_key);
  const u64* vkl = presorted ? b.vs_kl : (ref_v ? b.vr_kl : b.vc_kl);
  int len;
  if (presorted) {
    len = nvc < c.stream_cap ? nvc : c.stream_cap;
  } else {
    len = cta_select_sorted(vkh, vkl, nullptr, nvc, c.stream_cap, kh, kl, pv, hist);
    __syncthreads();
  }
  PTIME(57);
  const u64* vwh = presorted ? b.vs_whi : (ref_v ? b.vr_whi : b.vc_whi);
  const u64* vwl = presorted ? b.vs_wlo : (ref_v ? b.vr_wlo : b.vc_wlo);
  const u32* vrw = presorted ? b.vs_row : (ref_v ? b.vr_row : b.vc_row);
  const i32* vbk = presorted ? b.vs_blk : (ref_v ? b.vr_blk : b.vc_blk);
  for (int q = threadIdx.x; q < len; q += blockDim.x) {
    const u32 ci = presorted ? (u32)q : pv[q];
    VEnt e;
    e.key = presorted ? vkh[q] : kh[q];
    e.kl = presorted ? vkl[q] : kl[q];
    e.whi = vwh[ci];
    e.wlo = vwl[ci];
    e.row = vrw[ci];
    e.blk = vbk[ci];
    e.pinned = (e.key >> 63) == 0;
    e.dead = 0;
    e.wi = t.winpos[e.row];
    e.phase = t.phase[e.row];
    e.flags = t.flags[e.row];
    e.pre = t.pre[e.row];
    st[q] = e;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    S.stream_ready = 1;
    S.stream_len = len;
    S.stream_first = 0;
    // the stream holds every potential victim of the step
    S.stream_complete = (len == nvc && nvc == w->n_victims) ? 1 : 0;
  }
  __syncthreads();
  PTIME(39);
}

// build_plan's decode pass with its claims (scheduler.py:326-341, claim_blocks
// :313-324) on the whole CTA.  The pass selects the first min(max_decode,
// budget) decode-ready window rows, each allocating one block when its KV is
// block aligned; a claim evicts the shortest prefix of the eligible reclaim
// order that covers the shortfall.  When every stream entry those claims
// consume is outside the window and eligible for the last claiming decode
// (eligibility only narrows along the window order), the claims are plain
// prefix sums: with B(v) the blocks of the first v stream entries and N_i the
// block needs through decode i, decode i's claim evicts the entries
// [v(N_i - 1), v(N_i)) where v(x) = min{v : free + B(v) >= x}, and the journal
// interleaves them with the allocations in the same order the sequential walk
// would.  Otherwise (a window row among them, a tie-ineligible entry, a short
// stream) nothing is touched and the sequential walk runs the pass.
__device__ void walk_decode_claims(const Cfg& c, Tab& t, Bufs& b, WalkShared& S, VEnt* st,
                                   long long* B /* [len + 1] */) {
  __shared__ int s_e[4], s_n[4], s_s[4];
  __shared__ int s_ilast, s_vstar, s_ok;
  __shared__ long long s_wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const u32 lt = (1u << lane) - 1u;
  const int nwin = S.nwin, len = S.stream_len;
  const long long free0 = S.freeb;
  const long long lim_dec = c.max_dec < c.budget ? c.max_dec : c.budget;
  const bool win = tid < WIN_MAX && tid < nwin;
  const bool e = win && S.wph[tid] == MARS_DECODE && S.wrem[tid] >= 1;
  const u32 me = __ballot_sync(FULL, e);
  if (tid < WIN_MAX && lane == 0) s_e[wid] = __popc(me);
  if (tid == 0) {
    s_ilast = -1;
    s_vstar = 0;
    s_ok = 1;
  }
  __syncthreads();
  int eb = 0;
  if (tid < WIN_MAX)
    for (int k = 0; k < wid; ++k) eb += s_e[k];
  const bool sel = e && (eb + __popc(me & lt)) < lim_dec;
  const bool dn = sel && block_aligned(c, S.wkv[tid]);
  const u32 ms = __ballot_sync(FULL, sel), mn = __ballot_sync(FULL, dn);
  if (tid < WIN_MAX && lane == 0) {
    s_s[wid] = __popc(ms);
    s_n[wid] = __popc(mn);
  }
  __syncthreads();
  int sb = 0, nb = 0, Nd = 0, nsel = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const bool before = tid < WIN_MAX && k < wid;
    sb += before ? s_s[k] : 0;
    nb += before ? s_n[k] : 0;
    Nd += s_n[k];
    nsel += s_s[k];
  }
  const int Ni = nb + __popc(mn & lt) + (dn ? 1 : 0);  // needs through this decode
  if (dn && Ni == Nd) s_ilast = tid;                      // the last claiming beneficiary
  // stream prefix sums B(v) (no entry is dead yet)
  const long long blk = tid < len ? (long long)st[tid].blk : 0;
  long long incl = blk;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long x = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += x;
  }
  if (lane == 31) s_wsum[wid] = incl;
  __syncthreads();
  for (int k = 0; k < wid; ++k) incl += s_wsum[k];
  if (tid < len) B[tid + 1] = incl;
  if (tid == 0) B[0] = 0;
  const long long need_total = (long long)Nd - free0;  // blocks the claims must free
  if (need_total > 0 && tid < len && incl - blk < need_total && incl >= need_total)
    s_vstar = tid + 1;
  __syncthreads();
  const int vstar = s_vstar;
  if (need_total > 0 && vstar == 0) s_ok = 0;  // the stream cannot cover the pass
  __syncthreads();
  if (!s_ok) return;
  // every consumed entry: outside the window, eligible for the last claimer
  bool good = true;
  if (tid < vstar) {
    const VEnt& v = st[tid];
    good = v.wi < 0 && !v.dead && v.blk > 0 &&
           (v.pinned || run_eligible(c, S, v.row, v.whi, v.wlo, v.wi, s_ilast));
  }
  if (!__syncthreads_and(good)) return;
  PTIME(58);
  // apply: decodes, their claims' evictions and the interleaved journal
  if (sel) {
    b.dec_rows[sb + __popc(ms & lt)] = S.wrow[tid];
    S.wplanned[tid] = 1;
  }
  if (dn) {
    auto vof = [&](long long x) {  // min{v in [0, vstar] : free0 + B(v) >= x}
      int lo = 0, hi = vstar;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (free0 + B[mid] >= x) hi = mid; else lo = mid + 1;
      }
      return lo;
    };
    const int v1 = vof(Ni), v0 = vof(Ni - 1);
    for (int q = v0; q < v1; ++q) {
      VEnt& v = st[q];
      v.dead = 1;
      const u32 r = v.row;
      if (v.pinned) {
        t.flags[r] = (u8)(v.flags & ~MARS_F_PINNED);
      } else {
        t.pre[r] = v.pre + 1;
        if (v.phase == MARS_DECODE) t.phase[r] = MARS_PREFILL;
      }
      t.kv[r] = 0;
      b.ev_row[q] = r;
      b.ev_kind[q] = v.pinned ? 1 : 0;
      b.ev_blk[q] = v.blk;
      const int js = q + Ni - 1;
      b.j_op[js] = v.pinned ? MARS_J_EVICT_PINNED : MARS_J_EVICT_RUNNING;
      b.j_row[js] = r;
      b.j_n[js] = v.blk;
    }
    const int ja = v1 + Ni - 1;
    b.j_op[ja] = MARS_J_ALLOC;
    b.j_row[ja] = S.wrow[tid];
    b.j_n[ja] = 1;
  }
  __syncthreads();
  if (tid == 0) {
    S.ndec = nsel;
    S.total = nsel;
    S.freeb = free0 + B[vstar] - Nd;
    S.nev = vstar;
    S.nj = vstar + Nd;
    S.stream_first = vstar;
    S.pass = 1;
    S.idx = 0;
    S.sub = 0;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(WALK_TPB) k_walk(Tab t, Cfg c, Work* w, Bufs b,
                                                   mars_scalars* sc, i64 n_rows,
                                                   int admit_async) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ WalkShared S;
  __shared__ u32 hist[256];
  // dynamic smem: sort area (SORT_CAP x (8+8+4)) reused for the victim stream
  u64* kh = (u64*)smem;
  u64* kl = kh + SORT_CAP;
  u32* pv = (u32*)(kl + SORT_CAP);
  VEnt* st = (VEnt*)(pv + SORT_CAP);           // VSTREAM_CAP entries
  u32* fs_row = (u32*)(st + VSTREAM_CAP);       // FS_CAP
  u8* fs_pin = (u8*)(fs_row + FS_CAP);
  i32* fs_blk = (i32*)(((uintptr_t)(fs_pin + FS_CAP) + 15) & ~(uintptr_t)15);

  const double now = w->in.now;
  const long long freeb0 = threadIdx.x == 0 ? sc->free_blocks : 0;  // in flight early
  PTIME(16);
  // Admission runs concurrently on the side stream.  Admitted sessions hold no
  // KV (fresh arrivals), so they are never reclaim victims; they can only join
  // the window when their window digit (level << 10 | bucket(now) = 1023, or
  // the arrival bucket with the coordinator off) reaches the threshold -- then
  // wait for the admission to finish (its candidates and row state).
  if (admit_async) {
    if (threadIdx.x == 0) {
      const bool independent = c.coord && now > 0.0 && now < 1e300 && (u32)w->t_win < 1023u &&
                               w->n_queued_kv == 0;
      if (!independent) {
        // bounded: a missing completion flag is reported, never a hang
        long long spins = 0;
        while (atomicAdd(&w->admit_done, 0u) == 0u) {
          __nanosleep(128);
          if (++spins > (1ll << 24)) {
            w->status |= ST_BAD_INPUT;
            break;
          }
        }
        __threadfence();
      }
    }
    __syncthreads();
  }
  // 1. window = top-k of the candidates (k_scan + admitted rows)
  PTIME(35);
  const bool ref_w = w->ref_on[0] != 0;  // k_scan refined the window list
  int nwc = ref_w ? w->n_wr : w->n_wc;
  __shared__ WinGather wg;
  if (threadIdx.x == 0) {
    wg.kv = t.kv;
    wg.ctx = t.ctx;
    wg.rem = t.rem;
    wg.phase = t.phase;
    wg.okv = S.wkv;
    wg.octx = S.wctx;
    wg.orem = S.wrem;
    wg.oph = S.wph;
    wg.done = 0;
  }
  __syncthreads();
  int nwin = cta_select_sorted(ref_w ? b.wr_hi : b.wc_hi, ref_w ? b.wr_lo : b.wc_lo,
                               ref_w ? b.wr_row : b.wc_row, nwc, c.window, kh, kl, pv, hist, &wg);
  PTIME(24);
  const bool gathered = wg.done != 0;
  for (int i = threadIdx.x; i < nwin; i += blockDim.x) {
    u32 r = pv[i];
    S.whi[i] = kh[i];
    S.wlo[i] = kl[i];
    S.wrow[i] = r;
    if (!gathered) {
      S.wkv[i] = t.kv[r];
      S.wctx[i] = t.ctx[r];
      S.wrem[i] = t.rem[r];
      S.wph[i] = t.phase[r];
    }
    S.wplanned[i] = 0;
    t.winpos[r] = (int16_t)i;
    b.win_rows[i] = r;
  }
  if (threadIdx.x == 0) {
    S.nwin = nwin;
    S.pass = 0;
    S.idx = 0;
    S.sub = 0;
    S.ndec = S.npre = S.nev = S.nj = 0;
    S.total = 0;
    S.freeb = freeb0;
    S.stream_ready = 0;
    S.stream_len = 0;
    S.stream_first = 0;
    S.stream_complete = 0;
    S.fs_ready = 0;
    S.status = 0;
    S.fast_ok = 0;
    if (!w->vic_on) {
      // the free pool covers every allocation a plan can make, so k_scan built
      // no victim stream; a claim cannot fail (were one to, the exact
      // full-table reclaimer would serve it)
      S.stream_ready = 1;
      S.stream_complete = 0;
    }
  }
  __syncthreads();
  PTIME(17);

  // 2. fast path (warp 0): no claim can fail when the free pool covers every
  //    allocation of the greedy plan -> prefix sums reproduce build_plan.
  //    Four warps, one per 32 window entries (WIN_MAX = 128), exchange their
  //    per-warp counts through shared memory at three named barriers (the
  //    other warps do not take part): each stage is one pass, not four.
  if (threadIdx.x < WIN_MAX) {
    __shared__ int s_wc[4][6];         // per warp: eligible, selected, decode allocs,
                                       // granted, prefill allocs, (pad)
    __shared__ long long s_wl[4][3];   // per warp: need_dec, rp total, need_pre / grants
    const int lane = threadIdx.x & 31, q = threadIdx.x >> 5, i = threadIdx.x;
    const u32 lt = (1u << lane) - 1u;
    const long long budget = c.budget;
    const long long lim_dec = c.max_dec < budget ? c.max_dec : budget;
    const bool in = i < nwin;
    const u8 ph = in ? S.wph[i] : (u8)0;
    const i32 kv = in ? S.wkv[i] : 0;
    // stage 1: decode eligibility (window order) and the prefill requests
    const bool e = in && ph == MARS_DECODE && S.wrem[i] >= 1;
    const u32 me = __ballot_sync(FULL, e);
    const bool p = in && ph == MARS_PREFILL;
    const long long rp = p ? ((long long)S.wctx[i] - kv) : 0;
    const long long rpp = rp > 0 ? rp : 0;
    long long incl = rpp;  // inclusive warp scan of the prefill requests
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long x = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += x;
    }
    if (lane == 31) {
      s_wc[q][0] = __popc(me);
      s_wl[q][1] = incl;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(WIN_MAX) : "memory");
    int e_before = 0, e_total = 0;
    long long run = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      e_before += k < q ? s_wc[k][0] : 0;
      e_total += s_wc[k][0];
      run += k < q ? s_wl[k][1] : 0;
    }
    const int epos = e_before + __popc(me & lt);
    const bool sel = e && epos < lim_dec;
    const bool dneed = sel && block_aligned(c, kv);
    const long long ndec = e_total < lim_dec ? e_total : lim_dec;
    // stage 2: prefill grants S_j = min(P_j, left0), g_j = min(rp_j, left0 - S_j)
    const long long left0 = budget - ndec;
    const long long P = run + incl - rpp;
    const long long Sj = P < left0 ? P : left0;
    const long long lft = left0 - Sj;
    long long g = 0;
    if (p && lft >= 1 && rp >= 1) g = rp < lft ? rp : lft;
    const long long nd = g > 0 ? blocks_ceil(c, kv + g) - blocks_ceil(c, kv) : 0;
    const u32 msel = __ballot_sync(FULL, sel), mdn = __ballot_sync(FULL, dneed);
    const u32 mg = __ballot_sync(FULL, g > 0), mpn = __ballot_sync(FULL, nd > 0);
    const long long nd_w = warp_sum<long long>(nd), g_w = warp_sum<long long>(g);
    if (lane == 0) {
      s_wc[q][1] = __popc(msel);
      s_wc[q][2] = __popc(mdn);
      s_wc[q][3] = __popc(mg);
      s_wc[q][4] = __popc(mpn);
      s_wl[q][0] = nd_w;
      s_wl[q][2] = g_w;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(WIN_MAX) : "memory");
    int dbefore = 0, dn_before = 0, dn_total = 0, gbefore = 0, pn_before = 0;
    long long need_pre = 0, gsum = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool b4 = k < q;
      dbefore += b4 ? s_wc[k][1] : 0;
      dn_before += b4 ? s_wc[k][2] : 0;
      dn_total += s_wc[k][2];
      gbefore += b4 ? s_wc[k][3] : 0;
      pn_before += b4 ? s_wc[k][4] : 0;
      need_pre += s_wl[k][0];
      gsum += s_wl[k][2];
    }
    const long long need_dec = dn_total;
    PTIME(22);
    const bool ok = S.freeb >= need_dec + need_pre;
    if (ok) {
      // stage 3: emit in window order -- decodes, their allocations, then
      // prefill grants and their allocations after every decode allocation
      const u32 r = in ? S.wrow[i] : 0u;
      if (sel) {
        b.dec_rows[dbefore + __popc(msel & lt)] = r;
        S.wplanned[i] = 1;
      }
      if (dneed) {
        const int jp = dn_before + __popc(mdn & lt);
        b.j_op[jp] = MARS_J_ALLOC;
        b.j_row[jp] = r;
        b.j_n[jp] = 1;
      }
      if (g > 0) {
        const int pos = gbefore + __popc(mg & lt);
        b.pre_rows[pos] = r;
        b.pre_grant[pos] = (i32)g;
        S.wplanned[i] = 1;
      }
      if (nd > 0) {
        const int jp = dn_total + pn_before + __popc(mpn & lt);
        b.j_op[jp] = MARS_J_ALLOC;
        b.j_row[jp] = r;
        b.j_n[jp] = (i32)nd;
      }
      if (threadIdx.x == 0) {
        int dc = 0, pc = 0, pn = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          dc += s_wc[k][1];
          pc += s_wc[k][3];
          pn += s_wc[k][4];
        }
        S.fast_ok = 1;
        S.ndec = dc;
        S.npre = pc;
        S.nj = dn_total + pn;
        S.total = ndec + gsum;
        S.freeb -= need_dec + need_pre;
        S.request = REQ_DONE;
      }
    }
    PTIME(23);
  }
  __syncthreads();
  PTIME(20);

  // 3. the victim stream and the decode pass with its claims on the whole
  //    CTA, then the sequential walk (the prefill pass, or everything when the
  //    parallel decode pass does not apply) with on-demand help from the CTA
  if (!S.fast_ok) {
    if (!S.stream_ready) {
      walk_build_stream(c, t, w, b, S, st, kh, kl, pv, hist);
      walk_decode_claims(c, t, b, S, st, (long long*)kh);
    }
    while (true) {
      if (threadIdx.x == 0) S.request = walk_run(c, t, b, S, st, fs_row, fs_pin, fs_blk);
      __syncthreads();
      int rq = S.request;
      if (rq == REQ_DONE) break;
      if (rq == REQ_SORT) {
        walk_build_stream(c, t, w, b, S, st, kh, kl, pv, hist);
      } else if (rq == REQ_FULLSCAN) {
        if (threadIdx.x == 0) w->n_fullscan += 1;
        walk_fullscan(c, t, S, n_rows, now, fs_row, fs_pin, fs_blk);
      }
    }
  }
  PTIME(18);
  __syncthreads();

  // 4. drop-in epilogues on the planned rows: charge_service at tick end
  //    (baselines.py:362-367 via sim.py:364) and decide_retention for decodes
  //    that finish their round this tick, on post-tick values (sim.py:233-250,
  //    engine.py:503-512: kv+1, context+1, now + tick).
  const int mode = w->in.mode;
  if (mode & (MARS_MODE_SERVICE | MARS_MODE_FINISH_RETENTION)) {
    const double tick_end = now + c.tick_s;
    const int nd = S.ndec, np_ = S.npre;
    const i64 total = sc->total_blocks;
    const double usage = sc->kv_usage_ratio;
    const double ema = sc->has_ema_tool ? sc->ema_tool : c.tool_prior;
    for (int i = threadIdx.x; i < nd + np_; i += blockDim.x) {
      bool dec = i < nd;
      u32 r = dec ? b.dec_rows[i] : b.pre_rows[i - nd];
      i64 tokens = dec ? 1 : b.pre_grant[i - nd];
      u32 lv = t.level[r];
      if ((mode & MARS_MODE_SERVICE) && c.coord) {
        const i64 served0 = t.served[r];
        b.svc_pre[i] = (served0 << 8) | (i64)lv;
        i64 served = served0 + tokens;
        if (served > c.quotas[lv] && (int)lv < c.num_levels - 1) {
          lv += 1;
          served = 0;
        }
        t.served[r] = served;
        t.level[r] = (u8)lv;
        t.ws[r] = tick_end;
      }
      if (dec) b.dec_level[i] = (u8)lv;
      else b.pre_level[i - nd] = (u8)lv;
    }
    if (mode & MARS_MODE_FINISH_RETENTION) {
      int lim = ((nd + 31) / 32) * 32;
      for (int i = threadIdx.x; i < lim; i += blockDim.x) {
        bool fin = false;
        u32 r = 0;
        if (i < nd) {
          r = b.dec_rows[i];
          fin = t.rem[r] == 1;
        }
        int sl = warp_append(&w->n_finish, fin);
        if (sl >= 0) {
          u8 pin;
          double bb, cc, dd;
          decide_retention(c, (i64)t.ctx[r] + 1, (i64)t.kv[r] + 1, total, usage, ema, tick_end,
                           pin, bb, cc, dd);
          b.fin_row[sl] = r;
          b.fin_pin[sl] = pin;
          b.fin_b[sl] = bb;
          b.fin_c[sl] = cc;
          b.fin_d[sl] = dd;
        }
      }
    }
  }

  // 5. outputs, scalars, winpos reset
  for (int i = threadIdx.x; i < nwin; i += blockDim.x) t.winpos[S.wrow[i]] = -1;
  if (threadIdx.x == 0) {
    w->n_window = nwin;
    w->n_dec = S.ndec;
    w->n_pre = S.npre;
    w->n_evict = S.nev;
    w->n_journal = S.nj;
    w->total_tokens = S.total;
    w->walk_slow = S.fast_ok ? 0 : 1;
    w->status |= S.status;
    sc->free_blocks = S.freeb;
    w->free_after_plan = S.freeb;
    PTIME(21);
  }
}

// ---------------------------------------------------------------------------
// MARS_MODE_ADVANCE: the tick's tail on the device
// ---------------------------------------------------------------------------

// After the plan, the admission and the walk's tick-end charges (SERVICE):
// step_gpu on the planned rows (engine.py:459-514: a grant extends the KV and
// ends the prefill when it reaches the context; a decode slot emits one token
// into context and KV), then every round that ended this tick, in decode order
// as the sim walks the progress list (sim.py:355-375 -> finish_round,
// sim.py:233-279): Telemetry.note_round_blocks (a sequential EMA fold,
// telemetry.py:130-138), DONE and a full free on the last round, otherwise the
// policy's retention decision on post-tick values -- pin the held blocks
// (PinnedSession level = the post-charge level, baselines.py:386-394) or free
// them -- and phase TOOL.  The tool plane and resume_from_tool stay with the
// host (tool durations are trace data).  One CTA; the sequential part is at
// most max_decode_slots rows.
__global__ void __launch_bounds__(1024) k_advance(Tab t, Cfg c, Work* w, Bufs b,
                                                  mars_scalars* sc) {
  const int nd = w->n_dec, np = w->n_pre;
  const double tick_end = w->in.now + c.tick_s;
  for (int i = threadIdx.x; i < np; i += blockDim.x) {
    const u32 r = b.pre_rows[i];
    const i32 kv = t.kv[r] + b.pre_grant[i];
    t.kv[r] = kv;
    const bool done = kv == t.ctx[r];  // remaining_prefill == 0
    if (done) t.phase[r] = MARS_DECODE;
    b.pre_done[i] = done ? 1 : 0;
    if (c.policy == POL_PP) t.served[r] += b.pre_grant[i];  // Call.served_tokens
  }
  for (int i = threadIdx.x; i < nd; i += blockDim.x) {
    const u32 r = b.dec_rows[i];
    t.kv[r] += 1;
    t.ctx[r] += 1;
    t.rem[r] -= 1;
    if (c.policy == POL_PP) t.served[r] += 1;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  i64 freeb = sc->free_blocks;
  bool has_ema = sc->has_ema_blocks != 0;
  double ema_b = sc->ema_blocks;
  const i64 total = sc->total_blocks;
  const double usage = sc->kv_usage_ratio;
  const double ema_t = sc->has_ema_tool ? sc->ema_tool : c.tool_prior;
  const bool decides = (c.policy == POL_MARS && c.cosched) || c.policy == POL_STATIC_TTL ||
                       c.policy == POL_DYNAMIC_TTL;
  int n_end = 0, n_done = 0;
  for (int i = 0; i < nd; ++i) {
    const u32 r = b.dec_rows[i];
    if (t.rem[r] != 0) continue;
    n_end++;
    const i32 kv = t.kv[r], ctx = t.ctx[r];
    const i64 held = held_blocks(c, kv);
    const double x = (double)blocks_ceil(c, ctx);
    ema_b = has_ema ? c.ema_alpha * x + (1.0 - c.ema_alpha) * ema_b : x;  // telemetry.py:59-63
    has_ema = true;
    const u8 f = t.flags[r];
    const int e = n_end - 1;
    b.end_row[e] = r;
    b.end_blk[e] = (i32)held;
    if (t.rleft[r] == 0) {  // last round: DONE, every block freed
      t.phase[r] = MARS_DONE;
      t.flags[r] = f & ~MARS_F_ACTIVE;
      freeb += held;
      t.kv[r] = 0;
      n_done++;
      b.end_kind[e] = 0;
      b.end_pin[e] = 0;
      continue;
    }
    u8 pin = 0;
    double bb = 0.0, cc = 0.0, dd = 0.0;
    if (decides) decide_retention(c, ctx, kv, total, usage, ema_t, tick_end, pin, bb, cc, dd);
    b.end_pin[e] = pin;  // the `retention` event's payload (sim.py:251-260)
    b.end_b[e] = bb;
    b.end_c[e] = cc;
    b.end_d[e] = dd;
    if (pin && held > 0) {
      t.flags[r] = f | MARS_F_PINNED;
      t.dl[r] = dd;
      t.pb[r] = (i32)held;
      t.plevel[r] = c.policy == POL_MARS && c.coord ? t.level[r] : 0;
      b.end_kind[e] = 1;
    } else {
      freeb += held;
      t.kv[r] = 0;
      b.end_kind[e] = 2;
    }
    t.phase[r] = MARS_TOOL;
  }
  sc->free_blocks = freeb;
  sc->has_ema_blocks = has_ema ? 1 : 0;
  sc->ema_blocks = ema_b;
  w->n_round_end = n_end;
  w->n_done = n_done;
}

// resume_from_tool (sim.py:190-231) for a batch of finished tools (rows are
// distinct): per row in parallel -- round_index + 1, warm iff pinned with a
// deadline >= the finish time (unpin, KV kept), else an expired pin is
// evicted (release_pinned), then submit_round (context += the next round's
// new prefill, remaining_decode, ready_since = now, PREFILL) and on_resume
// (MARS: wait_since = now); the tool-duration EMA is folded in finish order
// on one thread (telemetry.py:96-120).
__global__ void __launch_bounds__(1024) k_resume(Tab t, Cfg c, mars_scalars* sc, i64 n,
                                                 const i64* rows, const double* fin,
                                                 const double* dur, const i32* newp,
                                                 const i32* dec, double now, int* counts,
                                                 u8* o_kind, i32* o_blk, i32* o_ctx, i32* o_need,
                                                 i32* o_proj) {
  __shared__ unsigned long long s_freed;
  __shared__ int s_warm, s_cold, s_ev, s_bad;
  if (threadIdx.x == 0) {
    s_freed = 0;
    s_warm = s_cold = s_ev = s_bad = 0;
  }
  __syncthreads();
  for (i64 i = threadIdx.x; i < n; i += blockDim.x) {
    const i64 r = rows[i];
    const u8 f = t.flags[r];
    const bool pinned = (f & MARS_F_PINNED) != 0;
    const bool warm = pinned && t.dl[r] >= fin[i];
    t.rleft[r] -= 1;
    i32 kv = t.kv[r];
    if (pinned) t.flags[r] = f & ~MARS_F_PINNED;  // unpin, or the return-time eviction
    if (warm) {
      atomicAdd(&s_warm, 1);
    } else {
      if (pinned) {
        atomicAdd(&s_freed, (unsigned long long)t.pb[r]);
        atomicAdd(&s_ev, 1);
        kv = 0;
        t.kv[r] = 0;
      }
      atomicAdd(&s_cold, 1);
    }
    const i64 ctx = (i64)t.ctx[r];
    const i64 need = warm ? (i64)newp[i] : ctx + newp[i];  // resume_cost (engine.py:333-342)
    t.ctx[r] = (i32)(ctx + newp[i]);
    t.rem[r] = dec[i];
    t.rs[r] = now;
    t.phase[r] = MARS_PREFILL;
    if (c.policy == POL_MARS) t.ws[r] = now;  // on_resume (baselines.py:357-360)
    if (ctx + newp[i] - kv != need) atomicAdd(&s_bad, 1);
    // per row, what the reference's log shows for it (sim.py:190-231): the
    // unpin or return-time release, then gpu_submit's payload
    o_kind[i] = warm ? 0 : (pinned ? 2 : 1);
    o_blk[i] = pinned ? t.pb[r] : 0;
    o_ctx[i] = (i32)(ctx + newp[i]);
    o_need[i] = (i32)need;
    o_proj[i] = (i32)(blocks_ceil(c, kv + need) - blocks_ceil(c, kv));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ema = sc->ema_tool;
    bool has = sc->has_ema_tool != 0;
    for (i64 i = 0; i < n; ++i) {
      const double x = dur[i];
      ema = has ? c.ema_alpha * x + (1.0 - c.ema_alpha) * ema : x;
      has = true;
    }
    sc->ema_tool = ema;
    sc->has_ema_tool = has ? 1 : 0;
    sc->free_blocks += (i64)s_freed;
    counts[0] = s_warm;
    counts[1] = s_cold;
    counts[2] = s_ev;
    counts[3] = s_bad;
  }
}

int mars_enqueue_resume(const Tab& t, const Cfg& c, mars_scalars* sc, cudaStream_t s, i64 n,
                        const i64* rows, const double* fin, const double* dur, const i32* newp,
                        const i32* dec, double now, int* counts, u8* o_kind, i32* o_blk,
                        i32* o_ctx, i32* o_need, i32* o_proj) {
  k_resume<<<1, 1024, 0, s>>>(t, c, sc, n, rows, fin, dur, newp, dec, now, counts, o_kind, o_blk,
                              o_ctx, o_need, o_proj);
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// standalone retention batch (mars_retention_batch)
// ---------------------------------------------------------------------------

__global__ void k_retention_batch(Cfg c, i64 n, const i32* ctx, const i32* kv, i64 total,
                                  double usage, double ema, double now, u8* pin, double* bb,
                                  double* cc, double* dd) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    u8 p;
    double x, y, z;
    decide_retention(c, ctx[i], kv[i], total, usage, ema, now, p, x, y, z);
    pin[i] = p;
    bb[i] = x;
    cc[i] = y;
    dd[i] = z;
  }
}

// fetch: every output array of the step into the pinned host arena in one
// launch (blockIdx.y = array), 16-byte stores where both sides allow

// The step's outputs into the mapped host arena, launched by the fetch behind
// the step (no host round trip for the counts first): every CTA lays them out
// from the final Work (out_layout) and copies its share of each array and of
// the Work struct itself (the arena's header).
__global__ void __launch_bounds__(256) k_out_fold(const Work* w, OutSrc S, unsigned char* dst,
                                                  long long cap) {
  __shared__ OutLay L;
  if (threadIdx.x == 0) out_layout(*w, S, cap, &L);
  __syncthreads();
  const unsigned long long nt = (unsigned long long)gridDim.x * blockDim.x;
  const unsigned long long t0 = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (int k = 0; k <= OS_N; ++k) {
    const unsigned char* src;
    unsigned char* out;
    unsigned long long bytes;
    if (k == OS_N) {  // the header, last: the host reads it after the synchronize
      src = (const unsigned char*)w;
      out = dst;
      bytes = sizeof(Work);
    } else {
      if (L.off[k] < 0 || L.bytes[k] == 0) continue;
      src = (const unsigned char*)S.p[k];
      out = dst + L.off[k];
      bytes = (unsigned long long)L.bytes[k];
    }
    const unsigned long long n16 = (((uintptr_t)src | (uintptr_t)out) & 15) == 0 ? bytes / 16 : 0;
    for (unsigned long long i = t0; i < n16; i += nt) ((uint4*)out)[i] = __ldcg((const uint4*)src + i);
    for (unsigned long long i = n16 * 16 + t0; i < bytes; i += nt) out[i] = src[i];
  }
}


__global__ void k_flush(u8* p, i64 n, u32 salt) {
  u32* q = (u32*)p;
  i64 m = n / 4;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (i64)gridDim.x * blockDim.x)
    q[i] = (u32)i ^ salt;
}

// Step head in one node: zero the work area, store this step's input and
// seed the min/max accumulators.  The input arrives as a by-value kernel
// parameter (the graph's node parameters are set before each launch,
// cudaGraphExecKernelNodeSetParams): no PCIe round trip to a mapped host
// copy (round 1-2 read it over PCIe: ~2 us on the step's critical path),
// no memcpy node.  The pre-step scalars the early pack needs are taken
// before the zeroing, stored after it.
__global__ void __launch_bounds__(1024) k_work_init(Work* w, const mars_step_in in,
                                                   const mars_scalars* sc) {
  PTIME(32);
  // k_scan may launch now: it waits (griddepcontrol.wait) for this grid's
  // completion before touching the work area
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  static_assert(sizeof(Work) % 16 == 0, "Work is zeroed in 16-byte words");
  int pre[5] = {0, 0, 0, 0, 0};
  long long pre_q = 0;
  if (threadIdx.x == 32) {
    pre[0] = sc->cpu_overloaded;
    pre[1] = sc->cpu_high_streak;
    pre[2] = sc->cpu_low_streak;
    pre[3] = sc->active_tools;
    pre[4] = sc->queued_tools;
    pre_q = sc->queue_len;
  }
  const size_t n16 = sizeof(Work) / 16;
  uint4* p = (uint4*)w;
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (size_t i = threadIdx.x; i < n16; i += blockDim.x) p[i] = z;
  __syncthreads();
  if (threadIdx.x == 0) w->in = in;  // (constant-bank loads, no local copy)
  if (threadIdx.x < 12) (&w->ref_gand[0][0][0])[threadIdx.x] = ~0ull;
  if (threadIdx.x == 0) {
    w->tmin_win = 0xffffffffu;
    w->tmin_vic = 0xffffffffu;
    w->min_req = 0x7fffffff;
    w->pk_min_req = 0x7fffffff;
  }
  if (threadIdx.x == 32) {
    w->pre_cpu_overloaded = pre[0];
    w->pre_cpu_high_streak = pre[1];
    w->pre_cpu_low_streak = pre[2];
    w->pre_active_tools = pre[3];
    w->pre_queued_tools = pre[4];
    w->pre_queue_len = pre_q;
  }
}

// row scatter / gather for the session-state store (element size 1, 4 or 8)
__global__ void k_scatter(u8* dst, const u8* src, const i64* rows, i64 n, int esz) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    i64 r = rows[i];
    if (esz == 1) dst[r] = src[i];
    else if (esz == 4) ((u32*)dst)[r] = ((const u32*)src)[i];
    else ((u64*)dst)[r] = ((const u64*)src)[i];
  }
}

__global__ void k_gather(u8* dst, const u8* src, const i64* rows, i64 n, int esz) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    i64 r = rows[i];
    if (esz == 1) dst[i] = src[r];
    else if (esz == 4) ((u32*)dst)[i] = ((const u32*)src)[r];
    else ((u64*)dst)[i] = ((const u64*)src)[r];
  }
}

// arrivals appended to the admission list on the device (sim.py:289-301: the
// queue keeps its packed order, new entries go to the end); one CTA
__global__ void __launch_bounds__(1024) k_queue_append(Queue Q, const i32* qsel_p, mars_scalars* sc,
                                                       i64 n, const u32* rows, const i32* req,
                                                       const u8* lng) {
  __shared__ i64 s_len;
  if (threadIdx.x == 0) s_len = sc->queue_len;
  __syncthreads();
  const int sel = *qsel_p;
  u32* qr = PICK2(Q.row, sel);
  i32* qq = PICK2(Q.req, sel);
  u8* ql = PICK2(Q.lng, sel);
  for (i64 i = threadIdx.x; i < n; i += blockDim.x) {
    qr[s_len + i] = rows[i];
    qq[s_len + i] = req[i];
    ql[s_len + i] = lng[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) sc->queue_len = s_len + n;
}

int mars_enqueue_queue_append(cudaStream_t s, const Queue& Q, const i32* qsel, mars_scalars* sc,
                              i64 n, const u32* rows, const i32* req, const u8* lng) {
  k_queue_append<<<1, 1024, 0, s>>>(Q, qsel, sc, n, rows, req, lng);
  return (int)cudaGetLastError();
}

// The drop-in's per-session MLFQ hooks on the device, batched per tick:
// MarsPolicy.on_admit (baselines.py:351-360: level = initial_level of the
// first round's new prefill, scheduler.py:87-97; no promotions, nothing
// served, wait_since = now, the session active) and on_service
// (baselines.py:362-367 -> charge_service scheduler.py:100-108, wait_since =
// tick end) from the device state, or from a given state (undoing the step's
// predicted charge).  Rows are distinct within a batch.
__global__ void k_admit_rows(Tab t, Cfg c, i64 n, const i64* rows, const i32* r0p,
                             const double* now, int* st) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i64 r = rows[i];
    if (r0p[i] < 1) {  // initial_level's ContractViolation
      atomicOr(st, ST_BAD_INPUT);
      continue;
    }
    t.level[r] = (u8)initial_level(c, r0p[i]);
    t.promos[r] = 0;
    t.served[r] = 0;
    t.ws[r] = now[i];
    t.flags[r] = (u8)(t.flags[r] | MARS_F_ACTIVE);
  }
}

__global__ void k_service_rows(Tab t, Cfg c, i64 n, const i64* rows, const i64* tokens,
                               const double* now, const i64* pre /* (served << 8) | level, or null */,
                               int* st) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i64 r = rows[i];
    if (tokens[i] < 0) {  // charge_service's ContractViolation
      atomicOr(st, ST_BAD_INPUT);
      continue;
    }
    u32 lv = pre ? (u32)(pre[i] & 0xff) : (u32)t.level[r];
    i64 served = (pre ? (pre[i] >> 8) : t.served[r]) + tokens[i];
    if (served > c.quotas[lv] && (int)lv < c.num_levels - 1) {
      lv += 1;
      served = 0;
    }
    t.level[r] = (u8)lv;
    t.served[r] = served;
    t.ws[r] = now[i];
  }
}

// MarsPolicy.expired_pins (baselines.py:396-399): the pinned rows whose
// deadline passed (any order; the caller sorts by session id); *cnt counts
// every match, rows past `cap` are not stored
__global__ void k_expired_rows(Tab t, i64 n_rows, double now, u32* out, i64 cap, int* cnt) {
  for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += (i64)gridDim.x * blockDim.x) {
    if ((t.flags[r] & MARS_F_PINNED) && t.dl[r] < now) {
      const int k = atomicAdd(cnt, 1);
      if (k < cap) out[k] = (u32)r;
    }
  }
}

int mars_enqueue_expired_rows(cudaStream_t s, const Tab& t, i64 n_rows, double now, u32* out,
                              i64 cap, int* cnt, int grid) {
  cudaMemsetAsync(cnt, 0, sizeof(int), s);
  k_expired_rows<<<grid, 256, 0, s>>>(t, n_rows, now, out, cap, cnt);
  return (int)cudaGetLastError();
}

int mars_enqueue_admit_rows(cudaStream_t s, const Tab& t, const Cfg& c, i64 n, const i64* rows,
                            const i32* r0p, const double* now, int* st) {
  k_admit_rows<<<(int)((n + 255) / 256), 256, 0, s>>>(t, c, n, rows, r0p, now, st);
  return (int)cudaGetLastError();
}

int mars_enqueue_service_rows(cudaStream_t s, const Tab& t, const Cfg& c, i64 n, const i64* rows,
                              const i64* tokens, const double* now, const i64* pre, int* st) {
  k_service_rows<<<(int)((n + 255) / 256), 256, 0, s>>>(t, c, n, rows, tokens, now, pre, st);
  return (int)cudaGetLastError();
}

// every column of an upsert in one launch: column c's values sit at
// src + L.off[c] (n entries of L.esz[c] bytes), row i goes to rows[i]
__global__ void k_scatter_cols(ScatterCols L, const u8* src, const i64* rows, i64 n) {
  for (i64 j = (i64)blockIdx.x * blockDim.x + threadIdx.x; j < n * L.n;
       j += (i64)gridDim.x * blockDim.x) {
    const int c = (int)(j / n);
    const i64 i = j - (i64)c * n, r = rows[i];
    const u8* sp = src + L.off[c];
    u8* dp = (u8*)L.dst[c];
    const int esz = L.esz[c];
    if (esz == 1) dp[r] = sp[i];
    else if (esz == 4) ((u32*)dp)[r] = ((const u32*)sp)[i];
    else ((u64*)dp)[r] = ((const u64*)sp)[i];
  }
}

int mars_enqueue_scatter_cols(cudaStream_t s, const ScatterCols& L, const void* src,
                              const i64* rows, i64 n) {
  if (n <= 0 || L.n <= 0) return 0;
  i64 g = (n * L.n + 255) / 256;
  if (g > 1184) g = 1184;
  k_scatter_cols<<<(int)g, 256, 0, s>>>(L, (const u8*)src, rows, n);
  return (int)cudaGetLastError();
}

int mars_enqueue_scatter(cudaStream_t s, void* dst, const void* src, const i64* rows, i64 n,
                         int esz) {
  if (n <= 0) return 0;
  int g = (int)((n + 255) / 256);
  if (g > 1184) g = 1184;
  k_scatter<<<g, 256, 0, s>>>((u8*)dst, (const u8*)src, rows, n, esz);
  return (int)cudaGetLastError();
}

int mars_enqueue_gather(cudaStream_t s, void* dst, const void* src, const i64* rows, i64 n,
                        int esz) {
  if (n <= 0) return 0;
  int g = (int)((n + 255) / 256);
  if (g > 1184) g = 1184;
  k_gather<<<g, 256, 0, s>>>((u8*)dst, (const u8*)src, rows, n, esz);
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// host-side launch sequence
// ---------------------------------------------------------------------------

static size_t walk_smem_bytes() {
  size_t s = (size_t)SORT_CAP * (8 + 8 + 4);
  s += (size_t)VSTREAM_CAP * sizeof(VEnt);
  s += (size_t)FS_CAP * (4 + 1) + 16 + (size_t)FS_CAP * 4;
  return s;
}

static size_t sort_smem_bytes() { return (size_t)SORT_CAP * (8 + 8 + 4); }

// k_scan geometry: <= 1 CTA per SM, contiguous row ranges of `chunk` rows
// (a multiple of SCAN_RPT), the digit record in shared memory when it fits
static int g_debug_launch = 0;  // MARS_DEBUG_LAUNCH=1: report each failing launch by name

static void lchk(const char* name) {
  if (!g_debug_launch) return;
  const cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) fprintf(stderr, "mars: launch of %s failed: %s\n", name, cudaGetErrorString(e));
}

static int g_no_pdl = 0;    // MARS_NO_PDL=1: plain stream order between the step head and k_scan
static int g_no_stage = 0;  // MARS_SCAN_NO_STAGE=1: k_scan emits without staging (tests)
static int g_no_ctl_pdl = 0;  // MARS_NO_CTL_PDL=1: k_control in plain stream order behind the push

static void scan_geometry(i64 n, int nsm, int* grid, i64* chunk) {
  i64 g = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (g > nsm) g = nsm;
  if (g > SCAN_TPB) g = SCAN_TPB;
  if (g < 1) g = 1;
  i64 units = (n + 15) / 16;  // TMA rounds start 16-row (16-byte) aligned
  *grid = (int)g;
  *chunk = ((units + g - 1) / g) * 16;
}

static void launch_scan(const LaunchArgs* a, int nsm, cudaStream_t s) {
  int grid;
  i64 chunk;
  scan_geometry(a->n_rows, nsm * SCAN_CTAS_PER_SM, &grid, &chunk);
  Tab t = a->tab;
  Cfg c = a->cfg;
  Work* w = a->work;
  Bufs b = a->bufs;
  mars_scalars* sc = a->sc;
  i64 n = a->n_rows;
  i64* xc = a->x.xc;
  Queue Q = a->queue;
  const i32* qsel = a->qsel;
  int no_stage = g_no_stage;
  // S5 expiry offsets laid out by the scan itself when the expired list is
  // already in rank order (no sort after the scan)
  int kv_fused = (a->kv && !a->exp_sort && !a->exp_may_be_big) ? 1 : 0;
  Kv kv;
  if (a->kv) kv = *a->kv; else memset(&kv, 0, sizeof kv);
  void* args[] = {&t, &c, &w, &b, &sc, &n, &xc, &chunk, &Q, &qsel, &no_stage, &kv, &kv_fused};
  // cooperative, and a programmatic dependent of the kernel before it on the
  // stream (k_work_init): its head and first ring fill overlap the step head
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(SCAN_TPB);
  cfg.dynamicSmemBytes = scan_stage_bytes();
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_no_pdl ? 1 : 2;
  cudaLaunchKernelExC(&cfg, (const void*)k_scan, args);
}

int mars_kernels_init() {
  {
    const char* v = getenv("MARS_SCAN_NO_STAGE");
    g_no_stage = (v && v[0] == '1') ? 1 : 0;
    const char* cp = getenv("MARS_NO_CTL_PDL");
    g_no_ctl_pdl = (cp && cp[0] == '1') ? 1 : 0;
    const char* pd = getenv("MARS_NO_PDL");
    g_no_pdl = (pd && pd[0] == '1') ? 1 : 0;
    const char* d = getenv("MARS_DEBUG_LAUNCH");
    g_debug_launch = (d && d[0] == '1') ? 1 : 0;
  }
  cudaError_t e;
  e = cudaFuncSetAttribute(k_scan, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)scan_stage_bytes());
  if (e != cudaSuccess) return (int)e;
  e = cudaFuncSetAttribute(k_walk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)walk_smem_bytes());
  if (e != cudaSuccess) return (int)e;
  e = cudaFuncSetAttribute(k_control, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sort_smem_bytes());
  if (e != cudaSuccess) return (int)e;
  e = cudaFuncSetAttribute(k_exp_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sort_smem_bytes());
  if (e != cudaSuccess) return (int)e;
  e = cudaFuncSetAttribute(k_pack, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sort_smem_bytes());
  return (int)e;
}

int mars_enqueue_step(const LaunchArgs* a) {
  cudaStream_t s = a->stream, s2 = a->side;
  int launches = 0;
  auto mark = [&](int k, int end, cudaStream_t st) {
    if (!a->prof) return;
    cudaEventRecord(a->prof[2 * k + end], st);
    if (end) a->prof_used[k] = 1;
  };
  const int nsm = a->num_sms;
  const i64 n = a->n_rows;
  const bool sharded = a->sharded != 0;
  if (a->phase != 2) {
    // ---- head: reset, k_scan (+ sharded: export the local admission list)
    if (a->prof)
      for (int k = 0; k < MARS_NUM_KTIMES; ++k) a->prof_used[k] = 0;
    k_work_init<<<1, 1024, 0, s>>>(a->work, *a->host_in, a->sc);
    lchk("k_work_init");
    launches++;
    int scan_sms = nsm;
    if (a->pack_early) {
      // pack_queue's sort on `pack_ctas` SMs (second side stream), k_scan on
      // the rest: both cooperative, together exactly one CTA per SM
      cudaEventRecord(a->ev_head, s);
      cudaStreamWaitEvent(a->side2, a->ev_head, 0);
      Cfg c = a->cfg;
      Work* w = a->work;
      Queue Q = a->queue;
      Lsd L = a->qlsd;
      const i32* qsel = a->qsel;
      int npass = a->queue_passes;
      void* args[] = {&c, &w, &Q, &L, &qsel, &npass};
      mark(4, 0, a->side2);
      cudaLaunchCooperativeKernel((const void*)k_pack, dim3(a->pack_ctas), dim3(1024), args,
                                  sort_smem_bytes(), a->side2);
      lchk("k_pack");
      mark(4, 1, a->side2);
      cudaEventRecord(a->ev_pack, a->side2);
      launches++;
      scan_sms = nsm - a->pack_ctas;
    }
    mark(0, 0, s);
    launch_scan(a, scan_sms, s);
    lchk("k_scan");
    mark(0, 1, s);
    launches++;
    if (sharded) {
      k_export_queue<<<nsm, 256, 0, s>>>(a->queue, a->qsel, a->sc, a->x, a->work);
      lchk("k_export_queue");
      launches++;
    }
    if (a->phase == 1) return launches;
  }
  // ---- tail (sharded: after the counter all-reduce and the list all-gather)
  if (sharded) {
    k_global_control<<<1, 32, 0, s>>>(a->cfg, a->work, a->sc, a->x);
    k_build_global_queue<<<nsm, 256, 0, s>>>(a->work, a->x, a->queue, a->qsel);
    lchk("k_global_control / k_build_global_queue");
    launches += 2;
  }
  // The walk runs on the side stream, concurrently with the main stream's
  // expired-pin rank sort (tables that are not rank-ordered) and control plane
  // (pack_queue sort, admission): the control plane is the longer branch, and
  // a kernel on the stream that launched k_scan starts sooner than one behind
  // a fork event.  The two grid-wide (cooperative) kernels stay serialised on
  // one stream; each leaves an SM for the walk.  The walk reads no state
  // admission writes unless an admitted session can enter the window, and
  // then waits for the admission's completion flag (k_walk, admit_async).
  // The KV journal apply needs the walk's journal and the rank-ordered
  // expired pins: after the join.
  const bool kv_fused = a->kv && !a->exp_sort && !a->exp_may_be_big;
  cudaEventRecord(a->ev_fork, s);
  cudaStreamWaitEvent(s2, a->ev_fork, 0);
  mark(3, 0, s2);
  k_walk<<<1, WALK_TPB, walk_smem_bytes(), s2>>>(a->tab, a->cfg, a->work, a->bufs, a->sc, n,
                                                 a->control_possible);
  lchk("k_walk");
  launches++;
  mark(3, 1, s2);
  // Host enqueue order matters beyond the streams' own order: streams can
  // share a hardware work queue (CUDA_DEVICE_MAX_CONNECTIONS), and there an
  // entry that waits for the walk would block everything queued after it --
  // the control plane the walk may be waiting for included.  So nothing that
  // depends on the walk is enqueued before the control plane is.
  if (kv_fused) {
    // S5, expired list in rank order (k_scan laid out the frees): the expired
    // tables go back to the free stack on the main stream beside the walk, as
    // a programmatic dependent of the scan (resident and waiting before the
    // scan ends).  On the pack's stream instead -- beside the control plane
    // rather than in front of it -- both slowed down (r2: 73.0 vs 71.6 us):
    // the push and the admission are latency-bound on the same memory.
    mark(5, 0, s);
    mars_kv_enqueue_exp_free(*a->kv, s, a->work, a->bufs, nsm, /*offsets_done=*/true,
                             /*pdl=*/!g_no_pdl);
    mark(5, 1, s);
    launches++;
    cudaEventRecord(a->ev_kvx, s);
  }
  // the early pack's SMs return before any other grid-wide kernel starts
  if (a->pack_early) cudaStreamWaitEvent(s, a->ev_pack, 0);
  if (a->exp_sort || a->exp_may_be_big) {
    mark(1, 0, s);
    if (a->exp_sort) {
      k_exp_small<<<1, 1024, sort_smem_bytes(), s>>>(a->work, a->bufs, a->xlsd);
      lchk("k_exp_small");
      launches++;
    }
    if (a->exp_may_be_big) {
      launch_lsd(a->xlsd, a->work, 1, 4, nsm - 1, s);  // the walk keeps one SM
      launches++;
      k_exp_gather<<<nsm, 256, 0, s>>>(a->work, a->bufs, a->xlsd);
      lchk("k_lsd_coop / k_exp_gather");
      launches++;
    }
    mark(1, 1, s);
  }
  if (a->control_possible) {
    i64 lgq = (a->queue_upper + a->ctl_per_cta - 1) / a->ctl_per_cta;  // list entries per CTA
    int lg = (int)(lgq < 1 ? 1 : (lgq > nsm - 1 ? nsm - 1 : lgq));  // the walk keeps one SM
    Tab t = a->tab;
    Cfg c = a->cfg;
    Work* w = a->work;
    Bufs b = a->bufs;
    Queue Q = a->queue;
    Lsd L = a->qlsd;
    mars_scalars* sc = a->sc;
    i32* qsel = a->qsel;
    Queue G = a->gq;
    Xchg x = a->x;
    int npass = a->queue_passes;
    void* args[] = {&t, &c, &w, &b, &Q, &L, &sc, &qsel, &G, &x, &npass};
    mark(2, 0, s);
    // right behind the S5 push: a programmatic dependent of it (launched once
    // every push CTA is past its wait for the scan, so the scan's results are
    // visible; the control plane reads nothing the push writes), its CTAs
    // placed as the push's drain instead of after the push's end
    const bool ctl_pdl = kv_fused && !a->exp_sort && !a->exp_may_be_big && !g_no_pdl &&
                         !g_no_ctl_pdl && !a->prof;
    cudaLaunchConfig_t cc = {};
    cc.gridDim = dim3(lg);
    cc.blockDim = dim3(1024);
    cc.dynamicSmemBytes = sort_smem_bytes();
    cc.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cc.attrs = at;
    cc.numAttrs = ctl_pdl ? 2 : 1;
    cudaLaunchKernelExC(&cc, (const void*)k_control, args);
    lchk("k_control");
    mark(2, 1, s);
    launches++;
  }
  if (a->kv && !kv_fused) {
    // S5, expired list sorted after the scan: the expired tables return to
    // the free stack (segment pushes by the whole grid) after the control
    // plane, while the walk is still running.  (Not on a third stream beside the control plane: the walk may
    // spin on the admission's completion flag, and with the early pack on the
    // second side stream that arrangement was seen to starve k_control, r2.)
    mark(5, 0, s);
    mars_kv_enqueue_exp_free(*a->kv, s, a->work, a->bufs, nsm, /*offsets_done=*/false,
                             /*pdl=*/false);
    mark(5, 1, s);
    launches += 2;
  }
  // the walk's stream, behind the walk: (S5, fused) its journal, after the
  // expired tables' pushes, beside the control plane; then the join
  if (kv_fused) {
    cudaStreamWaitEvent(s2, a->ev_kvx, 0);
    mark(6, 0, s2);
    mars_kv_enqueue_apply_step(*a->kv, s2, a->work, a->bufs, 1);
    mark(6, 1, s2);
    launches++;
  }
  cudaEventRecord(a->ev_join, s2);
  cudaStreamWaitEvent(s, a->ev_join, 0);
  if (a->advance) {
    k_advance<<<1, 1024, 0, s>>>(a->tab, a->cfg, a->work, a->bufs, a->sc);
    launches++;
  }
  if (a->kv && (!kv_fused || a->advance)) {  // (fused: only the tick tail's frees are left)
    if (!kv_fused) mark(6, 0, s);
    mars_kv_enqueue_apply_step(*a->kv, s, a->work, a->bufs, kv_fused ? 2 : 3);
    if (!kv_fused) mark(6, 1, s);
    launches++;
  }
#ifdef MARS_PHASE_TIMING
  k_ptime_dump<<<1, 1, 0, s>>>();
  mars_kv_ptime_dump(s);
#endif
  return launches;
}

int mars_enqueue_out_fold(cudaStream_t s, const Work* w, const OutSrc& S, unsigned char* arena,
                          long long cap) {
  static int ctas = -1;
  if (ctas < 0) {
    const char* v = getenv("MARS_FOLD_CTAS");
    ctas = v ? atoi(v) : 296;
    if (ctas < 1) ctas = 1;
  }
  k_out_fold<<<ctas, 256, 0, s>>>(w, S, arena, cap);
  return (int)cudaGetLastError();
}

int mars_enqueue_retention(const Cfg& c, cudaStream_t s, i64 n, const i32* ctx, const i32* kv,
                           i64 total, double usage, double ema, double now, u8* pin, double* bb,
                           double* cc, double* dd) {
  int g = (int)((n + 255) / 256);
  if (g > 1184) g = 1184;
  if (g < 1) g = 1;
  k_retention_batch<<<g, 256, 0, s>>>(c, n, ctx, kv, total, usage, ema, now, pin, bb, cc, dd);
  return (int)cudaGetLastError();
}

int mars_enqueue_flush(cudaStream_t s, u8* p, i64 n, u32 salt) {
  cudaError_t prior = cudaGetLastError();
  if (prior != cudaSuccess) return 1000 + (int)prior;  // an earlier call left an error
  k_flush<<<1184, 256, 0, s>>>(p, n, salt);
  return (int)cudaGetLastError();
}

// Every kernel of this file loaded now (CUDA loads modules lazily by default):
// a kernel first launched while the walk spins on the control plane's flag
// must not wait on its own loading (which can wait for the device).
const void* mars_work_init_fn() { return (const void*)k_work_init; }

int mars_kernels_preload() {
  cudaFuncAttributes fa;
  const void* fns[] = {(const void*)k_advance, (const void*)k_build_global_queue,
                       (const void*)k_out_fold,
                       (const void*)k_control, (const void*)k_exp_gather,
                       (const void*)k_exp_small, (const void*)k_export_queue,
                       (const void*)k_flush, (const void*)k_gather,
                       (const void*)k_global_control, (const void*)k_lsd_coop,
                       (const void*)k_pack, (const void*)k_resume,
                       (const void*)k_retention_batch, (const void*)k_scan,
                       (const void*)k_scatter, (const void*)k_walk, (const void*)k_work_init,
                       (const void*)k_queue_append, (const void*)k_admit_rows,
                       (const void*)k_service_rows, (const void*)k_expired_rows,
                       (const void*)k_scatter_cols};
  for (const void* f : fns) {
    cudaError_t e = cudaFuncGetAttributes(&fa, f);
    if (e != cudaSuccess) return (int)e;
  }
  return 0;
}
