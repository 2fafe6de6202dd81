// Internal device-side layout of the B200 MARS step.  See DESIGN.md for the
// data layout and the kernel pipeline; include/mars_b200.h for the C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mars_b200.h"

typedef uint8_t u8;
typedef uint16_t u16;
typedef uint32_t u32;
typedef uint64_t u64;
typedef int32_t i32;
typedef int64_t i64;

#define HIST_BINS 4096
#define WIN_MAX 128
#define SORT_CAP 4096         // bitonic sort capacity of the single-CTA selector
#define VSEL 512              // victim-stream target length (prefix of reclaim order): covers
                              // every victim one step can take (<= max_dec + budget/bs + window)
                              // plus the window rows a claim may skip
#define VSTREAM_CAP 1024      // victim stream entries kept in shared memory
#define REF_STOP 256          // grid radix refinement stops at a group this small
#define REF_TRIG_W 1024       // window candidates beyond this are refined in k_scan
#define REF_TRIG_V VSTREAM_CAP
#define VR_CAP 4096           // refined victim list capacity (<= VSEL + REF_STOP used)
#define LSD_G 592             // max CTAs of the cooperative LSD radix sort (>= #SMs)
#define SCAN_RPT 4            // consecutive rows per thread in the table scans
#define MAX_SCAN_CTAS 1024    // upper bound of k_scan's grid
#define ROW_PAD 2048          // row capacity is padded to this multiple
#define MAXH 0x0FFFFFFFull    // 28-bit complement base for -blocks in victim keys
#define PACK_SEG_ENTRIES 6144 // list entries one k_pack CTA ranks per pass (LSD_SEG_J x 1024)

// pack modes (control.py:101-122)
#define PACK_ASC 0
#define PACK_DESC 1
#define PACK_FF 2

// step status bits
#define ST_OK 0
#define ST_QUEUE_MISMATCH 1
#define ST_WALK_OVERFLOW 2
#define ST_BAD_INPUT 4

// policies (mars_config.policy)
#define POL_MARS MARS_POLICY_MARS
#define POL_FCFS MARS_POLICY_FCFS
#define POL_PP MARS_POLICY_PROGRAM_PRIORITY
#define POL_STATIC_TTL MARS_POLICY_STATIC_TTL
#define POL_DYNAMIC_TTL MARS_POLICY_DYNAMIC_TTL

// device copy of the configuration (mars_config + derived)
struct Cfg {
  i32 bs, bs_shift, budget, window, max_dec, num_levels, max_promos, hyst, w_min;
  i32 coord, cosched;
  i32 policy, strict;  // strict: head-of-line blocking in the prefill pass
  double ttl_s, ttl_mult;
  i64 bounds[4], quotas[4];
  double tick_s, prefill_rate, promo_wait, slack, horizon, pw_clip;
  double cpu_hi, cpu_lo, kv_hi, kv_lo, ema_alpha, tool_prior;
  double ai, md, ctl_interval, init_window, oversub, reserve, long_frac;
  i32 ref_trig_w, ref_trig_v, stream_cap;  // refinement triggers, victim stream length
};

// device column pointers (the session-state store, SoA in HBM)
struct Tab {
  u8 *phase, *flags, *level, *promos, *plevel;
  double *rs, *ws, *dl, *arr;
  i32 *ctx, *kv, *rem, *pb, *req, *r0p, *r0d, *pre;
  i64 *served;
  u32 *rank;
  i32 *rleft;  // rounds after the current one
  int16_t *winpos;  // row -> window index during the walk, -1 otherwise
  i64 cap;
};

// queue (admission list), double-buffered: q[sel] is current
struct Queue {
  u32 *row[2];
  i32 *req[2];
  u8 *lng[2];
  u32 *gpos[2];  // sharded mode: global list position of each local entry
  i64 cap;
};

// sharded (multi-GPU) exchange: counters all-reduced, queue entries all-gathered
#define XC_N 8          // i64 counters: free, total, active, qlen
#define XQ_NONE 0xffffffffu
struct Xchg {
  i64* xc;            // [XC_N] local, then (after the all-reduce) global sums
  u64* xsend;         // [1 + cap] : header count, then one gpos<<32 | req<<1 | long per entry
  u64* xrecv;         // [world][1 + cap]
  u32* gq_row;        // global queue by gpos: own local row or XQ_NONE
  i32* gq_req;
  u8* gq_lng;
  u32* adm_idx;       // packed index of each own admitted entry
  i32 world, rank;
  i64 cap;            // per-rank queue capacity
};

// generic multi-CTA LSD radix sort scratch (u64 keys, u32 vals)
struct Lsd {
  u64 *k[2];
  u32 *v[2];
  u32 *cnt;      // [256][LSD_G] counts, then offsets
  i64 cap;
};

// fixed-size per-step work area (device memory, zeroed at step start)
struct Work {
  mars_step_in in;
  // K_A accumulators
  unsigned long long exp_blocks;
  i32 n_exp, n_active, n_queued, n_long_q, n_ready, n_promoted, n_victims, n_boundary;
  i32 tab_long_q, tab_max_req, tab_min_req;  // queue stats from the table scan
  i32 max_req, min_req;
  u32 tmin_win, tmin_vic;
  u32 hist_win[HIST_BINS];
  u32 hist_vic[HIST_BINS];
  // thresholds
  i32 t_win, t_vic;
  i32 n_win_cand_expected, n_vic_cand_expected;
  // candidate counts (K_C / K_AP appends)
  i32 n_wc, n_vc, n_ret;
  // control plane
  i32 pack_mode, need_seed, big_queue;
  i64 qlen;
  double ff_median;
  i32 lsd_cur, lsd_skip[8], lsd_in[8];
  u64 lsd_maxkey;
  u64 lsd_raw_ptr;  // queue pass 0 reads req[] straight from the admission list
  i32 lsd_big, lsd_n;
  i32 xlsd_cur, xlsd_skip[8], xlsd_in[8];
  u64 xlsd_maxkey;
  i32 xlsd_big, xlsd_n;
  i64 limit, slots, take;
  long long projected;
  // the telemetry the control plane sees: the replica's probe, or the pooled
  // (all-reduced) view in sharded mode
  i64 adm_avail, adm_total, adm_active;
  double adm_usage;
  i32 n_adm_own, n_res_own;
  i64 global_residual;
  // plan
  i32 n_window, n_dec, n_pre, n_evict, n_journal;
  i64 total_tokens;
  i64 free_after_expiry;
  i32 status;
  i32 walk_slow;
  i32 n_queued_kv;  // queued rows holding KV (admission then touches reclaim state)
  u32 admit_done;   // set by k_control after admission; k_walk may wait on it
  u32 adm_ctas;     // k_control CTAs past admission (the last one publishes)
  u32 adm_next;     // admission: next 1024-entry chunk of the packed prefix to take
  u32 adm_pad[2];   // (Work stays a whole number of 16-byte words)
  // grid radix refinement of the candidate lists (k_scan phase 3): per list
  // (0 window, 1 victims) three rotating 256-bin histograms and group AND /
  // ORs, and the final bound: the refined list holds the keys with
  // (key >> ref_s) <= (ref_p >> ref_s)
  u32 ref_hist[2][3][256];
  unsigned long long ref_gand[2][3][2], ref_gor[2][3][2];  // per round: the group's AND / OR
  unsigned long long ref_p[2][2];
  i32 ref_on[2], ref_s[2];
  i32 n_wr, n_vr;     // refined list lengths
  i32 n_fullscan;     // exact full-table reclaimer passes taken by the walk
  i32 ref_iters;
  i32 vic_on;         // k_scan built a victim stream (the free pool may not cover a plan)
  i32 vs_on;          // ... and ranked it into the stream order (vs_*)
  i32 ref_pad[2];
  u32 ref_pad2[16];
  i32 n_finish;
  i32 sort_path;    // pack_queue: 1 grid LSD sort, 2 one CTA, 3 early grid LSD (k_pack)
  i32 n_round_end, n_done;  // MARS_MODE_ADVANCE: rounds that ended, sessions that finished
  i64 free_after_plan;      // the pool's free blocks after the plan (before the tick's tail)
  // pre-step copies (k_work_init) for k_pack, which runs concurrently with
  // k_scan (whose CTA 0 rewrites the scalars)
  i32 pre_cpu_overloaded, pre_cpu_high_streak, pre_cpu_low_streak;
  i32 pre_active_tools, pre_queued_tools;
  i64 pre_queue_len;
  // k_pack results: the packed permutation is L.v[pk_cur], keys L.k[pk_cur]
  i32 pk_done, pk_mode, pk_cur, pk_n_long, pk_max_req, pk_min_req;
};

// variable-length step buffers
struct Bufs {
  // expired pins: row order (k_scan), rank order (k_exp_*)
  i32 *tile_cnt;             // per-k_scan-CTA expired counts
  i64 *tile_kv;              // per-k_scan-CTA S5 sums of the expired tables: segments, loose IDs, tail chunks
  u32 *row_dig;              // k_scan: per CTA, the compacted rows' digit records
  u32 *cand_row;             // k_scan: per CTA, the compacted rows (row order)
  u32 *exp_row; i32 *exp_blk; u32 *exp_rank;
  u32 *exp_row_sorted; i32 *exp_blk_sorted;
  // window candidates
  u64 *wc_hi, *wc_lo; u32 *wc_row;
  // victim candidates: the policy's 128-bit reclaim key (vc_key, vc_kl), the
  // window key of running rows (eligibility), row, blocks
  u64 *vc_key, *vc_kl, *vc_whi, *vc_wlo; u32 *vc_row; i32 *vc_blk;
  // the same two lists after the grid radix refinement (k_scan phase 3)
  u64 *wr_hi, *wr_lo; u32 *wr_row;
  u64 *vr_key, *vr_kl, *vr_whi, *vr_wlo; u32 *vr_row; i32 *vr_blk;
  // the victim stream in reclaim order (k_scan's grid rank), VSTREAM_CAP entries
  u64 *vs_key, *vs_kl, *vs_whi, *vs_wlo; u32 *vs_row; i32 *vs_blk;
  // retention results
  u32 *ret_row; u8 *ret_pin; double *ret_b, *ret_c, *ret_d;
  // admission
  u32 *admitted;
  // plan outputs
  u32 *win_rows, *dec_rows, *pre_rows; i32 *pre_grant;
  u8 *dec_level, *pre_level;
  i64* svc_pre;                // (served << 8) | level before the tick-end charge
  u32 *fin_row; u8 *fin_pin; double *fin_b, *fin_c, *fin_d;
  u32 *end_row; u8 *end_kind;  // MARS_MODE_ADVANCE: rounds that ended, decode order
  i32 *end_blk; u8 *end_pin; double *end_b, *end_c, *end_d;  // blocks pinned/freed, decision
  u8 *pre_done;                // MARS_MODE_ADVANCE: the grant finished the prefill
  u32 *ev_row; u8 *ev_kind; i32 *ev_blk;
  u8 *j_op; u32 *j_row; i32 *j_n;
  i64 ev_cap, j_cap;
  // flush scratch
  u8 *flush; i64 flush_bytes;
};

// ---------------------------------------------------------------------------
// key helpers
// ---------------------------------------------------------------------------

// total order on finite doubles as an unsigned integer; -0.0 folds onto +0.0
// (Python compares them equal, the session-id tie-break then decides)
__device__ __forceinline__ u64 ord_f64(double x) {
  x = x + 0.0;
  u64 b = (u64)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// window order key (baselines.py:374-377): (level, ready_since, session_id) or,
// coordinator off, (arrival_time, session_id).  98 significant bits.
__device__ __forceinline__ void window_key(u32 level, double t, u32 rank, u64& hi, u64& lo) {
  u64 o = ord_f64(t);
  hi = ((u64)level << 62) | (o >> 2);
  lo = ((o & 3ull) << 62) | (u64)rank;
}

// monotone 12-bit digit of the window key
__device__ __forceinline__ u32 window_digit(u32 level, double t, double scale) {
  double y = t * scale;
  u32 b = (y >= 1023.0) ? 1023u : (y > 0.0 ? (u32)y : 0u);
  return (level << 10) | b;
}

// program_priority order key (baselines.py:170-171): (Call.served_tokens,
// arrival_time, session_id); served_tokens < 2^32 (k_scan flags larger ones)
__device__ __forceinline__ void pp_window_key(i64 served, double arr, u32 rank, u64& hi, u64& lo) {
  const u64 o = ord_f64(arr);
  const u64 s = served <= 0 ? 0ull : (served >= 0xffffffffll ? 0xffffffffull : (u64)served);
  hi = (s << 32) | (o >> 32);
  lo = (o << 32) | (u64)rank;
}

__device__ __forceinline__ u32 blocks_bucket(i64 h);

// monotone 12-bit digit of the program_priority key: a log-scale bucket of
// served_tokens (exact below 8), refined by arrival only where the bucket is
// a single served value
__device__ __forceinline__ u32 pp_window_digit(i64 served, double arr, double scale) {
  const u32 b = blocks_bucket(served);
  u32 sub = 0;
  if (served < 8) {
    const double y = arr * scale;
    sub = ((y >= 1023.0) ? 1023u : (y > 0.0 ? (u32)y : 0u)) >> 6;
  }
  return (b << 4) | sub;
}

// the policy's window order key for one row (baselines.py:104-105, 170-171,
// 374-377)
__device__ __forceinline__ void row_window_key(const Cfg& c, u32 level, double rs, double arr,
                                               i64 served, u32 rank, u64& hi, u64& lo) {
  if (c.policy == POL_PP)
    pp_window_key(served, arr, rank, hi, lo);
  else if (c.coord)
    window_key(level, rs, rank, hi, lo);
  else
    window_key(0u, arr, rank, hi, lo);
}

// policies that pin KV at tool boundaries (and so expire and reclaim pins)
__device__ __forceinline__ bool policy_pins(const Cfg& c) {
  return c.policy == POL_MARS || c.policy == POL_STATIC_TTL || c.policy == POL_DYNAMIC_TTL;
}

// monotone non-decreasing 8-bit bucket of a block count
__device__ __forceinline__ u32 blocks_bucket(i64 h) {
  if (h <= 0) return 0;
  if (h >= (1ll << 31)) return 255;
  u32 x = (u32)h;
  int e = 31 - __clz(x);
  if (e < 3) return x;
  return 8u * (u32)(e - 2) + ((x >> (e - 3)) & 7u);
}

// reclaim order (scheduler.py:249-259): pinned before running, expired pins
// first, then lowest level (largest level value) first, then largest
// footprint, then session id.
__device__ __forceinline__ u64 victim_key(bool running, bool nonexp, u32 level, i64 blocks,
                                          u32 rank) {
  u64 b = (blocks > (i64)MAXH) ? MAXH : (u64)blocks;
  return ((u64)running << 63) | ((u64)(nonexp ? 1 : 0) << 62) | ((u64)(3u - level) << 60) |
         ((MAXH - b) << 32) | (u64)rank;
}

__device__ __forceinline__ u32 victim_digit(bool running, bool nonexp, u32 level, i64 blocks) {
  return ((running ? 1u : 0u) << 11) | ((nonexp ? 1u : 0u) << 10) | ((3u - level) << 8) |
         (255u - blocks_bucket(blocks));
}

// monotone non-decreasing 11-bit bucket of a non-negative count: exact below
// 64, then 64 sub-buckets per octave (values are clamped to 2^32 - 1)
__device__ __forceinline__ u32 log_bucket11(i64 v) {
  if (v <= 0) return 0;
  const u64 x = v >= 0xffffffffll ? 0xffffffffull : (u64)v;
  if (x < 64) return (u32)x;
  const int e = 63 - __clzll((long long)x);
  return 64u * (u32)(e - 5) + (u32)((x >> (e - 6)) & 63u);
}

// The policy's reclaim order as one unique 128-bit key (kh, kl), pinned
// victims first (bit 127 clear):
//  mars     pinned (expired first, -level, -blocks, sid), then running
//           (-level, -blocks, sid)             scheduler.py:249-259
//  fcfs/ttl running: latest arrival first      baselines.py:120-130, 288-298
//  program_priority running: most service first baselines.py:176-186
//  ttl      pinned (expired first, deadline, -blocks, sid)  baselines.py:268-287
// `lv` is the row's MLFQ level (0 with the coordinator off).
__device__ __forceinline__ void run_reclaim_key(int policy, u32 lv, i64 held, double arr,
                                                i64 served, u32 rank, u64& kh, u64& kl) {
  if (policy == POL_MARS) {
    kh = victim_key(true, false, lv, held, rank);
    kl = 0;
  } else if (policy == POL_PP) {
    const u64 su = served <= 0 ? 0ull : (u64)served;
    kh = (1ull << 63) | (0x3fffffffffffffffull - (su & 0x3fffffffffffffffull));
    kl = rank;
  } else {
    const u64 o = ~ord_f64(arr);
    kh = (1ull << 63) | (o >> 1);
    kl = ((o & 1ull) << 63) | (u64)rank;
  }
}

__device__ __forceinline__ void pin_reclaim_key(int policy, bool nonexp, u32 plevel, i64 pb,
                                                double dl, u32 rank, u64& kh, u64& kl) {
  if (policy == POL_MARS) {
    kh = victim_key(false, nonexp, plevel, pb, rank);
    kl = 0;
  } else {
    const u64 o = ord_f64(dl);
    const u64 bb = pb > (i64)MAXH ? MAXH : (u64)(pb < 0 ? 0 : pb);
    kh = ((u64)(nonexp ? 1 : 0) << 62) | (o >> 2);
    kl = ((o & 3ull) << 62) | ((MAXH - bb) << 32) | (u64)rank;
  }
}

// 12-bit digits monotone in those keys (the k_scan histograms)
__device__ __forceinline__ u32 pin_reclaim_digit(int policy, bool nonexp, u32 plevel, i64 pb,
                                                 double dl, double now) {
  if (policy == POL_MARS) return victim_digit(false, nonexp, plevel, pb);
  const double y = (dl - now + 64.0) * 8.0;  // deadline, 1/8 s over now +- 64 s
  const u32 b = (y >= 1023.0) ? 1023u : (y > 0.0 ? (u32)y : 0u);
  return ((nonexp ? 1u : 0u) << 10) | b;
}

__device__ __forceinline__ u32 run_reclaim_digit(int policy, u32 lv, i64 held, double arr,
                                                 i64 served, double ascale) {
  if (policy == POL_MARS) return victim_digit(true, false, lv, held);
  if (policy == POL_PP) return (1u << 11) | (2047u - log_bucket11(served));
  const double y = arr * ascale;  // arrival over [0, now], 2048 buckets
  const u32 b = (y >= 2047.0) ? 2047u : (y > 0.0 ? (u32)y : 0u);
  return (1u << 11) | (2047u - b);
}

// 64-bit division kept out of line: the single-CTA kernels pay for every
// instruction-cache line they touch, so rarely taken slow paths stay compact
static __device__ __noinline__ i64 div64_slow(i64 a, i64 b) { return a / b; }
static __device__ __noinline__ i64 mod64_slow(i64 a, i64 b) { return a % b; }
__device__ __forceinline__ i64 ceil_div64(i64 a, i64 b) { return div64_slow(a + b - 1, b); }

// blocks_for_tokens (engine.py:112-113) for x >= 0: a shift when the block
// size is a power of two (no 64-bit division on the hot paths)
__device__ __forceinline__ i64 blocks_ceil(const Cfg& c, i64 x) {
  if (c.bs_shift >= 0) return (x + (i64)c.bs - 1) >> c.bs_shift;
  return ceil_div64(x, c.bs);
}
// (x // bs) * bs for x >= 0
__device__ __forceinline__ i64 blocks_floor_tokens(const Cfg& c, i64 x) {
  if (c.bs_shift >= 0) return x & ~((i64)c.bs - 1);
  return div64_slow(x, c.bs) * c.bs;
}
__device__ __forceinline__ bool block_aligned(const Cfg& c, i64 x) {
  return c.bs_shift >= 0 ? (x & ((i64)c.bs - 1)) == 0 : mod64_slow(x, c.bs) == 0;
}

// held_blocks / blocks_for_tokens (engine.py:112-113, 314-315) for kv >= 0
__device__ __forceinline__ i64 held_blocks(const Cfg& c, i32 kv) {
  if (c.bs_shift >= 0) return (i64)(((u32)kv + (u32)c.bs - 1u) >> c.bs_shift);
  return (i64)(((u32)kv + (u32)c.bs - 1u) / (u32)c.bs);
}

__device__ __forceinline__ bool key_lt(u64 ah, u64 al, u64 bh, u64 bl) {
  return ah < bh || (ah == bh && al < bl);
}

// initial_level (scheduler.py:87-97)
__device__ __forceinline__ u32 initial_level(const Cfg& c, i64 tokens) {
  for (int i = 0; i < c.num_levels; ++i)
    if (tokens <= c.bounds[i]) return (u32)i;
  return (u32)(c.num_levels - 1);
}

// pressure_weight + decide_retention (scheduler.py:183-213).  Operation order
// is the reference's, and this file is compiled with --fmad=false, so the
// results are bit-identical to CPython's IEEE doubles.
__device__ __forceinline__ void decide_retention(const Cfg& c, i64 context, i64 kv,
                                                 i64 total_blocks, double usage, double ema,
                                                 double now, u8& pin, double& benefit,
                                                 double& cost, double& deadline) {
  if (c.policy == POL_STATIC_TTL || c.policy == POL_DYNAMIC_TTL) {
    // TtlPolicy.retention_decision (baselines.py:238-243): always pin
    pin = 1;
    benefit = 0.0;
    cost = 0.0;
    deadline = (c.policy == POL_STATIC_TTL) ? now + c.ttl_s : now + c.ttl_mult * ema;
    return;
  }
  benefit = (double)context / c.prefill_rate;
  i64 foot = blocks_ceil(c, kv);
  double pw;
  if (usage >= 1.0) {
    pw = c.pw_clip;
  } else {
    double inv = 1.0 / (1.0 - usage);
    pw = (c.pw_clip < inv) ? c.pw_clip : inv;
  }
  cost = ((double)foot / (double)total_blocks) * ema * pw;
  pin = (benefit > cost && ema <= c.horizon) ? 1 : 0;
  double d = ema * c.slack;
  deadline = now + ((c.horizon < d) ? c.horizon : d);
}
