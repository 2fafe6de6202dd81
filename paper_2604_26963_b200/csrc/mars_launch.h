// Host-side launch interface between the C ABI (mars_abi.cu) and the kernels.
#pragma once

#include "mars_internal.cuh"
#include "mars_kv.h"

// The step's outputs in the pinned host arena, laid out by the device
// (k_out_fold, launched by mars_step_fetch behind the step) and parsed by the
// host after one stream synchronize: the Work struct at offset 0, then every
// output array, 16-byte aligned, in this slot order.  The same function runs
// on both sides.
enum {
  OS_EXP_ROW, OS_EXP_BLK, OS_ADM, OS_ADM_IDX, OS_WIN, OS_DEC, OS_PRE, OS_PRE_GRANT,
  OS_EV_ROW, OS_EV_KIND, OS_EV_BLK, OS_J_OP, OS_J_ROW, OS_J_N, OS_RET_ROW, OS_RET_PIN,
  OS_RET_B, OS_RET_C, OS_RET_D, OS_DEC_LEVEL, OS_PRE_LEVEL, OS_SVC_PRE, OS_END_ROW,
  OS_END_KIND, OS_END_BLK, OS_END_PIN, OS_END_B, OS_END_C, OS_END_D, OS_PRE_DONE,
  OS_FIN_ROW, OS_FIN_PIN, OS_FIN_B, OS_FIN_C, OS_FIN_D, OS_N
};
struct OutSrc {
  const void* p[OS_N];  // device sources per slot
  long long ev_cap, j_cap;
  int coord;
};
struct OutLay {
  long long off[OS_N];    // byte offset in the arena (-1: the arena is too small)
  long long bytes[OS_N];
};
#define OUT_HDR (((long long)sizeof(Work) + 15) & ~15ll)

__host__ __device__ inline void out_layout(const Work& w, const OutSrc& S, long long cap,
                                           OutLay* L) {
  const int mode = w.in.mode;
  const bool sharded = (mode & MARS_MODE_SHARDED) != 0;
  const long long n_adm = sharded ? (long long)w.n_adm_own : (long long)w.take;
  const long long ne = w.n_evict < S.ev_cap ? w.n_evict : S.ev_cap;
  const long long nj = w.n_journal < S.j_cap ? w.n_journal : S.j_cap;
  const long long ret = w.n_ret, ren = w.n_round_end, fin = w.n_finish;
  const long long dec = w.n_dec, pre = w.n_pre, ex = w.n_exp;
  const long long sz[OS_N] = {
      ex * 4, ex * 4, n_adm * 4, sharded ? n_adm * 4 : 0, (long long)w.n_window * 4, dec * 4,
      pre * 4, pre * 4, ne * 4, ne, ne * 4, nj, nj * 4, nj * 4, ret * 4, ret, ret * 8, ret * 8,
      ret * 8, dec, pre, ((mode & MARS_MODE_SERVICE) && S.coord) ? (dec + pre) * 8 : 0, ren * 4,
      ren, ren * 4, ren, ren * 8, ren * 8, ren * 8, (mode & MARS_MODE_ADVANCE) ? pre : 0,
      fin * 4, fin, fin * 8, fin * 8, fin * 8};
  long long off = OUT_HDR;
  for (int i = 0; i < OS_N; ++i) {
    off = (off + 15) & ~15ll;
    L->bytes[i] = sz[i];
    L->off[i] = off + sz[i] <= cap ? off : -1;
    off += sz[i];
  }
}

struct LaunchArgs {
  cudaStream_t stream, side, side2;
  cudaEvent_t ev_fork, ev_join, ev_head, ev_pack, ev_kvx;
  Tab tab;
  Cfg cfg;
  Work* work;
  Bufs bufs;
  mars_scalars* sc;
  Queue queue;
  Lsd qlsd, xlsd;
  i32* qsel;
  const mars_step_in* host_in;
  i64 n_rows;
  int num_sms;
  int control_possible;  // the step may run the control plane
  int queue_passes;      // LSD passes needed for the largest queue key (0 = small only)
  i64 queue_upper;       // upper bound of the queue length at step start
  int ctl_per_cta;       // admission-list entries per k_control CTA (grid sizing)
  int pack_early;        // pack_queue's sort runs concurrently with k_scan (k_pack)
  int pack_ctas;         // its grid; k_scan then takes the other SMs
  int advance;           // MARS_MODE_ADVANCE: k_advance after the join
  int exp_sort;          // expired pins need a rank sort (table not rank-ordered)
  int exp_may_be_big;    // more than SORT_CAP pins may expire
  cudaEvent_t* prof;     // 2*MARS_NUM_KTIMES events, or null
  int* prof_used;        // which pairs were recorded
  const Kv* kv;          // block manager to update with the step's journal, or null
  int phase;             // 0 whole step; sharded: 1 head (before the exchange), 2 tail
  int sharded;
  Xchg x;                // sharded exchange buffers
  Queue gq;              // view of the all-gathered global admission list
};
int mars_enqueue_out_fold(cudaStream_t s, const Work* w, const OutSrc& S, unsigned char* arena,
                          long long cap);

int mars_kernels_init();
int mars_kernels_preload();
// the step head kernel (its graph node takes each step's input as a parameter)
const void* mars_work_init_fn();
#define SCATTER_MAX_COLS 32
struct ScatterCols {  // the columns of one upsert (k_scatter_cols)
  int n;
  void* dst[SCATTER_MAX_COLS];
  long long off[SCATTER_MAX_COLS];
  int esz[SCATTER_MAX_COLS];
};
int mars_enqueue_scatter_cols(cudaStream_t s, const ScatterCols& L, const void* src,
                              const i64* rows, i64 n);
int mars_enqueue_expired_rows(cudaStream_t s, const Tab& t, i64 n_rows, double now, u32* out,
                              i64 cap, int* cnt, int grid);
int mars_enqueue_admit_rows(cudaStream_t s, const Tab& t, const Cfg& c, i64 n, const i64* rows,
                            const i32* r0p, const double* now, int* st);
int mars_enqueue_service_rows(cudaStream_t s, const Tab& t, const Cfg& c, i64 n, const i64* rows,
                              const i64* tokens, const double* now, const i64* pre, int* st);
int mars_enqueue_queue_append(cudaStream_t s, const Queue& Q, const i32* qsel, mars_scalars* sc,
                              i64 n, const u32* rows, const i32* req, const u8* lng);
int mars_enqueue_step(const LaunchArgs* a);
int mars_enqueue_retention(const Cfg& c, cudaStream_t s, i64 n, const i32* ctx, const i32* kv,
                           i64 total, double usage, double ema, double now, u8* pin, double* bb,
                           double* cc, double* dd);
int mars_enqueue_flush(cudaStream_t s, u8* p, i64 n, u32 salt);
int mars_enqueue_resume(const Tab& t, const Cfg& c, mars_scalars* sc, cudaStream_t s, i64 n,
                        const i64* rows, const double* fin, const double* dur, const i32* newp,
                        const i32* dec, double now, int* counts, u8* o_kind, i32* o_blk,
                        i32* o_ctx, i32* o_need, i32* o_proj);
int mars_enqueue_scatter(cudaStream_t s, void* dst, const void* src, const i64* rows, i64 n,
                         int esz);
int mars_enqueue_gather(cudaStream_t s, void* dst, const void* src, const i64* rows, i64 n,
                        int esz);
