// Host-side launch interface between the C ABI (mars_abi.cu) and the kernels.
#pragma once

#include "mars_internal.cuh"
#include "mars_kv.h"

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
// the step's outputs -> the pinned host arena in one launch (the kernel
// stores straight into the mapped host buffer; one descriptor per array)
#define OUT_MAX 48
struct OutDesc {
  const void* src;
  unsigned long long dst_off, bytes;
};
struct OutList {
  OutDesc d[OUT_MAX];
  int n;
};
int mars_enqueue_gather_out(cudaStream_t s, const OutList& L, unsigned char* host_dst);
int mars_enqueue_resume(const Tab& t, const Cfg& c, mars_scalars* sc, cudaStream_t s, i64 n,
                        const i64* rows, const double* fin, const double* dur, const i32* newp,
                        const i32* dec, double now, int* counts, u8* o_kind, i32* o_blk,
                        i32* o_ctx, i32* o_need, i32* o_proj);
int mars_enqueue_scatter(cudaStream_t s, void* dst, const void* src, const i64* rows, i64 n,
                         int esz);
int mars_enqueue_gather(cudaStream_t s, void* dst, const void* src, const i64* rows, i64 n,
                        int esz);
