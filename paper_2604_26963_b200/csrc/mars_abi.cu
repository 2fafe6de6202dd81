// C ABI of the B200 MARS step (include/mars_b200.h): context lifecycle,
// device allocation of the session-state store, uploads/downloads, the step.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <utility>
#include <vector>

#include "mars_internal.cuh"

#define UP_ARENA (8 << 20)  // row batches up to 8 MiB: rows + columns in one pinned copy
#include "mars_launch.h"

namespace {

struct ColSpec {
  size_t host_off;  // offset of the pointer inside mars_cols
  void** dev;       // address of the device pointer inside Tab
  int esz;
  void* ckpt;       // checkpoint copy
  size_t slab_off;  // the column's offset in the table slab (and the input arena)
};

}  // namespace

struct mars_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr, side = nullptr, side2 = nullptr;
  void* d_resume = nullptr;  // mars_resume staging + per-row outcome (lazily allocated)
  i64 last_resume_n = 0;
  bool own_stream = true;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_head = nullptr, ev_pack = nullptr;
  cudaEvent_t ev_kvx = nullptr;
  cudaEvent_t ev_up = nullptr;         // the small-upsert arena's last copy
  cudaEvent_t ev_sc = nullptr;         // the scalars' staging copy's last upload
  unsigned char* h_up = nullptr;       // pinned arena of small upserts (UP_ARENA bytes)
  int pack_ctas = 20;
  mars_config hcfg;
  Cfg cfg;
  i64 max_rows = 0, max_queue = 0, n_rows = 0, alloc_rows = 0;
  int ctl_per_cta = 1024;
  Tab tab;
  Queue queue;
  Lsd qlsd, xlsd;
  Work* work = nullptr;
  Bufs bufs;
  mars_scalars* sc = nullptr;
  i32* qsel = nullptr;
  std::vector<ColSpec> cols;
  // host staging
  mars_step_in* h_in = nullptr;
  Work* h_work = nullptr;
  mars_scalars* h_sc = nullptr;
  unsigned char* h_out = nullptr;  // pinned output arena
  // the session table: every column in ONE device slab, grouped by element
  // size (u8 x5 | f64/i64 x5 | 4-byte x10, each column alloc_rows long), and
  // a pinned host input arena with the same layout (mars_input_arena)
  unsigned char* slab = nullptr;
  size_t slab_bytes = 0;
  unsigned char* h_in_arena = nullptr;
  size_t h_out_bytes = 0;
  // device staging for row scatter/gather
  unsigned char* d_stage = nullptr;
  i64* d_rows = nullptr;
  int* d_hook_st = nullptr;          // contract bits of the drop-in hook kernels
  // checkpoint
  bool have_ckpt = false;
  void* ck_q[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  mars_scalars* ck_sc = nullptr;
  i32* ck_qsel = nullptr;
  i64 ck_q_upper = 0;
  int ck_q_maxreq = 0;
  // host knowledge of the queue (launch-shape decisions only)
  i64 q_upper = 0;
  int q_maxreq = 0;
  i64 pinned_upper = 0;
  int last_launches = 0;
  bool use_graph = false;
  // whole-step CUDA graphs by launch shape: a small cache, so a device-resident
  // run alternating control / non-control ticks replays instead of recapturing
  static constexpr int NGRAPH = 4;
  static constexpr int NKEY = 11;
  cudaGraphExec_t graph_exec[NGRAPH] = {};
  // the captured graph (kept: its k_work_init node takes each step's input
  // as a kernel parameter, cudaGraphExecKernelNodeSetParams before a launch)
  cudaGraph_t graph_g[NGRAPH] = {};
  cudaGraphNode_t init_node[NGRAPH] = {};
  cudaKernelNodeParams init_params[NGRAPH] = {};
  long long graph_key[NGRAPH][NKEY] = {};
  int graph_launches[NGRAPH] = {};
  unsigned long long graph_used[NGRAPH] = {};
  unsigned long long graph_clock = 0;
  bool profiling = false;
  cudaEvent_t prof[2 * MARS_NUM_KTIMES] = {};
  int prof_used[MARS_NUM_KTIMES] = {};
  unsigned flush_salt = 1;
  std::string err;
  // S5 block manager + host tier (mars_kv_init)
  bool kv_on = false;
  void* ck_kv[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  bool have_kv_ckpt = false;
  Kv kv = {};
  void* kv_host = nullptr;          // pinned, mapped
  unsigned char* kv_stage = nullptr; // device staging for op streams / ids
  i64 kv_stage_bytes = 0;
  u8* kv_dstage = nullptr;           // HBM staging for the staged host-tier path
  i64 kv_dstage_blocks = 0;
  i64 kv_ring = 0;                   // next host-tier slot (decision-driven tier, a ring)
  u32* kv_ids = nullptr;             // device ID list of the row offload / restore
  i64 kv_ids_cap = 0;
  // sharded replica (mars_shard_init)
  Xchg x = {};
};

static int fail(mars_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return code;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(ctx, MARS_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                    \
  } while (0)

static Cfg make_cfg(const mars_config& h) {
  Cfg c;
  memset(&c, 0, sizeof c);
  c.bs = h.block_size;
  c.bs_shift = -1;
  for (int k = 0; k < 31; ++k)
    if (h.block_size == (1 << k)) c.bs_shift = k;
  c.budget = h.token_budget;
  c.window = h.window_size;
  c.max_dec = h.max_decode_slots;
  c.num_levels = h.num_levels;
  c.max_promos = h.max_promotions;
  c.hyst = h.hysteresis_window;
  c.w_min = h.w_min;
  c.coord = h.enable_coordinator;
  c.cosched = h.enable_coscheduler;
  for (int i = 0; i < 4; ++i) {
    c.bounds[i] = h.level_bounds[i];
    c.quotas[i] = h.level_quotas[i];
  }
  c.tick_s = h.tick_duration_s;
  c.prefill_rate = (double)h.token_budget / h.tick_duration_s;  // engine.py:240-242
  c.promo_wait = h.promotion_wait_s;
  c.slack = h.deadline_slack;
  c.horizon = h.max_pin_horizon_s;
  c.pw_clip = h.pressure_weight_clip;
  c.cpu_hi = h.cpu_high_fraction;
  c.cpu_lo = h.cpu_low_fraction;
  c.kv_hi = h.kv_high_watermark;
  c.kv_lo = h.kv_low_watermark;
  c.ema_alpha = h.ema_smoothing;
  c.tool_prior = h.initial_tool_estimate_s;
  c.ai = h.aimd_increase;
  c.md = h.aimd_decrease;
  c.ctl_interval = h.control_interval_s;
  c.init_window = h.initial_window;
  c.oversub = h.cpu_oversubscription;
  c.reserve = h.reserve_fraction;
  c.long_frac = h.long_session_fraction;
  c.policy = h.policy;
  c.ttl_s = h.ttl_seconds;
  c.ttl_mult = h.ttl_multiplier;
  if (c.policy != POL_MARS) {
    // comparison policies: arrival (or served, arrival) order with no aging
    // and the coordinator-off victim eligibility; whole-chunk fitting
    // (shrink_chunks=False, baselines.py:149/201/309)
    c.coord = 0;
    c.cosched = 0;
  }
  c.strict = (c.policy == POL_FCFS || c.policy == POL_STATIC_TTL || c.policy == POL_DYNAMIC_TTL);
  // candidate-list refinement triggers and the victim stream length; tests
  // shrink them (MARS_REF_TRIG_W / _V, MARS_VSTREAM) to drive the refinement
  // and the exact full-table fallback on small tables
  auto env_int = [](const char* k, int dflt) {
    const char* v = getenv(k);
    return (v && v[0]) ? atoi(v) : dflt;
  };
  c.ref_trig_w = env_int("MARS_REF_TRIG_W", REF_TRIG_W);
  c.ref_trig_v = env_int("MARS_REF_TRIG_V", REF_TRIG_V);
  c.stream_cap = env_int("MARS_VSTREAM", VSTREAM_CAP);
  if (c.stream_cap < 1 || c.stream_cap > VSTREAM_CAP) c.stream_cap = VSTREAM_CAP;
  return c;
}

extern "C" {

int mars_abi_version(void) { return MARS_ABI_VERSION; }

void mars_config_default(mars_config* h) {
  memset(h, 0, sizeof *h);
  h->block_size = 16;
  h->token_budget = 512;
  h->tick_duration_s = 0.064;
  h->num_levels = 4;
  h->max_promotions = 3;
  h->max_decode_slots = 64;
  h->window_size = 128;
  const int64_t inf = INT64_MAX;
  int64_t b[4] = {4000, 32000, 128000, inf}, q[4] = {2000, 8000, 32000, inf};
  for (int i = 0; i < 4; ++i) {
    h->level_bounds[i] = b[i];
    h->level_quotas[i] = q[i];
  }
  h->promotion_wait_s = 10.0;
  h->deadline_slack = 2.0;
  h->max_pin_horizon_s = 60.0;
  h->pressure_weight_clip = 100.0;
  h->cpu_high_fraction = 0.90;
  h->cpu_low_fraction = 0.70;
  h->kv_high_watermark = 0.90;
  h->kv_low_watermark = 0.70;
  h->hysteresis_window = 3;
  h->ema_smoothing = 0.3;
  h->initial_tool_estimate_s = 5.0;
  h->w_min = 2;
  h->aimd_increase = 1.0;
  h->aimd_decrease = 0.5;
  h->control_interval_s = 2.0;
  h->initial_window = 8.0;
  h->cpu_oversubscription = 1.5;
  h->reserve_fraction = 0.10;
  h->long_session_fraction = 0.25;
  h->enable_coordinator = 1;
  h->enable_coscheduler = 1;
  h->policy = MARS_POLICY_MARS;
  h->ttl_seconds = 30.0;     // K_STATIC_TTL_S (baselines.py:50)
  h->ttl_multiplier = 1.5;   // K_DYNAMIC_TTL_MULTIPLIER (baselines.py:51)
}

const char* mars_last_error(mars_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int mars_last_launch_count(mars_ctx* ctx) { return ctx ? ctx->last_launches : -1; }

static int alloc(mars_ctx* ctx, void** p, size_t bytes) {
  CK(cudaMalloc(p, bytes ? bytes : 16));
  return MARS_OK;
}

#define ALLOC(ptr, bytes)                                      \
  do {                                                         \
    int rc_ = alloc(ctx, (void**)&(ptr), (size_t)(bytes));     \
    if (rc_) {                                                 \
      mars_destroy(ctx);                                       \
      return rc_;                                              \
    }                                                          \
  } while (0)

int mars_create(const mars_config* hcfg, int device, int64_t max_rows, int64_t max_queue,
                mars_ctx** out) {
  if (!hcfg || !out || max_rows < 1 || max_queue < 0) return MARS_ERR_ARG;
  if (hcfg->policy < MARS_POLICY_MARS || hcfg->policy > MARS_POLICY_DYNAMIC_TTL)
    return MARS_ERR_ARG;
  if (hcfg->window_size < 1 || hcfg->window_size > WIN_MAX || hcfg->num_levels < 1 ||
      hcfg->num_levels > 4 || hcfg->block_size < 1 || hcfg->token_budget < 1 ||
      hcfg->max_decode_slots < 0)
    return MARS_ERR_ARG;
  if (max_rows >= (1ll << 31)) return MARS_ERR_ARG;
  mars_ctx* ctx = new mars_ctx();
  ctx->device = device;
  ctx->hcfg = *hcfg;
  ctx->cfg = make_cfg(*hcfg);
  ctx->max_rows = max_rows;
  ctx->alloc_rows = (max_rows + ROW_PAD - 1) / ROW_PAD * ROW_PAD;
  ctx->max_queue = max_queue < 1 ? 1 : max_queue;
  {
    const char* e = getenv("MARS_CTL_PER_CTA");  // tuning knob (graph key follows it)
    ctx->ctl_per_cta = (e && atoi(e) > 0) ? atoi(e) : 1024;
  }
  CK(cudaSetDevice(device));
  CK(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
  CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
  CK(cudaStreamCreateWithFlags(&ctx->side2, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&ctx->ev_head, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_pack, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_kvx, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_up, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_sc, cudaEventDisableTiming));
  CK(cudaMallocHost((void**)&ctx->h_up, UP_ARENA));
  {
    const char* e = getenv("MARS_PACK_CTAS");  // tuning knob: 0 disables the early pack
    if (e) ctx->pack_ctas = atoi(e);
  }
  {
    int rc = mars_kernels_init();
    if (!rc) rc = mars_kernels_preload();
    if (!rc) rc = mars_kv_preload();
    if (rc) return fail(ctx, MARS_ERR_CUDA, "kernel init: %s", cudaGetErrorString((cudaError_t)rc));
  }
  const i64 R = ctx->alloc_rows, Qc = ctx->max_queue;
  Tab& t = ctx->tab;
  memset(&t, 0, sizeof t);
  t.cap = R;
  {
    // slab order: a default step's 17 columns first (u8 x5, f64 x3, 4-byte
    // x9: one contiguous range, one linear copy of the whole table in
    // mars_upsert_arena), then rounds_left, arrival, served; adjacent columns
    // of one element size form one pitched copy otherwise
    struct {
      void** p;
      int esz;
    } lay[] = {{(void**)&t.phase, 1}, {(void**)&t.flags, 1}, {(void**)&t.level, 1},
               {(void**)&t.promos, 1}, {(void**)&t.plevel, 1}, {(void**)&t.rs, 8},
               {(void**)&t.ws, 8},     {(void**)&t.dl, 8},     {(void**)&t.ctx, 4},
               {(void**)&t.kv, 4},     {(void**)&t.rem, 4},    {(void**)&t.pb, 4},
               {(void**)&t.req, 4},    {(void**)&t.r0p, 4},    {(void**)&t.r0d, 4},
               {(void**)&t.pre, 4},    {(void**)&t.rank, 4},   {(void**)&t.rleft, 4},
               {(void**)&t.arr, 8},    {(void**)&t.served, 8}};
    size_t tot = 0;
    for (auto& l : lay) tot += (size_t)R * l.esz;
    ALLOC(ctx->slab, tot);
    ctx->slab_bytes = tot;
    size_t off = 0;
    for (auto& l : lay) {
      *l.p = ctx->slab + off;
      off += (size_t)R * l.esz;
    }
  }
  CK(cudaMemset(t.rleft, 0, R * 4));
  ALLOC(t.winpos, R * 2);
  CK(cudaMemset(t.winpos, 0xff, R * 2));
  CK(cudaMemset(t.phase, MARS_EMPTY, R));
  CK(cudaMemset(t.flags, 0, R));
  Queue& q = ctx->queue;
  q.cap = Qc;
  for (int i = 0; i < 2; ++i) {
    ALLOC(q.row[i], Qc * 4);
    ALLOC(q.req[i], Qc * 4);
    ALLOC(q.lng[i], Qc);
    ALLOC(q.gpos[i], Qc * 4);
  }
  i64 Lc = Qc > R ? Qc : R;
  Lsd* ls[2] = {&ctx->qlsd, &ctx->xlsd};
  for (int j = 0; j < 2; ++j) {
    ls[j]->cap = Lc;
    for (int i = 0; i < 2; ++i) {
      ALLOC(ls[j]->k[i], Lc * 8);
      ALLOC(ls[j]->v[i], Lc * 4);
    }
    ALLOC(ls[j]->cnt, (size_t)LSD_G * 256 * 4);
  }
  ALLOC(ctx->work, sizeof(Work));
  ALLOC(ctx->sc, sizeof(mars_scalars));
  ALLOC(ctx->qsel, sizeof(i32));
  CK(cudaMemset(ctx->qsel, 0, sizeof(i32)));
  Bufs& b = ctx->bufs;
  memset(&b, 0, sizeof b);
  // one entry per k_scan CTA (<= the scan's block size, mars_kernels.cu)
  ALLOC(b.tile_cnt, 1024 * 4);
  ALLOC(b.tile_kv, 1024 * 3 * 8);
  ALLOC(b.row_dig, R * 4);
  ALLOC(b.cand_row, R * 4);
  ALLOC(b.exp_row, R * 4);
  ALLOC(b.exp_blk, R * 4);
  ALLOC(b.exp_rank, R * 4);
  ALLOC(b.exp_row_sorted, R * 4);
  ALLOC(b.exp_blk_sorted, R * 4);
  ALLOC(b.wc_hi, R * 8);
  ALLOC(b.wc_lo, R * 8);
  ALLOC(b.wc_row, R * 4);
  ALLOC(b.vc_key, R * 8);
  ALLOC(b.vc_kl, R * 8);
  ALLOC(b.vc_whi, R * 8);
  ALLOC(b.vc_wlo, R * 8);
  ALLOC(b.vc_row, R * 4);
  ALLOC(b.vc_blk, R * 4);
  // refined lists (k_scan phase 3): the window list can grow by admitted rows
  ALLOC(b.wr_hi, R * 8);
  ALLOC(b.wr_lo, R * 8);
  ALLOC(b.wr_row, R * 4);
  ALLOC(b.vr_key, (size_t)VR_CAP * 8);
  ALLOC(b.vr_kl, (size_t)VR_CAP * 8);
  ALLOC(b.vr_whi, (size_t)VR_CAP * 8);
  ALLOC(b.vr_wlo, (size_t)VR_CAP * 8);
  ALLOC(b.vr_row, (size_t)VR_CAP * 4);
  ALLOC(b.vr_blk, (size_t)VR_CAP * 4);
  ALLOC(b.vs_key, (size_t)VSTREAM_CAP * 8);
  ALLOC(b.vs_kl, (size_t)VSTREAM_CAP * 8);
  ALLOC(b.vs_whi, (size_t)VSTREAM_CAP * 8);
  ALLOC(b.vs_wlo, (size_t)VSTREAM_CAP * 8);
  ALLOC(b.vs_row, (size_t)VSTREAM_CAP * 4);
  ALLOC(b.vs_blk, (size_t)VSTREAM_CAP * 4);
  ALLOC(b.ret_row, R * 4);
  ALLOC(b.ret_pin, R);
  ALLOC(b.ret_b, R * 8);
  ALLOC(b.ret_c, R * 8);
  ALLOC(b.ret_d, R * 8);
  ALLOC(b.admitted, Qc * 4);
  ALLOC(b.win_rows, WIN_MAX * 4);
  ALLOC(b.dec_rows, WIN_MAX * 4);
  ALLOC(b.pre_rows, WIN_MAX * 4);
  ALLOC(b.pre_grant, WIN_MAX * 4);
  ALLOC(b.dec_level, WIN_MAX);
  ALLOC(b.pre_level, WIN_MAX);
  ALLOC(b.svc_pre, WIN_MAX * 8);
  ALLOC(b.fin_row, WIN_MAX * 4);
  ALLOC(b.fin_pin, WIN_MAX);
  ALLOC(b.fin_b, WIN_MAX * 8);
  ALLOC(b.fin_c, WIN_MAX * 8);
  ALLOC(b.fin_d, WIN_MAX * 8);
  ALLOC(b.end_row, WIN_MAX * 4);
  ALLOC(b.end_kind, WIN_MAX);
  ALLOC(b.end_blk, WIN_MAX * 4);
  ALLOC(b.end_pin, WIN_MAX);
  ALLOC(b.end_b, WIN_MAX * 8);
  ALLOC(b.end_c, WIN_MAX * 8);
  ALLOC(b.end_d, WIN_MAX * 8);
  ALLOC(b.pre_done, WIN_MAX);
  b.ev_cap = R;
  ALLOC(b.ev_row, R * 4);
  ALLOC(b.ev_kind, R);
  ALLOC(b.ev_blk, R * 4);
  b.j_cap = R + 2 * WIN_MAX;
  ALLOC(b.j_op, b.j_cap);
  ALLOC(b.j_row, b.j_cap * 4);
  ALLOC(b.j_n, b.j_cap * 4);
  ALLOC(ctx->d_stage, R * 8);
  ALLOC(ctx->d_rows, R * 8);
  ALLOC(ctx->d_hook_st, 16);
  CK(cudaMemset(ctx->d_hook_st, 0, 16));
  // host pinned
  CK(cudaMallocHost((void**)&ctx->h_in, sizeof(mars_step_in)));
  CK(cudaMallocHost((void**)&ctx->h_work, sizeof(Work)));
  CK(cudaMallocHost((void**)&ctx->h_sc, sizeof(mars_scalars)));
  ctx->h_out_bytes = (size_t)OUT_HDR + (size_t)R * 48 + (size_t)Qc * 4 + (size_t)b.j_cap * 9 +
                     4 * WIN_MAX * 4 + WIN_MAX * 80 + 8192;
  CK(cudaMallocHost((void**)&ctx->h_out, ctx->h_out_bytes));
  memset(ctx->h_in, 0, sizeof(mars_step_in));
  // scalars: empty pool of one block until mars_set_scalars
  mars_scalars s0;
  memset(&s0, 0, sizeof s0);
  s0.total_blocks = 1;
  s0.free_blocks = 1;
  s0.available_kv = 1;
  s0.w_adm = hcfg->initial_window;
  CK(cudaMemcpy(ctx->sc, &s0, sizeof s0, cudaMemcpyHostToDevice));
  // column table
  auto add = [&](size_t off, void** dev, int esz) {
    ctx->cols.push_back({off, dev, esz, nullptr, (size_t)((unsigned char*)*dev - ctx->slab)});
  };
  add(offsetof(mars_cols, phase), (void**)&t.phase, 1);
  add(offsetof(mars_cols, flags), (void**)&t.flags, 1);
  add(offsetof(mars_cols, level), (void**)&t.level, 1);
  add(offsetof(mars_cols, promos), (void**)&t.promos, 1);
  add(offsetof(mars_cols, plevel), (void**)&t.plevel, 1);
  add(offsetof(mars_cols, ready_since), (void**)&t.rs, 8);
  add(offsetof(mars_cols, wait_since), (void**)&t.ws, 8);
  add(offsetof(mars_cols, deadline), (void**)&t.dl, 8);
  add(offsetof(mars_cols, arrival), (void**)&t.arr, 8);
  add(offsetof(mars_cols, context), (void**)&t.ctx, 4);
  add(offsetof(mars_cols, kv), (void**)&t.kv, 4);
  add(offsetof(mars_cols, rem_decode), (void**)&t.rem, 4);
  add(offsetof(mars_cols, pinned_blocks), (void**)&t.pb, 4);
  add(offsetof(mars_cols, req_blocks), (void**)&t.req, 4);
  add(offsetof(mars_cols, r0_prefill), (void**)&t.r0p, 4);
  add(offsetof(mars_cols, r0_decode), (void**)&t.r0d, 4);
  add(offsetof(mars_cols, preempt), (void**)&t.pre, 4);
  add(offsetof(mars_cols, served), (void**)&t.served, 8);
  add(offsetof(mars_cols, rank), (void**)&t.rank, 4);
  add(offsetof(mars_cols, rounds_left), (void**)&t.rleft, 4);
  CK(cudaDeviceSynchronize());
  *out = ctx;
  return MARS_OK;
}

int mars_destroy(mars_ctx* ctx) {
  if (!ctx) return MARS_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  Tab& t = ctx->tab;
  cudaFree(ctx->slab);  // every table column
  cudaFree(t.winpos);
  if (ctx->h_in_arena) cudaFreeHost(ctx->h_in_arena);
  for (int i = 0; i < 2; ++i) {
    cudaFree(ctx->queue.row[i]);
    cudaFree(ctx->queue.req[i]);
    cudaFree(ctx->queue.lng[i]);
    cudaFree(ctx->queue.gpos[i]);
    cudaFree(ctx->qlsd.k[i]);
    cudaFree(ctx->qlsd.v[i]);
    cudaFree(ctx->xlsd.k[i]);
    cudaFree(ctx->xlsd.v[i]);
  }
  cudaFree(ctx->qlsd.cnt);
  cudaFree(ctx->xlsd.cnt);
  cudaFree(ctx->work);
  cudaFree(ctx->sc);
  cudaFree(ctx->qsel);
  Bufs& b = ctx->bufs;
  void* bs[] = {b.tile_cnt, b.tile_kv, b.row_dig, b.cand_row, b.exp_row, b.exp_blk, b.exp_rank, b.exp_row_sorted, b.exp_blk_sorted, b.wc_hi,
                b.wc_lo, b.wc_row, b.vc_key, b.vc_whi, b.vc_wlo, b.vc_row, b.vc_blk, b.ret_row,
                b.ret_pin, b.ret_b, b.ret_c, b.ret_d, b.admitted, b.win_rows, b.dec_rows,
                b.pre_rows, b.pre_grant, b.ev_row, b.ev_kind, b.ev_blk, b.j_op, b.j_row, b.j_n,
                b.dec_level, b.pre_level, b.svc_pre, b.fin_row, b.fin_pin, b.fin_b, b.fin_c, b.fin_d,
                b.flush, b.end_row, b.end_kind, b.end_blk, b.end_pin, b.end_b, b.end_c,
                b.end_d, b.pre_done, b.vc_kl, b.wr_hi, b.wr_lo, b.wr_row, b.vr_key, b.vr_kl,
                b.vr_whi, b.vr_wlo, b.vr_row, b.vr_blk, b.vs_key, b.vs_kl, b.vs_whi,
                b.vs_wlo, b.vs_row, b.vs_blk};
  for (void* p : bs) cudaFree(p);
  cudaFree(ctx->d_stage);
  cudaFree(ctx->d_resume);
  cudaFree(ctx->d_rows);
  cudaFree(ctx->d_hook_st);
  for (auto& cs : ctx->cols) cudaFree(cs.ckpt);
  for (void* p : ctx->ck_q) cudaFree(p);
  cudaFree(ctx->ck_sc);
  for (void* p : ctx->ck_kv) cudaFree(p);
  cudaFree(ctx->ck_qsel);
  cudaFreeHost(ctx->h_in);
  cudaFreeHost(ctx->h_work);
  cudaFreeHost(ctx->h_sc);
  cudaFreeHost(ctx->h_out);
  {
    Kv& k = ctx->kv;
    void* kp[] = {k.seg, k.chunks, k.cfs, k.dir, k.len, k.s, k.data, ctx->kv_stage,
                  ctx->kv_dstage, k.xoff, k.xlen, k.xbase, k.arena, k.xaoff, k.xroff, k.cap,
                  ctx->kv_ids};
    for (void* p : kp) cudaFree(p);
    if (ctx->kv_host) cudaFreeHost(ctx->kv_host);
  }
  {
    Xchg& x = ctx->x;
    void* xp[] = {x.xc, x.xsend, x.xrecv, x.gq_row, x.gq_req, x.gq_lng, x.adm_idx};
    for (void* p : xp) cudaFree(p);
  }
  for (auto& e : ctx->prof)
    if (e) cudaEventDestroy(e);
  for (auto& g : ctx->graph_exec)
    if (g) cudaGraphExecDestroy(g);
  for (auto& g : ctx->graph_g)
    if (g) cudaGraphDestroy(g);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->ev_head) cudaEventDestroy(ctx->ev_head);
  if (ctx->ev_pack) cudaEventDestroy(ctx->ev_pack);
  if (ctx->ev_kvx) cudaEventDestroy(ctx->ev_kvx);
  if (ctx->ev_up) cudaEventDestroy(ctx->ev_up);
  if (ctx->ev_sc) cudaEventDestroy(ctx->ev_sc);
  if (ctx->h_up) cudaFreeHost(ctx->h_up);
  if (ctx->side2) cudaStreamDestroy(ctx->side2);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  delete ctx;
  return MARS_OK;
}

int mars_set_stream(mars_ctx* ctx, void* stream) {
  if (!ctx) return MARS_ERR_ARG;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  ctx->stream = (cudaStream_t)stream;
  ctx->own_stream = false;
  return MARS_OK;
}

int mars_set_rows(mars_ctx* ctx, int64_t n) {
  if (!ctx || n < 0 || n > ctx->max_rows) return fail(ctx, MARS_ERR_CAPACITY, "rows %lld", (long long)n);
  ctx->n_rows = n;
  return MARS_OK;
}

int mars_upsert_rows(mars_ctx* ctx, int64_t n, const int64_t* rows, const mars_cols* cols) {
  if (!ctx || !cols || n < 0) return MARS_ERR_ARG;
  if (n == 0) return MARS_OK;
  CK(cudaSetDevice(ctx->device));
  if (!rows) {
    if (n > ctx->max_rows) return fail(ctx, MARS_ERR_CAPACITY, "upsert %lld rows", (long long)n);
    for (auto& cs : ctx->cols) {
      const void* hp = *(void* const*)((const char*)cols + cs.host_off);
      if (!hp) continue;
      CK(cudaMemcpyAsync(*cs.dev, hp, (size_t)n * cs.esz, cudaMemcpyHostToDevice, ctx->stream));
    }
    if (n > ctx->n_rows) ctx->n_rows = n;
  } else {
    for (int64_t i = 0; i < n; ++i)
      if (rows[i] < 0 || rows[i] >= ctx->max_rows)
        return fail(ctx, MARS_ERR_CAPACITY, "row %lld out of range", (long long)rows[i]);
    if (n > ctx->max_rows) return MARS_ERR_CAPACITY;
    // every given column staged side by side, then ONE scatter launch; a
    // batch larger than the staging buffer goes column by column
    ScatterCols L;
    L.n = 0;
    size_t off = 0;
    bool fits = true;
    for (auto& cs : ctx->cols) {
      const void* hp = *(void* const*)((const char*)cols + cs.host_off);
      if (!hp) continue;
      off = (off + 15) & ~(size_t)15;
      if (off + (size_t)n * cs.esz > (size_t)ctx->alloc_rows * 8 || L.n == SCATTER_MAX_COLS) {
        fits = false;
        break;
      }
      L.dst[L.n] = *cs.dev;
      L.off[L.n] = (long long)off;
      L.esz[L.n] = cs.esz;
      ++L.n;
      off += (size_t)n * cs.esz;
    }
    const size_t rows_off = (off + 15) & ~(size_t)15;
    const size_t small = rows_off + (size_t)n * 8;
    if (fits && small <= UP_ARENA && small <= (size_t)ctx->alloc_rows * 8) {
      // a small batch (the drop-in's per-tick writes): rows and columns
      // packed into a pinned host arena, ONE copy, ONE scatter, no wait --
      // the caller's arrays are copied before the return, the arena is
      // reused only once its previous copy completed (ev_up)
      CK(cudaEventSynchronize(ctx->ev_up));
      int k = 0;
      for (auto& cs : ctx->cols) {
        const void* hp = *(void* const*)((const char*)cols + cs.host_off);
        if (!hp) continue;
        memcpy(ctx->h_up + L.off[k], hp, (size_t)n * cs.esz);
        ++k;
      }
      memcpy(ctx->h_up + rows_off, rows, (size_t)n * 8);
      CK(cudaMemcpyAsync(ctx->d_stage, ctx->h_up, small, cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaEventRecord(ctx->ev_up, ctx->stream));
      int rc = mars_enqueue_scatter_cols(ctx->stream, L, ctx->d_stage,
                                         (const i64*)(ctx->d_stage + rows_off), n);
      if (rc) return fail(ctx, MARS_ERR_CUDA, "scatter: %s", cudaGetErrorString((cudaError_t)rc));
      for (int64_t i = 0; i < n; ++i)
        if (rows[i] + 1 > ctx->n_rows) ctx->n_rows = rows[i] + 1;
      return MARS_OK;
    }
    CK(cudaMemcpyAsync(ctx->d_rows, rows, (size_t)n * 8, cudaMemcpyHostToDevice, ctx->stream));
    if (fits) {
      int k = 0;
      for (auto& cs : ctx->cols) {
        const void* hp = *(void* const*)((const char*)cols + cs.host_off);
        if (!hp) continue;
        CK(cudaMemcpyAsync(ctx->d_stage + L.off[k], hp, (size_t)n * cs.esz, cudaMemcpyHostToDevice,
                           ctx->stream));
        ++k;
      }
      int rc = mars_enqueue_scatter_cols(ctx->stream, L, ctx->d_stage, ctx->d_rows, n);
      if (rc) return fail(ctx, MARS_ERR_CUDA, "scatter: %s", cudaGetErrorString((cudaError_t)rc));
    } else {
      for (auto& cs : ctx->cols) {
        const void* hp = *(void* const*)((const char*)cols + cs.host_off);
        if (!hp) continue;
        CK(cudaMemcpyAsync(ctx->d_stage, hp, (size_t)n * cs.esz, cudaMemcpyHostToDevice, ctx->stream));
        int rc = mars_enqueue_scatter(ctx->stream, *cs.dev, ctx->d_stage, ctx->d_rows, n, cs.esz);
        if (rc) return fail(ctx, MARS_ERR_CUDA, "scatter: %s", cudaGetErrorString((cudaError_t)rc));
      }
    }
    for (int64_t i = 0; i < n; ++i)
      if (rows[i] + 1 > ctx->n_rows) ctx->n_rows = rows[i] + 1;
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return MARS_OK;
}

int mars_input_arena(mars_ctx* ctx, void** base, int64_t* bytes, mars_cols* cols) {
  if (!ctx || !base || !bytes) return MARS_ERR_ARG;
  CK(cudaSetDevice(ctx->device));
  if (!ctx->h_in_arena) {
    CK(cudaMallocHost((void**)&ctx->h_in_arena, ctx->slab_bytes));
    memset(ctx->h_in_arena, 0, ctx->slab_bytes);
    // the capacity padding rows [max_rows, alloc_rows) hold the device's
    // initial values (a whole-table upload copies them along)
    const i64 R = ctx->alloc_rows, M = ctx->max_rows;
    memset(ctx->h_in_arena + (size_t)((unsigned char*)ctx->tab.phase - ctx->slab) + M, MARS_EMPTY,
           (size_t)(R - M));
  }
  *base = ctx->h_in_arena;
  *bytes = (int64_t)ctx->slab_bytes;
  if (cols)
    for (auto& cs : ctx->cols)
      *(void**)((char*)cols + cs.host_off) = ctx->h_in_arena + cs.slab_off;
  return MARS_OK;
}

int mars_upsert_arena(mars_ctx* ctx, int64_t n, uint64_t mask) {
  if (!ctx || n < 0) return MARS_ERR_ARG;
  if (!ctx->h_in_arena) return fail(ctx, MARS_ERR_ARG, "mars_upsert_arena before mars_input_arena");
  if (n > ctx->max_rows) return fail(ctx, MARS_ERR_CAPACITY, "upsert %lld rows", (long long)n);
  if (n == 0 || mask == 0) return MARS_OK;
  CK(cudaSetDevice(ctx->device));
  // the masked columns in slab order; a run of slab-adjacent columns of one
  // element size is one pitched copy (rows [0, n) of each)
  std::vector<std::pair<size_t, int>> sel;  // (slab offset, esz)
  for (size_t i = 0; i < ctx->cols.size(); ++i)
    if (mask >> i & 1) sel.push_back({ctx->cols[i].slab_off, ctx->cols[i].esz});
  std::sort(sel.begin(), sel.end());
  const size_t R = (size_t)ctx->alloc_rows;
  if (n == ctx->max_rows) {
    // the whole table of slab-contiguous columns: ONE linear copy (the padding
    // rows past max_rows carry the device's initial values, set above)
    bool contiguous = true;
    for (size_t i = 1; i < sel.size(); ++i)
      contiguous &= sel[i].first == sel[i - 1].first + R * (size_t)sel[i - 1].second;
    if (contiguous) {
      const size_t a = sel.front().first, b = sel.back().first + R * (size_t)sel.back().second;
      CK(cudaMemcpyAsync(ctx->slab + a, ctx->h_in_arena + a, b - a, cudaMemcpyHostToDevice,
                         ctx->stream));
      if (n > ctx->n_rows) ctx->n_rows = n;
      CK(cudaStreamSynchronize(ctx->stream));
      return MARS_OK;
    }
  }
  for (size_t i = 0; i < sel.size();) {
    size_t j = i + 1;
    while (j < sel.size() && sel[j].second == sel[i].second &&
           sel[j].first == sel[j - 1].first + R * (size_t)sel[i].second)
      ++j;
    const size_t pitch = R * (size_t)sel[i].second;
    CK(cudaMemcpy2DAsync(ctx->slab + sel[i].first, pitch, ctx->h_in_arena + sel[i].first, pitch,
                         (size_t)n * sel[i].second, j - i, cudaMemcpyHostToDevice, ctx->stream));
    i = j;
  }
  if (n > ctx->n_rows) ctx->n_rows = n;
  CK(cudaStreamSynchronize(ctx->stream));
  return MARS_OK;
}

int mars_read_rows(mars_ctx* ctx, int64_t n, const int64_t* rows, mars_cols* out) {
  if (!ctx || !out || n < 0) return MARS_ERR_ARG;
  if (n == 0) return MARS_OK;
  CK(cudaSetDevice(ctx->device));
  if (!rows) {
    if (n > ctx->max_rows) return MARS_ERR_CAPACITY;
    for (auto& cs : ctx->cols) {
      void* hp = *(void**)((char*)out + cs.host_off);
      if (!hp) continue;
      CK(cudaMemcpyAsync(hp, *cs.dev, (size_t)n * cs.esz, cudaMemcpyDeviceToHost, ctx->stream));
    }
  } else {
    if (n > ctx->max_rows) return MARS_ERR_CAPACITY;
    CK(cudaMemcpyAsync(ctx->d_rows, rows, (size_t)n * 8, cudaMemcpyHostToDevice, ctx->stream));
    for (auto& cs : ctx->cols) {
      void* hp = *(void**)((char*)out + cs.host_off);
      if (!hp) continue;
      int rc = mars_enqueue_gather(ctx->stream, ctx->d_stage, *cs.dev, ctx->d_rows, n, cs.esz);
      if (rc) return fail(ctx, MARS_ERR_CUDA, "gather: %s", cudaGetErrorString((cudaError_t)rc));
      CK(cudaMemcpyAsync(hp, ctx->d_stage, (size_t)n * cs.esz, cudaMemcpyDeviceToHost, ctx->stream));
    }
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return MARS_OK;
}

int mars_set_queue(mars_ctx* ctx, int64_t n, const uint32_t* rows, const int32_t* req,
                   const uint8_t* lng) {
  if (!ctx || n < 0) return MARS_ERR_ARG;
  if (n > ctx->max_queue) return fail(ctx, MARS_ERR_CAPACITY, "queue %lld > %lld", (long long)n,
                                      (long long)ctx->max_queue);
  CK(cudaSetDevice(ctx->device));
  int mx = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (req[i] < 1) return fail(ctx, MARS_ERR_CONTRACT, "queue entry needs req_blocks >= 1");
    if (req[i] > mx) mx = req[i];
  }
  CK(cudaMemsetAsync(ctx->qsel, 0, sizeof(i32), ctx->stream));
  if (n) {
    CK(cudaMemcpyAsync(ctx->queue.row[0], rows, n * 4, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->queue.req[0], req, n * 4, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->queue.lng[0], lng, n, cudaMemcpyHostToDevice, ctx->stream));
  }
  // queue_len lives in the device scalars
  CK(cudaMemcpyAsync(&ctx->sc->queue_len, &n, sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->q_upper = n;
  ctx->q_maxreq = mx;
  return MARS_OK;
}

int mars_queue_append(mars_ctx* ctx, int64_t n, const uint32_t* rows, const int32_t* req,
                      const uint8_t* lng) {
  if (!ctx || n < 0 || (n > 0 && (!rows || !req || !lng))) return MARS_ERR_ARG;
  if (n == 0) return MARS_OK;
  if (ctx->q_upper + n > ctx->max_queue)
    return fail(ctx, MARS_ERR_CAPACITY, "queue %lld + %lld > %lld", (long long)ctx->q_upper,
                (long long)n, (long long)ctx->max_queue);
  if (n * 9 > ctx->alloc_rows * 8) {  // through the staging buffer in chunks, in order
    const int64_t m = ctx->alloc_rows * 8 / 9;
    for (int64_t o = 0; o < n; o += m) {
      int rc = mars_queue_append(ctx, std::min(m, n - o), rows + o, req + o, lng + o);
      if (rc) return rc;
    }
    return MARS_OK;
  }
  int mx = ctx->q_maxreq;
  for (int64_t i = 0; i < n; ++i) {
    if (req[i] < 1) return fail(ctx, MARS_ERR_CONTRACT, "queue entry needs req_blocks >= 1");
    if (req[i] > mx) mx = req[i];
    if ((i64)rows[i] >= ctx->max_rows) return fail(ctx, MARS_ERR_CAPACITY, "row out of range");
  }
  CK(cudaSetDevice(ctx->device));
  u8* st = ctx->d_stage;
  CK(cudaMemcpyAsync(st, rows, n * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(st + n * 4, req, n * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(st + n * 8, lng, n, cudaMemcpyHostToDevice, ctx->stream));
  int rc = mars_enqueue_queue_append(ctx->stream, ctx->queue, ctx->qsel, ctx->sc, n, (const u32*)st,
                                     (const i32*)(st + n * 4), st + n * 8);
  if (rc) return fail(ctx, MARS_ERR_CUDA, "queue append: %s", cudaGetErrorString((cudaError_t)rc));
  CK(cudaStreamSynchronize(ctx->stream));  // (the staging buffer is reused next)
  ctx->q_upper += n;
  ctx->q_maxreq = mx;
  return MARS_OK;
}

// the drop-in's batched MLFQ hooks (k_admit_rows / k_service_rows); the
// work area's status carries a contract break back
static int hook_rows_check(mars_ctx* ctx, int64_t n, const int64_t* rows) {
  if (!ctx || n < 0 || (n > 0 && !rows)) return MARS_ERR_ARG;
  for (int64_t i = 0; i < n; ++i)
    if (rows[i] < 0 || rows[i] >= ctx->max_rows) return fail(ctx, MARS_ERR_CAPACITY, "row out of range");
  return MARS_OK;
}

// entries per pass through the row staging buffer (24 bytes each at most)
static int64_t hook_chunk(const mars_ctx* ctx) { return ctx->alloc_rows * 8 / 24; }

static int hook_status(mars_ctx* ctx) {
  int32_t st = 0;
  CK(cudaMemcpyAsync(&st, ctx->d_hook_st, sizeof st, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemsetAsync(ctx->d_hook_st, 0, sizeof(int32_t), ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (st & ST_BAD_INPUT) return fail(ctx, MARS_ERR_CONTRACT, "hook input violates the contract");
  return MARS_OK;
}

int mars_on_admit(mars_ctx* ctx, int64_t n, const int64_t* rows, const int32_t* r0_prefill,
                  const double* now) {
  int rc = hook_rows_check(ctx, n, rows);
  if (rc || n == 0) return rc;
  const int64_t m = hook_chunk(ctx);
  if (n > m) {  // (rows are distinct: the chunks are independent)
    for (int64_t o = 0; o < n; o += m) {
      rc = mars_on_admit(ctx, std::min(m, n - o), rows + o, r0_prefill + o, now + o);
      if (rc) return rc;
    }
    return MARS_OK;
  }
  CK(cudaSetDevice(ctx->device));
  u8* st = ctx->d_stage;
  CK(cudaMemcpyAsync(st, rows, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(st + n * 8, now, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(st + n * 16, r0_prefill, n * 4, cudaMemcpyHostToDevice, ctx->stream));
  rc = mars_enqueue_admit_rows(ctx->stream, ctx->tab, ctx->cfg, n, (const i64*)st,
                               (const i32*)(st + n * 16), (const double*)(st + n * 8),
                               ctx->d_hook_st);
  if (rc) return fail(ctx, MARS_ERR_CUDA, "admit rows: %s", cudaGetErrorString((cudaError_t)rc));
  return hook_status(ctx);
}

int mars_on_service(mars_ctx* ctx, int64_t n, const int64_t* rows, const int64_t* tokens,
                    const double* now, const int64_t* pre_charge) {
  int rc = hook_rows_check(ctx, n, rows);
  if (rc || n == 0) return rc;
  const int64_t m = hook_chunk(ctx);
  if (n > m) {
    for (int64_t o = 0; o < n; o += m) {
      rc = mars_on_service(ctx, std::min(m, n - o), rows + o, tokens + o, now + o,
                           pre_charge ? pre_charge + o : nullptr);
      if (rc) return rc;
    }
    return MARS_OK;
  }
  CK(cudaSetDevice(ctx->device));
  u8* st = ctx->d_stage;
  CK(cudaMemcpyAsync(st, rows, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(st + n * 8, tokens, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(st + n * 16, now, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  const i64* pre = nullptr;
  if (pre_charge) {
    // (the rows' staging slot is reused: pre-charge states go to the upsert index buffer)
    CK(cudaMemcpyAsync(ctx->d_rows, pre_charge, n * 8, cudaMemcpyHostToDevice, ctx->stream));
    pre = ctx->d_rows;
  }
  rc = mars_enqueue_service_rows(ctx->stream, ctx->tab, ctx->cfg, n, (const i64*)st,
                                 (const i64*)(st + n * 8), (const double*)(st + n * 16), pre,
                                 ctx->d_hook_st);
  if (rc) return fail(ctx, MARS_ERR_CUDA, "service rows: %s", cudaGetErrorString((cudaError_t)rc));
  return hook_status(ctx);
}

int mars_expired_pins(mars_ctx* ctx, double now, int64_t cap, uint32_t* rows, int64_t* n) {
  if (!ctx || !n || cap < 0 || (cap > 0 && !rows)) return MARS_ERR_ARG;
  CK(cudaSetDevice(ctx->device));
  u8* st = ctx->d_stage;  // [count][rows...]
  const i64 room = std::min<i64>(cap, (ctx->alloc_rows * 8 - 16) / 4);
  int rc = mars_enqueue_expired_rows(ctx->stream, ctx->tab, ctx->n_rows, now, (u32*)(st + 16),
                                     room, (int*)st, ctx->num_sms * 4);
  if (rc) return fail(ctx, MARS_ERR_CUDA, "expired rows: %s", cudaGetErrorString((cudaError_t)rc));
  int cnt = 0;
  CK(cudaMemcpyAsync(&cnt, st, sizeof cnt, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  *n = cnt;
  if (cnt > room) return fail(ctx, MARS_ERR_CAPACITY, "%d expired pins > %lld", cnt, (long long)room);
  if (cnt > 0) {
    CK(cudaMemcpyAsync(rows, st + 16, (size_t)cnt * 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  return MARS_OK;
}

int mars_get_queue(mars_ctx* ctx, int64_t cap, uint32_t* rows, int64_t* n) {
  if (!ctx || !n) return MARS_ERR_ARG;
  CK(cudaSetDevice(ctx->device));
  int64_t len = 0;
  i32 sel = 0;
  CK(cudaMemcpyAsync(&len, &ctx->sc->queue_len, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(&sel, ctx->qsel, 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  *n = len;
  if (rows && len) {
    int64_t m = len < cap ? len : cap;
    CK(cudaMemcpy(rows, ctx->queue.row[sel], m * 4, cudaMemcpyDeviceToHost));
  }
  ctx->q_upper = len;
  return MARS_OK;
}

int mars_set_scalars(mars_ctx* ctx, const mars_scalars* s) {
  if (!ctx || !s) return MARS_ERR_ARG;
  if (s->total_blocks < 1 || s->free_blocks < 0 || s->free_blocks > s->total_blocks)
    return fail(ctx, MARS_ERR_CONTRACT, "bad pool counters");
  CK(cudaSetDevice(ctx->device));
  // stream-ordered, no host wait: the pinned staging copy is rewritten only
  // once its previous upload completed (ev_sc)
  CK(cudaEventSynchronize(ctx->ev_sc));
  *ctx->h_sc = *s;
  CK(cudaMemcpyAsync(ctx->sc, ctx->h_sc, sizeof(mars_scalars), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaEventRecord(ctx->ev_sc, ctx->stream));
  ctx->q_upper = s->queue_len;
  return MARS_OK;
}

int mars_get_scalars(mars_ctx* ctx, mars_scalars* s) {
  if (!ctx || !s) return MARS_ERR_ARG;
  CK(cudaSetDevice(ctx->device));
  CK(cudaMemcpyAsync(ctx->h_sc, ctx->sc, sizeof(mars_scalars), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  *s = *ctx->h_sc;
  return MARS_OK;
}

static LaunchArgs launch_args(mars_ctx* ctx, const mars_step_in* in) {
  LaunchArgs a;
  a.stream = ctx->stream;
  a.side = ctx->side;
  a.ev_fork = ctx->ev_fork;
  a.ev_join = ctx->ev_join;
  a.side2 = ctx->side2;
  a.ev_head = ctx->ev_head;
  a.ev_pack = ctx->ev_pack;
  a.ev_kvx = ctx->ev_kvx;
  a.tab = ctx->tab;
  a.cfg = ctx->cfg;
  a.work = ctx->work;
  a.bufs = ctx->bufs;
  a.sc = ctx->sc;
  a.queue = ctx->queue;
  a.qlsd = ctx->qlsd;
  a.xlsd = ctx->xlsd;
  a.qsel = ctx->qsel;
  a.host_in = ctx->h_in;
  a.n_rows = ctx->n_rows;
  a.num_sms = ctx->num_sms;
  a.control_possible = in->control_due ? 1 : 0;
  a.queue_upper = ctx->q_upper;
  a.ctl_per_cta = ctx->ctl_per_cta;
  int passes = 0;
  if (ctx->q_upper > SORT_CAP) {
    unsigned mx = (unsigned)(ctx->q_maxreq > 0 ? ctx->q_maxreq : 1);
    passes = 1;
    while (passes < 4 && (mx >> (8 * passes)) != 0) passes++;
  }
  a.queue_passes = passes;
  a.exp_sort = (!(in->mode & MARS_MODE_SKIP_EXPIRY) && !(in->mode & MARS_MODE_RANK_ORDERED)) ? 1 : 0;
  a.exp_may_be_big = (a.exp_sort && ctx->n_rows > SORT_CAP) ? 1 : 0;
  a.prof = ctx->profiling ? ctx->prof : nullptr;
  a.prof_used = ctx->prof_used;
  a.kv = ctx->kv_on ? &ctx->kv : nullptr;
  a.phase = 0;
  a.sharded = (in->mode & MARS_MODE_SHARDED) ? 1 : 0;
  a.x = ctx->x;
  // pack_queue's big-list sort concurrently with k_scan: table-backed local
  // queues only (the sharded list exists only after the exchange)
  a.pack_ctas = ctx->pack_ctas;
  a.advance = (in->mode & MARS_MODE_ADVANCE) ? 1 : 0;
  // only lists the few pack CTAs rank in one warp-segment batch per pass
  // (<= LSD_SEG_J x 1024 entries each); longer lists sort on the whole grid
  // inside k_control, after the scan
  a.pack_early = (a.control_possible && !(in->mode & (MARS_MODE_SHARDED | MARS_MODE_NO_ROWS)) &&
                  a.queue_passes > 0 && a.queue_passes <= 3 && ctx->pack_ctas > 0 &&
                  ctx->pack_ctas < ctx->num_sms / 2 &&
                  ctx->q_upper <= (i64)ctx->pack_ctas * PACK_SEG_ENTRIES)
                     ? 1 : 0;
  a.gq.row[0] = a.gq.row[1] = ctx->x.gq_row;
  a.gq.req[0] = a.gq.req[1] = ctx->x.gq_req;
  a.gq.lng[0] = a.gq.lng[1] = ctx->x.gq_lng;
  a.gq.gpos[0] = a.gq.gpos[1] = nullptr;
  a.gq.cap = ctx->x.cap * ctx->x.world;
  if (a.sharded) {
    a.queue_upper = ctx->x.cap * ctx->x.world;
    a.queue_passes = a.queue_upper > SORT_CAP ? 4 : 0;
  }
  return a;
}

// one cached step graph dropped (exec, the captured graph it came from)
static void drop_graph(mars_ctx* ctx, int i) {
  if (ctx->graph_exec[i]) cudaGraphExecDestroy(ctx->graph_exec[i]);
  if (ctx->graph_g[i]) cudaGraphDestroy(ctx->graph_g[i]);
  ctx->graph_exec[i] = nullptr;
  ctx->graph_g[i] = nullptr;
  ctx->init_node[i] = nullptr;
}

int mars_step_enqueue(mars_ctx* ctx, const mars_step_in* in) {
  if (!ctx || !in) return MARS_ERR_ARG;
  if (in->control_due && ctx->cfg.policy != POL_MARS)  // PolicyBase.uses_admission_control
    return fail(ctx, MARS_ERR_ARG, "the comparison policies have no admission control");
  CK(cudaSetDevice(ctx->device));
  *ctx->h_in = *in;
  // the device tick tail includes the tick-end MLFQ charges (sim.py:364)
  if (in->mode & MARS_MODE_ADVANCE) ctx->h_in->mode |= MARS_MODE_SERVICE;
  LaunchArgs a = launch_args(ctx, in);
  if (!ctx->use_graph || ctx->profiling) {  // event timing does not work inside graphs
    ctx->last_launches = mars_enqueue_step(&a);
    CK(cudaGetLastError());
    return MARS_OK;
  }
  // whole-step CUDA graph, re-captured only when the launch shape changes
  i64 qb = 1;
  while (qb < a.queue_upper) qb <<= 1;
  long long key[mars_ctx::NKEY] = {a.n_rows, a.control_possible, a.queue_passes, qb, a.exp_sort,
                                   a.exp_may_be_big, a.prof ? 1 : 0,
                                   (long long)(uintptr_t)ctx->stream, a.pack_early, a.advance,
                                   a.kv ? 1 : 0};
  int gi = -1;
  for (int i = 0; i < mars_ctx::NGRAPH; ++i)
    if (ctx->graph_exec[i] && memcmp(key, ctx->graph_key[i], sizeof key) == 0) gi = i;
  if (gi < 0) {
    // evict the least recently used entry (or take an empty one)
    gi = 0;
    for (int i = 0; i < mars_ctx::NGRAPH; ++i) {
      if (!ctx->graph_exec[i]) {
        gi = i;
        break;
      }
      if (ctx->graph_used[i] < ctx->graph_used[gi]) gi = i;
    }
    drop_graph(ctx, gi);
    cudaGraph_t g = nullptr;
    if (ctx->stream == nullptr || ctx->stream == cudaStreamLegacy ||
        ctx->stream == cudaStreamPerThread)
      return fail(ctx, MARS_ERR_ARG, "graph mode needs a non-default stream");
    CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    ctx->graph_launches[gi] = mars_enqueue_step(&a);
    cudaError_t ce = cudaStreamEndCapture(ctx->stream, &g);
    if (ce != cudaSuccess) {
      cudaGetLastError();
      return fail(ctx, MARS_ERR_CUDA, "graph capture failed: %s", cudaGetErrorString(ce));
    }
    CK(cudaGraphInstantiate(&ctx->graph_exec[gi], g, 0));
    ctx->graph_g[gi] = g;
    // the step head's node: this step's input goes in as its parameter
    size_t nn = 0;
    CK(cudaGraphGetNodes(g, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    CK(cudaGraphGetNodes(g, nodes.data(), &nn));
    for (size_t i = 0; i < nn; ++i) {
      cudaGraphNodeType ty;
      CK(cudaGraphNodeGetType(nodes[i], &ty));
      if (ty != cudaGraphNodeTypeKernel) continue;
      cudaKernelNodeParams kp;
      CK(cudaGraphKernelNodeGetParams(nodes[i], &kp));
      if (kp.func == mars_work_init_fn()) {
        ctx->init_node[gi] = nodes[i];
        ctx->init_params[gi] = kp;
      }
    }
    if (!ctx->init_node[gi]) return fail(ctx, MARS_ERR_CUDA, "step graph without its head node");
    memcpy(ctx->graph_key[gi], key, sizeof key);
  }
  ctx->graph_used[gi] = ++ctx->graph_clock;
  {
    cudaKernelNodeParams kp = ctx->init_params[gi];
    Work* w = ctx->work;
    mars_step_in v = *ctx->h_in;
    const mars_scalars* sc = ctx->sc;
    void* args[] = {&w, &v, &sc};
    kp.kernelParams = args;
    kp.extra = nullptr;
    CK(cudaGraphExecKernelNodeSetParams(ctx->graph_exec[gi], ctx->init_node[gi], &kp));
  }
  CK(cudaGraphLaunch(ctx->graph_exec[gi], ctx->stream));
  ctx->last_launches = ctx->graph_launches[gi];
  return MARS_OK;
}

int mars_sync(mars_ctx* ctx) {
  if (!ctx) return MARS_ERR_ARG;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaStreamSynchronize(ctx->side));
  CK(cudaStreamSynchronize(ctx->side2));
  CK(cudaGetLastError());
  return MARS_OK;
}

int mars_set_graph(mars_ctx* ctx, int on) {
  if (!ctx) return MARS_ERR_ARG;
  ctx->use_graph = on != 0;
  return MARS_OK;
}

int mars_set_config(mars_ctx* ctx, const mars_config* hcfg) {
  if (!ctx || !hcfg) return MARS_ERR_ARG;
  if (hcfg->policy != ctx->hcfg.policy)
    return fail(ctx, MARS_ERR_ARG, "mars_set_config cannot change the policy");
  if (hcfg->window_size < 1 || hcfg->window_size > WIN_MAX || hcfg->num_levels < 1 ||
      hcfg->num_levels > 4 || hcfg->block_size < 1 || hcfg->token_budget < 1 ||
      hcfg->max_decode_slots < 0)
    return fail(ctx, MARS_ERR_ARG, "invalid mars_config");
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  // the captured step graphs carry the old configuration as kernel parameters
  for (int i = 0; i < mars_ctx::NGRAPH; ++i) drop_graph(ctx, i);
  memset(ctx->graph_key, 0, sizeof ctx->graph_key);
  ctx->hcfg = *hcfg;
  ctx->cfg = make_cfg(*hcfg);
  return MARS_OK;
}

int mars_step_fetch(mars_ctx* ctx, mars_step_out* o) {
  if (!ctx || !o) return MARS_ERR_ARG;
  CK(cudaSetDevice(ctx->device));
  // ONE kernel behind the step writes the final Work and every output array
  // into the mapped arena (laid out on the device from the counts), then ONE
  // synchronize: no host round trip for the counts first
  const Bufs& b = ctx->bufs;
  OutSrc S;
  {
    const void* src[OS_N] = {b.exp_row_sorted, b.exp_blk_sorted, b.admitted, ctx->x.adm_idx,
                             b.win_rows, b.dec_rows, b.pre_rows, b.pre_grant, b.ev_row,
                             b.ev_kind, b.ev_blk, b.j_op, b.j_row, b.j_n, b.ret_row, b.ret_pin,
                             b.ret_b, b.ret_c, b.ret_d, b.dec_level, b.pre_level, b.svc_pre,
                             b.end_row, b.end_kind, b.end_blk, b.end_pin, b.end_b, b.end_c,
                             b.end_d, b.pre_done, b.fin_row, b.fin_pin, b.fin_b, b.fin_c,
                             b.fin_d};
    memcpy(S.p, src, sizeof src);
    S.ev_cap = b.ev_cap;
    S.j_cap = b.j_cap;
    S.coord = ctx->cfg.coord;
  }
  {
    int rc = mars_enqueue_out_fold(ctx->stream, ctx->work, S, ctx->h_out,
                                   (long long)ctx->h_out_bytes);
    if (rc) return fail(ctx, MARS_ERR_CUDA, "fetch: %s", cudaGetErrorString((cudaError_t)rc));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaGetLastError());
  memcpy(ctx->h_work, ctx->h_out, sizeof(Work));
  const Work& w = *ctx->h_work;
  OutLay L;
  out_layout(w, S, (long long)ctx->h_out_bytes, &L);
  auto at = [&](int k) -> const void* { return L.off[k] < 0 ? nullptr : ctx->h_out + L.off[k]; };
  memset(o, 0, sizeof *o);
  o->status = w.status;
  o->n_expired = w.n_exp;
  const bool sharded = (w.in.mode & MARS_MODE_SHARDED) != 0;
  const i64 n_adm = sharded ? (i64)w.n_adm_own : w.take;
  o->n_admitted = (int32_t)n_adm;
  o->n_window = w.n_window;
  o->n_decode = w.n_dec;
  o->n_prefill = w.n_pre;
  o->n_evict = w.n_evict;
  o->n_journal = w.n_journal;
  o->n_retention = w.n_ret;
  o->n_ready = w.n_ready;
  o->n_promoted = w.n_promoted;
  o->pack_mode = w.pack_mode;
  o->total_tokens = w.total_tokens;
  o->free_after_expiry = w.free_after_expiry;
  o->limit = w.limit;
  o->slots = w.slots;
  o->expired_rows = (const uint32_t*)at(OS_EXP_ROW);
  o->expired_blocks = (const int32_t*)at(OS_EXP_BLK);
  o->admitted_rows = (const uint32_t*)at(OS_ADM);
  const uint32_t* adm_idx = (const uint32_t*)at(OS_ADM_IDX);
  o->window_rows = (const uint32_t*)at(OS_WIN);
  o->decode_rows = (const uint32_t*)at(OS_DEC);
  o->prefill_rows = (const uint32_t*)at(OS_PRE);
  o->prefill_grants = (const int32_t*)at(OS_PRE_GRANT);
  o->evict_rows = (const uint32_t*)at(OS_EV_ROW);
  o->evict_kind = (const uint8_t*)at(OS_EV_KIND);
  o->evict_blocks = (const int32_t*)at(OS_EV_BLK);
  o->journal_op = (const uint8_t*)at(OS_J_OP);
  o->journal_row = (const uint32_t*)at(OS_J_ROW);
  o->journal_n = (const int32_t*)at(OS_J_N);
  o->ret_rows = (const uint32_t*)at(OS_RET_ROW);
  o->ret_pin = (const uint8_t*)at(OS_RET_PIN);
  o->ret_benefit = (const double*)at(OS_RET_B);
  o->ret_cost = (const double*)at(OS_RET_C);
  o->ret_deadline = (const double*)at(OS_RET_D);
  o->decode_level = (const uint8_t*)at(OS_DEC_LEVEL);
  o->prefill_level = (const uint8_t*)at(OS_PRE_LEVEL);
  if (L.bytes[OS_SVC_PRE]) o->plan_pre_charge = (const int64_t*)at(OS_SVC_PRE);
  o->n_finish = w.n_finish;
  o->n_window_cand = w.n_wc;
  o->n_victim_cand = w.n_vc;
  o->walk_slow = w.walk_slow;
  o->sort_path = w.sort_path;
  o->n_fullscan = w.n_fullscan;
  o->ref_flags = (w.ref_on[0] ? 1 : 0) | (w.ref_on[1] ? 2 : 0);
  o->ref_rounds = w.ref_iters;
  o->n_window_ref = w.n_wr;
  o->n_victim_ref = w.n_vr;
  o->n_round_end = w.n_round_end;
  o->n_done = w.n_done;
  o->end_rows = (const uint32_t*)at(OS_END_ROW);
  o->end_kind = (const uint8_t*)at(OS_END_KIND);
  o->end_blocks = (const int32_t*)at(OS_END_BLK);
  o->end_pin = (const uint8_t*)at(OS_END_PIN);
  o->end_benefit = (const double*)at(OS_END_B);
  o->end_cost = (const double*)at(OS_END_C);
  o->end_deadline = (const double*)at(OS_END_D);
  o->prefill_done = (w.in.mode & MARS_MODE_ADVANCE) ? (const uint8_t*)at(OS_PRE_DONE) : nullptr;
  o->fin_rows = (const uint32_t*)at(OS_FIN_ROW);
  o->fin_pin = (const uint8_t*)at(OS_FIN_PIN);
  o->fin_benefit = (const double*)at(OS_FIN_B);
  o->fin_cost = (const double*)at(OS_FIN_C);
  o->fin_deadline = (const double*)at(OS_FIN_D);
  if (sharded && n_adm > 1) {
    // this replica's admitted rows in global packed order
    std::vector<std::pair<uint32_t, uint32_t>> pr((size_t)n_adm);
    for (i64 i = 0; i < n_adm; ++i) pr[i] = {adm_idx[i], o->admitted_rows[i]};
    std::sort(pr.begin(), pr.end());
    uint32_t* dst = const_cast<uint32_t*>(o->admitted_rows);
    for (i64 i = 0; i < n_adm; ++i) dst[i] = pr[i].second;
  }
  // free_blocks after the plan (MARS_MODE_ADVANCE's tail frees come after)
  o->free_blocks = w.free_after_plan;
  if (sharded) {
    int64_t ql = 0;
    CK(cudaMemcpy(&ql, &ctx->sc->queue_len, 8, cudaMemcpyDeviceToHost));
    ctx->q_upper = ql;
  } else {
    ctx->q_upper -= w.take;
  }
  if (ctx->q_upper < 0) ctx->q_upper = 0;
  return MARS_OK;
}

int mars_output_arena(mars_ctx* ctx, void** base, int64_t* bytes) {
  if (!ctx || !base || !bytes) return MARS_ERR_ARG;
  *base = ctx->h_out;
  *bytes = (int64_t)ctx->h_out_bytes;
  return MARS_OK;
}

int mars_step(mars_ctx* ctx, const mars_step_in* in, mars_step_out* out) {
  int rc = mars_step_enqueue(ctx, in);
  if (rc) return rc;
  return mars_step_fetch(ctx, out);
}

// ---------------------------------------------------------------------------
// sharded replicas
// ---------------------------------------------------------------------------

int mars_shard_init(mars_ctx* ctx, int world, int rank) {
  if (!ctx || world < 1 || rank < 0 || rank >= world) return MARS_ERR_ARG;
  CK(cudaSetDevice(ctx->device));
  Xchg& x = ctx->x;
  if (x.xc) return fail(ctx, MARS_ERR_ARG, "already sharded");
  x.world = world;
  x.rank = rank;
  x.cap = ctx->max_queue;
  const i64 words = 1 + x.cap;  // count, then one word per entry
  CK(cudaMalloc((void**)&x.xc, XC_N * 8));
  CK(cudaMemset(x.xc, 0, XC_N * 8));
  CK(cudaMalloc((void**)&x.xsend, words * 8));
  CK(cudaMalloc((void**)&x.xrecv, words * 8 * world));
  CK(cudaMalloc((void**)&x.gq_row, x.cap * world * 4));
  CK(cudaMalloc((void**)&x.gq_req, x.cap * world * 4));
  CK(cudaMalloc((void**)&x.gq_lng, x.cap * world));
  CK(cudaMalloc((void**)&x.adm_idx, x.cap * 4));
  // the all-gathered list can be world x longer than the local one
  for (Lsd* l : {&ctx->qlsd}) {
    if (l->cap < x.cap * world) {
      for (int i = 0; i < 2; ++i) {
        cudaFree(l->k[i]);
        cudaFree(l->v[i]);
        CK(cudaMalloc((void**)&l->k[i], x.cap * world * 8));
        CK(cudaMalloc((void**)&l->v[i], x.cap * world * 4));
      }
      l->cap = x.cap * world;
    }
  }
  return MARS_OK;
}

int mars_shard_buffers(mars_ctx* ctx, void** xc, void** xsend, void** xrecv, int64_t* send_words) {
  if (!ctx || !ctx->x.xc) return MARS_ERR_ARG;
  if (xc) *xc = ctx->x.xc;
  if (xsend) *xsend = ctx->x.xsend;
  if (xrecv) *xrecv = ctx->x.xrecv;
  if (send_words) *send_words = 1 + ctx->x.cap;
  return MARS_OK;
}

int mars_set_queue_gpos(mars_ctx* ctx, int64_t n, const uint32_t* gpos) {
  if (!ctx || n < 0) return MARS_ERR_ARG;
  if (n > ctx->max_queue) return MARS_ERR_CAPACITY;
  CK(cudaSetDevice(ctx->device));
  i32 sel = 0;
  CK(cudaMemcpyAsync(&sel, ctx->qsel, 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (n) CK(cudaMemcpy(ctx->queue.gpos[sel], gpos, n * 4, cudaMemcpyHostToDevice));
  return MARS_OK;
}

int mars_get_queue_gpos(mars_ctx* ctx, int64_t cap, uint32_t* gpos, int64_t* n) {
  if (!ctx || !n) return MARS_ERR_ARG;
  CK(cudaSetDevice(ctx->device));
  int64_t len = 0;
  i32 sel = 0;
  CK(cudaMemcpyAsync(&len, &ctx->sc->queue_len, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(&sel, ctx->qsel, 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  *n = len;
  if (gpos && len) CK(cudaMemcpy(gpos, ctx->queue.gpos[sel], (len < cap ? len : cap) * 4,
                                 cudaMemcpyDeviceToHost));
  return MARS_OK;
}

int mars_step_phase(mars_ctx* ctx, const mars_step_in* in, int phase) {
  if (!ctx || !in || phase < 1 || phase > 2) return MARS_ERR_ARG;
  if (!ctx->x.xc || !(in->mode & MARS_MODE_SHARDED))
    return fail(ctx, MARS_ERR_ARG, "mars_step_phase needs mars_shard_init + MARS_MODE_SHARDED");
  CK(cudaSetDevice(ctx->device));
  if (phase == 1) {
    *ctx->h_in = *in;
    if (in->mode & MARS_MODE_ADVANCE) ctx->h_in->mode |= MARS_MODE_SERVICE;
  }
  LaunchArgs a = launch_args(ctx, ctx->h_in);
  a.phase = phase;
  ctx->last_launches = mars_enqueue_step(&a) + (phase == 2 ? ctx->last_launches : 0);
  CK(cudaGetLastError());
  return MARS_OK;
}

int mars_resume(mars_ctx* ctx, int64_t n, const int64_t* rows, const double* finish_time,
                const double* duration, const int32_t* new_prefill, const int32_t* decode_tokens,
                double now, int32_t* counts) {
  if (!ctx || n < 0 || !counts) return MARS_ERR_ARG;
  counts[0] = counts[1] = counts[2] = 0;
  if (n == 0) return MARS_OK;
  if (n > ctx->max_rows) return MARS_ERR_CAPACITY;
  for (i64 i = 0; i < n; ++i)
    if (rows[i] < 0 || rows[i] >= ctx->n_rows) return fail(ctx, MARS_ERR_ARG, "resume row out of range");
  CK(cudaSetDevice(ctx->device));
  if (!ctx->d_resume) {
    CK(cudaMalloc(&ctx->d_resume, (size_t)ctx->max_rows * 52 + 256));
  }
  unsigned char* p = (unsigned char*)ctx->d_resume;
  i64* drows = (i64*)p;
  double* dfin = (double*)(drows + n);
  double* ddur = dfin + n;
  i32* dnew = (i32*)(ddur + n);
  i32* ddec = dnew + n;
  int* dcnt = (int*)(ddec + ((n + 1) & ~1ll));
  // per-row outcome (mars_resume_rows): after the counts, 16-byte aligned
  const i64 mr = ctx->max_rows;
  i32* o_blk = (i32*)((unsigned char*)ctx->d_resume + mr * 32 + 64);
  i32* o_ctx = o_blk + mr;
  i32* o_need = o_ctx + mr;
  i32* o_proj = o_need + mr;
  u8* o_kind = (u8*)(o_proj + mr);
  ctx->last_resume_n = n;
  CK(cudaMemcpyAsync(drows, rows, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(dfin, finish_time, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ddur, duration, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(dnew, new_prefill, n * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ddec, decode_tokens, n * 4, cudaMemcpyHostToDevice, ctx->stream));
  int rc = mars_enqueue_resume(ctx->tab, ctx->cfg, ctx->sc, ctx->stream, n, drows, dfin, ddur,
                               dnew, ddec, now, dcnt, o_kind, o_blk, o_ctx, o_need, o_proj);
  if (rc) return fail(ctx, MARS_ERR_CUDA, "resume: %s", cudaGetErrorString((cudaError_t)rc));
  if (ctx->kv_on) {
    rc = mars_kv_enqueue_resume_free(ctx->kv, ctx->stream, n, drows, o_kind);
    if (rc) return fail(ctx, MARS_ERR_CUDA, "resume kv: %s", cudaGetErrorString((cudaError_t)rc));
  }
  int hc[4] = {0, 0, 0, 0};
  CK(cudaMemcpyAsync(hc, dcnt, sizeof hc, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  counts[0] = hc[0];
  counts[1] = hc[1];
  counts[2] = hc[2];
  if (hc[3]) return fail(ctx, MARS_ERR_CONTRACT, "resume owes a prefill other than its cost");
  return MARS_OK;
}

int mars_resume_rows(mars_ctx* ctx, int64_t n, uint8_t* kind, int32_t* blocks, int32_t* context,
                     int32_t* need, int32_t* projected) {
  if (!ctx || n < 0) return MARS_ERR_ARG;
  if (n != ctx->last_resume_n) return fail(ctx, MARS_ERR_ARG, "resume_rows: %lld rows, the last resume had %lld",
                                           (long long)n, (long long)ctx->last_resume_n);
  if (n == 0) return MARS_OK;
  CK(cudaSetDevice(ctx->device));
  const i64 mr = ctx->max_rows;
  i32* o_blk = (i32*)((unsigned char*)ctx->d_resume + mr * 32 + 64);
  CK(cudaMemcpyAsync(blocks, o_blk, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(context, o_blk + mr, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(need, o_blk + 2 * mr, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(projected, o_blk + 3 * mr, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(kind, (u8*)(o_blk + 4 * mr), n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return MARS_OK;
}

int mars_retention_batch(mars_ctx* ctx, int64_t n, const int32_t* context, const int32_t* kv,
                         int64_t total_blocks, double usage, double ema, double now,
                         uint8_t* pin, double* benefit, double* cost, double* deadline) {
  if (!ctx || n < 0) return MARS_ERR_ARG;
  if (n == 0) return MARS_OK;
  if (n > ctx->max_rows) return MARS_ERR_CAPACITY;
  if (total_blocks < 1) return fail(ctx, MARS_ERR_CONTRACT, "total_blocks must be >= 1");
  CK(cudaSetDevice(ctx->device));
  // staging: ctx[n] | kv[n] in d_stage (8 B per row), outputs in the retention buffers
  i32* dctx = (i32*)ctx->d_stage;
  i32* dkv = dctx + n;
  CK(cudaMemcpyAsync(dctx, context, n * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(dkv, kv, n * 4, cudaMemcpyHostToDevice, ctx->stream));
  const Bufs& b = ctx->bufs;
  int rc = mars_enqueue_retention(ctx->cfg, ctx->stream, n, dctx, dkv, total_blocks, usage, ema,
                                  now, b.ret_pin, b.ret_b, b.ret_c, b.ret_d);
  if (rc) return fail(ctx, MARS_ERR_CUDA, "retention: %s", cudaGetErrorString((cudaError_t)rc));
  CK(cudaMemcpyAsync(pin, b.ret_pin, n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(benefit, b.ret_b, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(cost, b.ret_c, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(deadline, b.ret_d, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return MARS_OK;
}

// every admission-list array (both buffers) and its size
static void queue_arrays(mars_ctx* ctx, void** qp, size_t* qs) {
  const size_t Qc = (size_t)ctx->max_queue;
  for (int b = 0; b < 2; ++b) {
    qp[4 * b + 0] = ctx->queue.row[b];
    qs[4 * b + 0] = Qc * 4;
    qp[4 * b + 1] = ctx->queue.req[b];
    qs[4 * b + 1] = Qc * 4;
    qp[4 * b + 2] = ctx->queue.lng[b];
    qs[4 * b + 2] = Qc;
    qp[4 * b + 3] = ctx->queue.gpos[b];
    qs[4 * b + 3] = Qc * 4;
  }
}

int mars_checkpoint(mars_ctx* ctx) {
  if (!ctx) return MARS_ERR_ARG;
  CK(cudaSetDevice(ctx->device));
  for (auto& cs : ctx->cols) {
    if (!cs.ckpt) CK(cudaMalloc(&cs.ckpt, (size_t)ctx->alloc_rows * cs.esz));
    CK(cudaMemcpyAsync(cs.ckpt, *cs.dev, (size_t)ctx->n_rows * cs.esz, cudaMemcpyDeviceToDevice,
                       ctx->stream));
  }
  size_t qs[8];
  void* qp[8];
  queue_arrays(ctx, qp, qs);
  for (int i = 0; i < 8; ++i) {
    if (!ctx->ck_q[i]) CK(cudaMalloc(&ctx->ck_q[i], qs[i]));
    CK(cudaMemcpyAsync(ctx->ck_q[i], qp[i], qs[i], cudaMemcpyDeviceToDevice, ctx->stream));
  }
  if (!ctx->ck_sc) CK(cudaMalloc((void**)&ctx->ck_sc, sizeof(mars_scalars)));
  if (!ctx->ck_qsel) CK(cudaMalloc((void**)&ctx->ck_qsel, sizeof(i32)));
  CK(cudaMemcpyAsync(ctx->ck_sc, ctx->sc, sizeof(mars_scalars), cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->ck_qsel, ctx->qsel, sizeof(i32), cudaMemcpyDeviceToDevice, ctx->stream));
  if (ctx->kv_on) {  // the block manager's state with the table
    Kv& k = ctx->kv;
    const size_t kb[7] = {(size_t)k.rows * 4, (size_t)k.rows * k.D * 4,
                          (size_t)k.nchunks * KV_CH * 4, (size_t)k.seg_cap * 8,
                          (size_t)k.nchunks * 4, sizeof(KvScal), (size_t)k.total * 4};
    void* kp[7] = {k.len, k.dir, k.chunks, k.seg, k.cfs, k.s, k.arena};
    for (int i = 0; i < 7; ++i) {
      if (!ctx->ck_kv[i]) CK(cudaMalloc(&ctx->ck_kv[i], kb[i]));
      CK(cudaMemcpyAsync(ctx->ck_kv[i], kp[i], kb[i], cudaMemcpyDeviceToDevice, ctx->stream));
    }
    ctx->have_kv_ckpt = true;
  }
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->ck_q_upper = ctx->q_upper;
  ctx->ck_q_maxreq = ctx->q_maxreq;
  ctx->have_ckpt = true;
  return MARS_OK;
}

int mars_restore(mars_ctx* ctx) {
  if (!ctx) return MARS_ERR_ARG;
  if (!ctx->have_ckpt) return fail(ctx, MARS_ERR_ARG, "no checkpoint");
  CK(cudaSetDevice(ctx->device));
  const i64 Qc = ctx->max_queue;
  for (auto& cs : ctx->cols)
    CK(cudaMemcpyAsync(*cs.dev, cs.ckpt, (size_t)ctx->n_rows * cs.esz, cudaMemcpyDeviceToDevice,
                       ctx->stream));
  (void)Qc;
  size_t qs[8];
  void* qp[8];
  queue_arrays(ctx, qp, qs);
  for (int i = 0; i < 8; ++i)
    CK(cudaMemcpyAsync(qp[i], ctx->ck_q[i], qs[i], cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->sc, ctx->ck_sc, sizeof(mars_scalars), cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->qsel, ctx->ck_qsel, sizeof(i32), cudaMemcpyDeviceToDevice, ctx->stream));
  ctx->q_upper = ctx->ck_q_upper;
  ctx->q_maxreq = ctx->ck_q_maxreq;
  if (ctx->kv_on && ctx->have_kv_ckpt) {
    Kv& k = ctx->kv;
    const size_t kb[7] = {(size_t)k.rows * 4, (size_t)k.rows * k.D * 4,
                          (size_t)k.nchunks * KV_CH * 4, (size_t)k.seg_cap * 8,
                          (size_t)k.nchunks * 4, sizeof(KvScal), (size_t)k.total * 4};
    void* kp[7] = {k.len, k.dir, k.chunks, k.seg, k.cfs, k.s, k.arena};
    for (int i = 0; i < 7; ++i)
      CK(cudaMemcpyAsync(kp[i], ctx->ck_kv[i], kb[i], cudaMemcpyDeviceToDevice, ctx->stream));
  }
  return MARS_OK;
}

int mars_set_profiling(mars_ctx* ctx, int on) {
  if (!ctx) return MARS_ERR_ARG;
  CK(cudaSetDevice(ctx->device));
  if (on && !ctx->prof[0])
    for (auto& e : ctx->prof) CK(cudaEventCreate(&e));
  ctx->profiling = on != 0;
  return MARS_OK;
}

int mars_kernel_times(mars_ctx* ctx, float* ms, int n) {
  if (!ctx || !ms) return MARS_ERR_ARG;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int k = 0; k < n && k < MARS_NUM_KTIMES; ++k) {
    ms[k] = -1.0f;
    if (ctx->profiling && ctx->prof_used[k]) {
      float t = 0;
      if (cudaEventElapsedTime(&t, ctx->prof[2 * k], ctx->prof[2 * k + 1]) == cudaSuccess)
        ms[k] = t;
      else
        cudaGetLastError();  // do not leave the failure pending for the next call
    }
  }
  return MARS_OK;
}

int mars_flush_l2(mars_ctx* ctx, int64_t bytes) {
  if (!ctx || bytes < 0) return MARS_ERR_ARG;
  CK(cudaSetDevice(ctx->device));
  if (bytes > ctx->bufs.flush_bytes) {
    cudaFree(ctx->bufs.flush);
    ctx->bufs.flush = nullptr;
    CK(cudaMalloc((void**)&ctx->bufs.flush, (size_t)bytes));
    ctx->bufs.flush_bytes = bytes;
  }
  int rc = mars_enqueue_flush(ctx->stream, ctx->bufs.flush, bytes, ctx->flush_salt++);
  if (rc >= 1000)
    return fail(ctx, MARS_ERR_CUDA, "flush: pending error from an earlier call: %s",
                cudaGetErrorString((cudaError_t)(rc - 1000)));
  if (rc) return fail(ctx, MARS_ERR_CUDA, "flush: %s", cudaGetErrorString((cudaError_t)rc));
  return MARS_OK;
}

// ---------------------------------------------------------------------------
// S5: block manager + host tier
// ---------------------------------------------------------------------------

static int kv_stage(mars_ctx* ctx, i64 bytes) {
  if (bytes <= ctx->kv_stage_bytes) return MARS_OK;
  cudaFree(ctx->kv_stage);
  ctx->kv_stage = nullptr;
  CK(cudaMalloc((void**)&ctx->kv_stage, (size_t)bytes));
  ctx->kv_stage_bytes = bytes;
  return MARS_OK;
}

int mars_kv_init(mars_ctx* ctx, const mars_kv_config* kc) {
  if (!ctx || !kc) return MARS_ERR_ARG;
  if (kc->total_blocks < 1 || kc->total_blocks > 0xffffffffll || kc->max_blocks_per_row < 1)
    return fail(ctx, MARS_ERR_ARG, "bad kv config");
  const i32 layers = kc->layers < 1 ? 1 : kc->layers;
  if (kc->block_bytes % (16ll * layers) != 0)
    return fail(ctx, MARS_ERR_ARG, "block_bytes must be a multiple of 16 * layers");
  CK(cudaSetDevice(ctx->device));
  if (ctx->kv_on) return fail(ctx, MARS_ERR_ARG, "kv manager already initialised");
  Kv& k = ctx->kv;
  k.total = kc->total_blocks;
  k.D = (kc->max_blocks_per_row + KV_CH - 1) / KV_CH;
  k.rows = ctx->alloc_rows;
  // table chunks (<= total/64 + rows) plus whole chunks on the free stack
  k.nchunks = 2 * ((k.total + KV_CH - 1) / KV_CH) + k.rows + 64;
  k.seg_cap = (k.total + KV_CH - 1) / KV_CH + 4 * k.rows + 65536;
  k.layers = layers;
  k.block_bytes = kc->block_bytes;
  k.host_blocks = kc->host_blocks;
  CK(cudaMalloc((void**)&k.seg, (size_t)k.seg_cap * 8));
  CK(cudaMalloc((void**)&k.arena, (size_t)k.total * 4));
  CK(cudaMalloc((void**)&k.xaoff, (size_t)k.rows * 8));
  CK(cudaMalloc((void**)&k.xroff, (size_t)k.rows * 8));
  CK(cudaMalloc((void**)&k.chunks, (size_t)k.nchunks * KV_CH * 4));
  CK(cudaMalloc((void**)&k.xoff, (size_t)k.rows * 8));
  CK(cudaMalloc((void**)&k.xlen, (size_t)k.rows * 4));
  CK(cudaMalloc((void**)&k.xbase, 32));
  CK(cudaMalloc((void**)&k.cfs, (size_t)k.nchunks * 4));
  CK(cudaMalloc((void**)&k.dir, (size_t)k.rows * k.D * 4));
  CK(cudaMalloc((void**)&k.len, (size_t)k.rows * 4));
  CK(cudaMalloc((void**)&k.s, sizeof(KvScal)));
  CK(cudaMemset(k.len, 0, (size_t)k.rows * 4));
  {
    std::vector<u32> iota((size_t)k.nchunks);
    for (i64 i = 0; i < k.nchunks; ++i) iota[i] = (u32)(k.nchunks - 1 - i);  // pops 0,1,2,..
    CK(cudaMemcpy(k.cfs, iota.data(), (size_t)k.nchunks * 4, cudaMemcpyHostToDevice));
  }
  KvScal s0 = {0, 0, 0, 0, k.nchunks, 0};
  CK(cudaMemcpy(k.s, &s0, sizeof s0, cudaMemcpyHostToDevice));
  if (k.block_bytes > 0) {
    CK(cudaMalloc((void**)&k.data, (size_t)k.total * k.block_bytes));
    if (k.host_blocks > 0) {
      CK(cudaHostAlloc(&ctx->kv_host, (size_t)k.host_blocks * k.block_bytes, cudaHostAllocMapped));
      void* dp = nullptr;
      CK(cudaHostGetDevicePointer(&dp, ctx->kv_host, 0));
      k.host = (u8*)dp;
    }
  }
  ctx->kv_on = true;
  return MARS_OK;
}

int mars_kv_apply(mars_ctx* ctx, int64_t n, const uint8_t* op, const uint32_t* row,
                  const int32_t* cnt) {
  if (!ctx || n < 0) return MARS_ERR_ARG;
  if (!ctx->kv_on) return fail(ctx, MARS_ERR_ARG, "kv manager not initialised");
  if (n == 0) return MARS_OK;
  for (int64_t i = 0; i < n; ++i)
    if ((i64)row[i] >= ctx->kv.rows) return fail(ctx, MARS_ERR_CAPACITY, "kv row out of range");
  CK(cudaSetDevice(ctx->device));
  int rc = kv_stage(ctx, n * 9 + 64);
  if (rc) return rc;
  u32* drow = (u32*)ctx->kv_stage;
  i32* dn = (i32*)(drow + n);
  u8* dop = (u8*)(dn + n);
  CK(cudaMemcpyAsync(drow, row, n * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(dn, cnt, n * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(dop, op, n, cudaMemcpyHostToDevice, ctx->stream));
  rc = mars_kv_enqueue_apply(ctx->kv, ctx->stream, n, dop, drow, dn);
  if (rc) return fail(ctx, MARS_ERR_CUDA, "kv apply: %s", cudaGetErrorString((cudaError_t)rc));
  KvScal s;
  CK(cudaMemcpyAsync(&s, ctx->kv.s, sizeof s, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (s.status) return fail(ctx, MARS_ERR_CONTRACT, "kv op stream broke the pool (status %d)", s.status);
  return MARS_OK;
}

int mars_kv_bulk_alloc(mars_ctx* ctx, int64_t n, const uint32_t* row, const int32_t* cnt) {
  if (!ctx || n < 0) return MARS_ERR_ARG;
  if (!ctx->kv_on) return fail(ctx, MARS_ERR_ARG, "kv manager not initialised");
  if (n == 0) return MARS_OK;
  for (int64_t i = 0; i < n; ++i) {
    if ((i64)row[i] >= ctx->kv.rows) return fail(ctx, MARS_ERR_CAPACITY, "kv row out of range");
    if (cnt[i] < 0) return fail(ctx, MARS_ERR_ARG, "negative block count");
  }
  {  // rows must be distinct (each row's IDs are one contiguous fresh range)
    std::vector<uint32_t> r(row, row + n);
    std::sort(r.begin(), r.end());
    if (std::adjacent_find(r.begin(), r.end()) != r.end())
      return fail(ctx, MARS_ERR_ARG, "bulk alloc rows must be distinct");
  }
  CK(cudaSetDevice(ctx->device));
  int rc = kv_stage(ctx, n * 8 + 64);
  if (rc) return rc;
  u32* drow = (u32*)ctx->kv_stage;
  i32* dn = (i32*)(drow + n);
  CK(cudaMemcpyAsync(drow, row, n * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(dn, cnt, n * 4, cudaMemcpyHostToDevice, ctx->stream));
  rc = mars_kv_enqueue_bulk(ctx->kv, ctx->stream, n, drow, dn, ctx->num_sms * 8);
  if (rc) return fail(ctx, MARS_ERR_CUDA, "kv bulk: %s", cudaGetErrorString((cudaError_t)rc));
  KvScal s;
  CK(cudaMemcpyAsync(&s, ctx->kv.s, sizeof s, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (s.status) return fail(ctx, MARS_ERR_CONTRACT, "kv bulk alloc needs a fresh pool (status %d)", s.status);
  return MARS_OK;
}

int mars_kv_table(mars_ctx* ctx, uint32_t row, int64_t cap, uint32_t* ids, int64_t* n) {
  if (!ctx || !n) return MARS_ERR_ARG;
  if (!ctx->kv_on) return fail(ctx, MARS_ERR_ARG, "kv manager not initialised");
  if ((i64)row >= ctx->kv.rows) return MARS_ERR_CAPACITY;
  CK(cudaSetDevice(ctx->device));
  i32 len = 0;
  CK(cudaMemcpyAsync(&len, ctx->kv.len + row, 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  *n = len;
  i64 m = len < cap ? len : cap;
  if (ids && m > 0) {
    int rc = kv_stage(ctx, m * 4);
    if (rc) return rc;
    rc = mars_kv_enqueue_table(ctx->kv, ctx->stream, row, m, (u32*)ctx->kv_stage);
    if (rc) return fail(ctx, MARS_ERR_CUDA, "kv table: %s", cudaGetErrorString((cudaError_t)rc));
    CK(cudaMemcpyAsync(ids, ctx->kv_stage, m * 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  return MARS_OK;
}

int mars_kv_state(mars_ctx* ctx, int64_t k, uint32_t* top_ids, int64_t* explicit_depth,
                  int64_t* fresh, int32_t* status) {
  if (!ctx) return MARS_ERR_ARG;
  if (!ctx->kv_on) return fail(ctx, MARS_ERR_ARG, "kv manager not initialised");
  CK(cudaSetDevice(ctx->device));
  KvScal s;
  CK(cudaMemcpyAsync(&s, ctx->kv.s, sizeof s, cudaMemcpyDeviceToHost, ctx->stream));
  if (top_ids && k > 0) {
    int rc = kv_stage(ctx, k * 4);
    if (rc) return rc;
    rc = mars_kv_enqueue_top(ctx->kv, ctx->stream, k, (u32*)ctx->kv_stage);
    if (rc) return fail(ctx, MARS_ERR_CUDA, "kv top: %s", cudaGetErrorString((cudaError_t)rc));
    CK(cudaMemcpyAsync(top_ids, ctx->kv_stage, k * 4, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  if (explicit_depth) *explicit_depth = s.fs_ids;
  if (fresh) *fresh = s.fresh;
  if (status) *status = s.status;
  return MARS_OK;
}

static int kv_move(mars_ctx* ctx, int64_t n, const uint32_t* ids, int64_t slot0, int method,
                   int dir) {
  if (!ctx || n < 0 || !ids) return MARS_ERR_ARG;
  Kv& k = ctx->kv;
  if (!ctx->kv_on || !k.data || !k.host) return fail(ctx, MARS_ERR_ARG, "no kv data tier");
  if (slot0 < 0 || slot0 + n > k.host_blocks) return fail(ctx, MARS_ERR_CAPACITY, "host slots");
  for (int64_t i = 0; i < n; ++i)
    if ((i64)ids[i] >= k.total) return fail(ctx, MARS_ERR_CONTRACT, "block id out of range");
  if (n == 0) return MARS_OK;
  CK(cudaSetDevice(ctx->device));
  const i64 piece = k.block_bytes / k.layers;
  if (method == 1) {
    int rc = kv_stage(ctx, n * 4);
    if (rc) return rc;
    CK(cudaMemcpyAsync(ctx->kv_stage, ids, n * 4, cudaMemcpyHostToDevice, ctx->stream));
    int grid = ctx->num_sms * 4;
    rc = mars_kv_enqueue_copy(k, ctx->stream, (const u32*)ctx->kv_stage, n, slot0, dir, grid);
    if (rc) return fail(ctx, MARS_ERR_CUDA, "kv copy: %s", cudaGetErrorString((cudaError_t)rc));
  } else if (method == 2) {
    // staged: HBM gather/scatter kernel + one large copy-engine DMA per chunk
    int rc = kv_stage(ctx, n * 4);
    if (rc) return rc;
    CK(cudaMemcpyAsync(ctx->kv_stage, ids, n * 4, cudaMemcpyHostToDevice, ctx->stream));
    const i64 chunk = KV_STAGE_BLOCKS;
    if (!ctx->kv_dstage) {
      CK(cudaMalloc((void**)&ctx->kv_dstage, (size_t)chunk * k.block_bytes));
      ctx->kv_dstage_blocks = chunk;
    }
    u8* hbase = (u8*)ctx->kv_host;
    for (i64 c0 = 0; c0 < n; c0 += chunk) {
      const i64 m = (n - c0) < chunk ? (n - c0) : chunk;
      const u32* cid = (const u32*)ctx->kv_stage + c0;
      const size_t bytes = (size_t)m * k.block_bytes;
      u8* hp = hbase + (size_t)(slot0 + c0) * k.block_bytes;
      if (dir == 0) {
        rc = mars_kv_enqueue_stage(k, ctx->stream, cid, m, ctx->kv_dstage, 0, ctx->num_sms * 2);
        if (rc) return fail(ctx, MARS_ERR_CUDA, "kv stage: %s", cudaGetErrorString((cudaError_t)rc));
        CK(cudaMemcpyAsync(hp, ctx->kv_dstage, bytes, cudaMemcpyDeviceToHost, ctx->stream));
      } else {
        CK(cudaMemcpyAsync(ctx->kv_dstage, hp, bytes, cudaMemcpyHostToDevice, ctx->stream));
        rc = mars_kv_enqueue_stage(k, ctx->stream, cid, m, ctx->kv_dstage, 1, ctx->num_sms * 2);
        if (rc) return fail(ctx, MARS_ERR_CUDA, "kv stage: %s", cudaGetErrorString((cudaError_t)rc));
      }
    }
  } else {
    u8* hbase = (u8*)ctx->kv_host;
    for (int64_t i = 0; i < n; ++i) {
      for (int l = 0; l < k.layers; ++l) {
        u8* dp = k.data + ((i64)l * k.total + ids[i]) * piece;
        u8* hp = hbase + ((slot0 + i) * k.layers + l) * piece;
        if (dir == 0)
          CK(cudaMemcpyAsync(hp, dp, piece, cudaMemcpyDeviceToHost, ctx->stream));
        else
          CK(cudaMemcpyAsync(dp, hp, piece, cudaMemcpyHostToDevice, ctx->stream));
      }
    }
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return MARS_OK;
}

// ---- host tier driven by the step's decisions ------
// Staged copies between scattered pool blocks and consecutive host slots
// [slot0, slot0 + n): gather / scatter kernels into an HBM staging area and
// one copy-engine DMA per ~128 MiB.
static int kv_stage_copy(mars_ctx* ctx, const u32* d_ids, i64 n, i64 slot0, int dir) {
  Kv& k = ctx->kv;
  const i64 chunk = std::max<i64>(KV_STAGE_BLOCKS, ((i64)128 << 20) / k.block_bytes);
  if (ctx->kv_dstage_blocks < chunk) {
    if (ctx->kv_dstage) cudaFree(ctx->kv_dstage);
    ctx->kv_dstage = nullptr;
    ctx->kv_dstage_blocks = 0;
    CK(cudaMalloc((void**)&ctx->kv_dstage, (size_t)chunk * k.block_bytes));
    ctx->kv_dstage_blocks = chunk;
  }
  u8* hbase = (u8*)ctx->kv_host;
  for (i64 c0 = 0; c0 < n; c0 += chunk) {
    const i64 m = (n - c0) < chunk ? (n - c0) : chunk;
    const size_t bytes = (size_t)m * k.block_bytes;
    u8* hp = hbase + (size_t)(slot0 + c0) * k.block_bytes;
    int rc;
    if (dir == 0) {
      rc = mars_kv_enqueue_stage(k, ctx->stream, d_ids + c0, m, ctx->kv_dstage, 0, ctx->num_sms * 4);
      if (rc) return fail(ctx, MARS_ERR_CUDA, "kv stage: %s", cudaGetErrorString((cudaError_t)rc));
      CK(cudaMemcpyAsync(hp, ctx->kv_dstage, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    } else {
      CK(cudaMemcpyAsync(ctx->kv_dstage, hp, bytes, cudaMemcpyHostToDevice, ctx->stream));
      rc = mars_kv_enqueue_stage(k, ctx->stream, d_ids + c0, m, ctx->kv_dstage, 1, ctx->num_sms * 4);
      if (rc) return fail(ctx, MARS_ERR_CUDA, "kv stage: %s", cudaGetErrorString((cudaError_t)rc));
    }
  }
  return MARS_OK;
}

// n IDs to the ring (wrapping); returns the first slot
static int kv_ring_put(mars_ctx* ctx, const u32* d_ids, i64 n, i64* slot0) {
  Kv& k = ctx->kv;
  if (n > k.host_blocks) return fail(ctx, MARS_ERR_CAPACITY, "host tier smaller than one offload");
  if (ctx->kv_ring + n > k.host_blocks) ctx->kv_ring = 0;
  *slot0 = ctx->kv_ring;
  int rc = kv_stage_copy(ctx, d_ids, n, ctx->kv_ring, 0);
  if (rc) return rc;
  ctx->kv_ring += n;
  return MARS_OK;
}

static int kv_tier_ready(mars_ctx* ctx) {
  if (!ctx) return MARS_ERR_ARG;
  if (!ctx->kv_on || !ctx->kv.data || !ctx->kv.host) return fail(ctx, MARS_ERR_ARG, "no kv data tier");
  return MARS_OK;
}

int mars_kv_capture(mars_ctx* ctx, int on) {
  int rc = kv_tier_ready(ctx);
  if (rc) return rc;
  Kv& k = ctx->kv;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  if (on && !k.cap) CK(cudaMalloc((void**)&k.cap, (size_t)k.total * 4));
  if (!on && k.cap) {
    cudaFree(k.cap);
    k.cap = nullptr;
  }
  // the step graphs carry the Kv struct as a kernel parameter
  for (int i = 0; i < mars_ctx::NGRAPH; ++i) drop_graph(ctx, i);
  memset(ctx->graph_key, 0, sizeof ctx->graph_key);
  return MARS_OK;
}

int mars_kv_offload_captured(mars_ctx* ctx, int64_t* n_blocks, int64_t* slot0, uint32_t* ids,
                             int64_t ids_cap) {
  int rc = kv_tier_ready(ctx);
  if (rc) return rc;
  Kv& k = ctx->kv;
  if (!k.cap) return fail(ctx, MARS_ERR_ARG, "capture is off");
  CK(cudaSetDevice(ctx->device));
  KvScal s;
  CK(cudaMemcpyAsync(&s, k.s, sizeof s, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (s.status & 128) return fail(ctx, MARS_ERR_CAPACITY, "capture list overflow");
  i64 s0 = -1;
  if (s.cap_n > 0) {
    rc = kv_ring_put(ctx, k.cap, s.cap_n, &s0);
    if (rc) return rc;
    if (ids && ids_cap > 0)
      CK(cudaMemcpyAsync(ids, k.cap, (size_t)std::min<i64>(ids_cap, s.cap_n) * 4,
                         cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemsetAsync(&k.s->cap_n, 0, sizeof(i64), ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  if (n_blocks) *n_blocks = s.cap_n;
  if (slot0) *slot0 = s0;
  return MARS_OK;
}

// the tables of n rows (row i holds counts[i] IDs) -> one device ID list
static int kv_rows_ids(mars_ctx* ctx, int64_t n, const int64_t* rows, const int32_t* counts,
                       i64* total) {
  Kv& k = ctx->kv;
  std::vector<i64> off((size_t)n + 1, 0);
  for (int64_t i = 0; i < n; ++i) {
    if (rows[i] < 0 || rows[i] >= k.rows || counts[i] < 0) return MARS_ERR_ARG;
    off[i + 1] = off[i] + counts[i];
  }
  *total = off[n];
  if (off[n] > ctx->kv_ids_cap) {
    if (ctx->kv_ids) cudaFree(ctx->kv_ids);
    ctx->kv_ids = nullptr;
    ctx->kv_ids_cap = 0;
    CK(cudaMalloc((void**)&ctx->kv_ids, (size_t)off[n] * 4 + 4));
    ctx->kv_ids_cap = off[n];
  }
  // rows (u32) and offsets (i64) through the op staging buffer
  int rc = kv_stage(ctx, n * 4 + (n + 1) * 8 + 16);
  if (rc) return rc;
  std::vector<u32> r32((size_t)n);
  for (int64_t i = 0; i < n; ++i) r32[i] = (u32)rows[i];
  i64* doff = (i64*)(ctx->kv_stage + (((size_t)n * 4 + 15) & ~(size_t)15));
  CK(cudaMemcpyAsync(ctx->kv_stage, r32.data(), (size_t)n * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(doff, off.data(), (size_t)(n + 1) * 8, cudaMemcpyHostToDevice, ctx->stream));
  rc = mars_kv_enqueue_gather_ids(k, ctx->stream, n, (const u32*)ctx->kv_stage, doff, ctx->kv_ids,
                                  ctx->num_sms * 4);
  if (rc) return fail(ctx, MARS_ERR_CUDA, "kv gather ids: %s", cudaGetErrorString((cudaError_t)rc));
  CK(cudaStreamSynchronize(ctx->stream));  // (the staging buffer is reused next)
  return MARS_OK;
}

int mars_kv_offload_rows(mars_ctx* ctx, int64_t n, const int64_t* rows, const int32_t* counts,
                         int64_t* slot0) {
  int rc = kv_tier_ready(ctx);
  if (rc) return rc;
  if (n < 0 || (n > 0 && (!rows || !counts))) return MARS_ERR_ARG;
  CK(cudaSetDevice(ctx->device));
  i64 tot = 0, s0 = -1;
  if (n > 0) {
    rc = kv_rows_ids(ctx, n, rows, counts, &tot);
    if (rc) return rc;
    if (tot > 0) {
      rc = kv_ring_put(ctx, ctx->kv_ids, tot, &s0);
      if (rc) return rc;
    }
  }
  CK(cudaStreamSynchronize(ctx->stream));
  KvScal s;
  CK(cudaMemcpy(&s, ctx->kv.s, sizeof s, cudaMemcpyDeviceToHost));
  if (s.status & 256) return fail(ctx, MARS_ERR_CONTRACT, "row table length != count");
  if (slot0) *slot0 = s0;
  return MARS_OK;
}

int mars_kv_restore_rows(mars_ctx* ctx, int64_t n, const int64_t* rows, const int32_t* counts,
                         const int64_t* slots) {
  int rc = kv_tier_ready(ctx);
  if (rc) return rc;
  if (n < 0 || (n > 0 && (!rows || !counts || !slots))) return MARS_ERR_ARG;
  CK(cudaSetDevice(ctx->device));
  i64 tot = 0;
  if (n > 0) {
    rc = kv_rows_ids(ctx, n, rows, counts, &tot);
    if (rc) return rc;
    i64 o = 0;
    for (int64_t i = 0; i < n; ++i) {  // every row from its own slots
      if (slots[i] < 0 || slots[i] + counts[i] > ctx->kv.host_blocks)
        return fail(ctx, MARS_ERR_ARG, "host slots");
      if (counts[i] > 0) {
        rc = kv_stage_copy(ctx, ctx->kv_ids + o, counts[i], slots[i], 1);
        if (rc) return rc;
      }
      o += counts[i];
    }
  }
  CK(cudaStreamSynchronize(ctx->stream));
  KvScal s;
  CK(cudaMemcpy(&s, ctx->kv.s, sizeof s, cudaMemcpyDeviceToHost));
  if (s.status & 256) return fail(ctx, MARS_ERR_CONTRACT, "row table length != count");
  return MARS_OK;
}

int mars_kv_evict(mars_ctx* ctx, int64_t n, const uint32_t* ids, int64_t slot0, int method) {
  return kv_move(ctx, n, ids, slot0, method, 0);
}

int mars_kv_restore(mars_ctx* ctx, int64_t n, const uint32_t* ids, int64_t slot0, int method) {
  return kv_move(ctx, n, ids, slot0, method, 1);
}

int mars_kv_host_ptr(mars_ctx* ctx, void** host, void** device) {
  if (!ctx) return MARS_ERR_ARG;
  if (host) *host = ctx->kv_host;
  if (device) *device = ctx->kv.data;
  return MARS_OK;
}

int mars_host_link_peak(mars_ctx* ctx, int64_t bytes, int reps, double* d2h, double* h2d,
                        double* bidir) {
  if (!ctx || bytes < 1 || reps < 1) return MARS_ERR_ARG;
  CK(cudaSetDevice(ctx->device));
  void *h0 = nullptr, *h1 = nullptr, *d0 = nullptr, *d1 = nullptr;
  cudaStream_t s2 = nullptr;
  cudaEvent_t e0, e1, e2;
  CK(cudaHostAlloc(&h0, bytes, cudaHostAllocDefault));
  CK(cudaHostAlloc(&h1, bytes, cudaHostAllocDefault));
  CK(cudaMalloc(&d0, bytes));
  CK(cudaMalloc(&d1, bytes));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventCreate(&e2));
  memset(h0, 1, bytes);
  memset(h1, 2, bytes);
  double best[3] = {0, 0, 0};
  for (int r = 0; r < reps; ++r) {
    for (int mode = 0; mode < 3; ++mode) {
      CK(cudaStreamSynchronize(ctx->stream));
      CK(cudaEventRecord(e0, ctx->stream));
      if (mode == 0 || mode == 2)
        CK(cudaMemcpyAsync(h0, d0, bytes, cudaMemcpyDeviceToHost, ctx->stream));
      if (mode == 1) CK(cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, ctx->stream));
      if (mode == 2) {
        CK(cudaStreamWaitEvent(s2, e0, 0));
        CK(cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, s2));
        CK(cudaEventRecord(e2, s2));
        CK(cudaStreamWaitEvent(ctx->stream, e2, 0));
      }
      CK(cudaEventRecord(e1, ctx->stream));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      double gbs = (mode == 2 ? 2.0 : 1.0) * (double)bytes / (ms * 1e-3) / 1e9;
      if (gbs > best[mode]) best[mode] = gbs;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  cudaStreamDestroy(s2);
  cudaFree(d0);
  cudaFree(d1);
  cudaFreeHost(h0);
  cudaFreeHost(h1);
  if (d2h) *d2h = best[0];
  if (h2d) *h2d = best[1];
  if (bidir) *bidir = best[2];
  return MARS_OK;
}

}  // extern "C"
