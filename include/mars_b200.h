/*
 * mars_b200.h -- C ABI of the B200-native MARS scheduling step.
 *
 * The reference (arXiv 2604.26963, /root/reference/pkg/src/agentsched) has no
 * FFI: its pluggable boundary is the Python PolicyBase object
 * (baselines.py:56-101) plus the module-level balance_and_admit
 * (control.py:166-208).  These entry points are what a ctypes/cffi binding of
 * that boundary needs; every one names the reference interface it replaces.
 * The Python mirror of the plugin API (paper_2604_26963_b200/policy.py,
 * admission.py) sits on top of exactly this surface.
 *
 * Conventions
 *   - plain pointers and sizes, no framework types; every function returns
 *     MARS_OK (0) or an error category (mars_last_error() has the text).
 *     MARS_ERR_CONTRACT maps to agentsched ContractViolation (engine.py:30),
 *     everything else to RuntimeError.
 *   - one host thread per context; all device work is ordered on the
 *     context's stream (mars_set_stream), calls marked "sync" return after the
 *     stream drained.
 *   - row = slot index in the device session table, 0 <= row < max_rows.
 *     rank = dense lexicographic rank of the session-id string (the
 *     reference's final tie-break, baselines.py:374-377).
 */
#ifndef MARS_B200_H
#define MARS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MARS_OK 0
#define MARS_ERR_CONTRACT 1
#define MARS_ERR_CUDA 2
#define MARS_ERR_CAPACITY 3
#define MARS_ERR_ARG 4

#define MARS_ABI_VERSION 7

/* phase codes: agentsched/engine.py:250-256 */
#define MARS_WAITING_ADMISSION 0
#define MARS_PREFILL 1
#define MARS_DECODE 2
#define MARS_TOOL 3
#define MARS_WAITING_RESUME 4
#define MARS_DONE 5
#define MARS_EMPTY 7

/* row flag bits */
#define MARS_F_ACTIVE 1u   /* admitted, not finished (sim.py:133 `active`) */
#define MARS_F_QUEUED 2u   /* in the admission queue (sim.py:132) */
#define MARS_F_PINNED 4u   /* in the pin registry (baselines.py:349) */
#define MARS_F_BOUNDARY 8u /* S2 retention requested this step */
#define MARS_F_LONG 16u    /* QueueEntry.is_long_session (control.py:91) */

/* journal op codes (KvPool observer ops, engine.py:129-143 + evict) */
#define MARS_J_ALLOC 1
#define MARS_J_EVICT_RUNNING 2
#define MARS_J_EVICT_PINNED 3
#define MARS_J_EXPIRE 4

typedef struct mars_ctx mars_ctx;

/* All constants of GpuModel, MlfqConfig, RetentionConfig, PressureConfig,
 * ControllerConfig and the MarsPolicy ablation switches.  Infinite level
 * boundaries / quotas are INT64_MAX.  mars_config_default() fills the
 * reference defaults (engine.py:24-27, scheduler.py:34-41,
 * telemetry.py:14-19, control.py:20-27). */
typedef struct mars_config {
  int32_t block_size;          /* engine.py:26 */
  int32_t token_budget;        /* engine.py:24 */
  double tick_duration_s;      /* engine.py:25 */
  int32_t num_levels;          /* scheduler.py:34 (<= 4) */
  int32_t max_promotions;      /* scheduler.py:50 */
  int32_t max_decode_slots;    /* scheduler.py:38 */
  int32_t window_size;         /* scheduler.py:61-63 (<= 128) */
  int64_t level_bounds[4];     /* scheduler.py:35 */
  int64_t level_quotas[4];     /* scheduler.py:36 */
  double promotion_wait_s;     /* scheduler.py:37 */
  double deadline_slack;       /* scheduler.py:39 */
  double max_pin_horizon_s;    /* scheduler.py:40 */
  double pressure_weight_clip; /* scheduler.py:41 */
  double cpu_high_fraction, cpu_low_fraction;   /* telemetry.py:16-17 */
  double kv_high_watermark, kv_low_watermark;   /* telemetry.py:18-19 */
  int32_t hysteresis_window;                    /* telemetry.py:15 */
  double ema_smoothing;                         /* telemetry.py:14 */
  double initial_tool_estimate_s;               /* telemetry.py:56 */
  int32_t w_min;                                /* control.py:20 */
  double aimd_increase, aimd_decrease;          /* control.py:21-22 */
  double control_interval_s;                    /* control.py:23 */
  double initial_window;                        /* control.py:24 */
  double cpu_oversubscription;                  /* control.py:25 */
  double reserve_fraction;                      /* control.py:26 */
  double long_session_fraction;                 /* control.py:27 */
  int32_t enable_coordinator;                   /* baselines.py:339 */
  int32_t enable_coscheduler;                   /* baselines.py:340 */
  /* which policy the step runs (POLICY_KINDS, baselines.py:48): MARS, or one
   * of the comparison policies on the same build_plan walk
   * (baselines.py:108-315).  The comparison policies order the window by
   * arrival (fcfs, ttl) or by (served_tokens, arrival) (program_priority,
   * the `served` column then holding Call.served_tokens), never age, fit
   * whole chunks, and fcfs/ttl block at the head of line. */
  int32_t policy;                               /* MARS_POLICY_* */
  double ttl_seconds;                           /* static_ttl deadline, baselines.py:50 */
  double ttl_multiplier;                        /* dynamic_ttl x EMA tool time, :51 */
} mars_config;

#define MARS_POLICY_MARS 0
#define MARS_POLICY_FCFS 1
#define MARS_POLICY_PROGRAM_PRIORITY 2
#define MARS_POLICY_STATIC_TTL 3
#define MARS_POLICY_DYNAMIC_TTL 4

/* Structure-of-arrays column pointers (host side).  NULL = column not
 * transferred.  Widths are the minimal exact widths of the reference values
 * (SURVEY.md §8 canonical SoA). */
typedef struct mars_cols {
  uint8_t *phase, *flags, *level, *promos, *plevel;
  double *ready_since, *wait_since, *deadline, *arrival;
  int32_t *context, *kv, *rem_decode, *pinned_blocks, *req_blocks, *r0_prefill, *r0_decode,
      *preempt;
  int64_t *served;
  uint32_t *rank;
  int32_t *rounds_left;  /* rounds after the current one (Call.is_last_round, engine.py:302-304) */
} mars_cols;

/* Device-resident scalar state: KvPool counters, the Telemetry value
 * (telemetry.py:66-96) and ControllerState (control.py:52-61). */
typedef struct mars_scalars {
  int64_t total_blocks, free_blocks;
  double w_adm, last_update;
  int32_t cpu_overloaded, kv_overloaded;
  int32_t cpu_high_streak, cpu_low_streak, kv_high_streak, kv_low_streak;
  int32_t has_ema_tool, has_ema_blocks, has_blocks_seed;
  double ema_tool, ema_blocks, blocks_seed;
  double last_w_adm, last_window_update;
  int32_t has_last_w_adm;
  int64_t available_kv;
  double kv_usage_ratio;
  int64_t active_sessions;
  int32_t active_tools, queued_tools;
  int64_t queue_len;
} mars_scalars;

/* mars_step_in.mode bits.  0 = the device-resident engine step.  The
 * reference-plugin drop-in (policy.py / admission.py) lets the reference's
 * own tick loop do what it does itself and asks the device only for the rest. */
#define MARS_MODE_SKIP_EXPIRY 1       /* the caller evicts expired pins (sim.py:324-325) */
#define MARS_MODE_SKIP_PROBE 2        /* telemetry scalars come from mars_set_scalars */
#define MARS_MODE_SKIP_REFRESH 4      /* refresh_pressure already ran (sim.py:330) */
#define MARS_MODE_NO_ROWS 8           /* admission only: queue entries have no table rows */
#define MARS_MODE_SERVICE 16          /* charge_service at tick end for planned rows
                                         (baselines.py:362-367, sim.py:364) */
#define MARS_MODE_FINISH_RETENTION 32 /* decide_retention for decodes finishing their round
                                         this tick, on post-tick values (sim.py:250) */
#define MARS_MODE_RANK_ORDERED 64     /* caller asserts rank[row] == row order (row order is
                                         session-id order): expired pins need no sort */
#define MARS_MODE_SHARDED 128         /* this context is one replica of a sharded engine:
                                         the control plane runs on all-reduced counters and
                                         the all-gathered admission list (mars_step_phase) */
#define MARS_MODE_ADVANCE 256         /* the tick's tail on the device after the plan:
                                         step_gpu (engine.py:459-514) on the planned rows,
                                         then each ending round in decode order
                                         (sim.py:233-279: note_round_blocks, DONE + free on
                                         the last round, else the retention decision's pin
                                         or free, phase TOOL).  Implies SERVICE. */

typedef struct mars_step_in {
  double now;
  int32_t control_due;     /* sim.py:329: run refresh_pressure + balance_and_admit */
  int32_t active_tools;    /* ToolPlane.active_count() at the probe (sim.py:327) */
  int32_t queued_tools;    /* ToolPlane.queued_count() */
  int32_t worker_slots;    /* ToolPlane.worker_slots */
  int32_t mode;            /* MARS_MODE_* bits */
} mars_step_in;

/* Step result.  Pointers refer to pinned host buffers owned by the context,
 * valid until the next call on it. */
typedef struct mars_step_out {
  int32_t status;          /* 0 ok */
  int32_t n_expired, n_admitted, n_window, n_decode, n_prefill, n_evict, n_journal, n_retention;
  int32_t n_ready, n_promoted, pack_mode;
  int64_t total_tokens;
  int64_t free_after_expiry, free_blocks;
  int64_t limit, slots;
  const uint32_t *expired_rows; const int32_t *expired_blocks;   /* rank order */
  const uint32_t *admitted_rows;                                 /* packed order */
  const uint32_t *window_rows;                                   /* priority order */
  const uint32_t *decode_rows;
  const uint32_t *prefill_rows; const int32_t *prefill_grants;
  const uint32_t *evict_rows; const uint8_t *evict_kind; const int32_t *evict_blocks;
  const uint8_t *journal_op; const uint32_t *journal_row; const int32_t *journal_n;
  const uint32_t *ret_rows; const uint8_t *ret_pin;
  const double *ret_benefit, *ret_cost, *ret_deadline;
  /* MARS_MODE_SERVICE: MLFQ level of each planned row after its charge */
  const uint8_t *decode_level, *prefill_level;
  /* MARS_MODE_FINISH_RETENTION: decode rows with remaining_decode == 1 */
  int32_t n_finish;
  const uint32_t *fin_rows; const uint8_t *fin_pin;
  const double *fin_benefit, *fin_cost, *fin_deadline;
  /* diagnostics: candidate counts at the exact thresholds, 1 if the walk
   * left the prefix-sum fast path; how pack_queue sorted the list (0 not
   * run, 1 grid LSD radix sort, 2 one CTA: small list or first fit) */
  int32_t n_window_cand, n_victim_cand, walk_slow, sort_path;
  /* MARS_MODE_ADVANCE: rounds that ended this tick, sessions that finished;
   * per ended round in decode order: its row and what the boundary did
   * (0 session done, 1 KV pinned -> tool, 2 KV freed -> tool) */
  int32_t n_round_end, n_done;
  const uint32_t* end_rows;
  const uint8_t* end_kind;
  /* ... and the payloads the reference logs for it (sim.py:233-279): the
   * blocks pinned or freed, the retention decision (when the policy makes
   * one: pin, benefit_s, cost_s, deadline); per planned prefill, 1 if its
   * grant finished the prefill (engine.py:489-497, gpu_1st_token) (ABI v4) */
  const int32_t* end_blocks;
  const uint8_t* end_pin;
  const double *end_benefit, *end_cost, *end_deadline;
  const uint8_t* prefill_done;
  /* diagnostics (ABI v5): exact full-table reclaimer passes the walk took (0
   * whenever the victim stream covered the step's claims), which candidate
   * lists k_scan's grid radix refinement cut (bit 0 window, bit 1 victims),
   * its rounds, and the refined lists' lengths */
  int32_t n_fullscan, ref_flags, ref_rounds, n_window_ref, n_victim_ref;
  /* MARS_MODE_SERVICE (ABI v6): per planned row (decodes, then prefills) its
   * MLFQ state before the tick-end charge, (served_tokens_at_level << 8) |
   * level, so a host that charges a different amount can undo the prediction */
  const int64_t* plan_pre_charge;
} mars_step_out;

/* ---- lifecycle ------------------------------------------------------- */
int mars_abi_version(void);
void mars_config_default(mars_config* cfg);
int mars_create(const mars_config* cfg, int device, int64_t max_rows, int64_t max_queue,
                mars_ctx** out);
int mars_destroy(mars_ctx* ctx);
const char* mars_last_error(mars_ctx* ctx);
int mars_set_stream(mars_ctx* ctx, void* cuda_stream);

/* ---- session-state store (replaces Call/PriorityState/PinnedSession/QueueEntry
 *      objects: engine.py:259-319, scheduler.py:78-84,165-172, control.py:64-73) */
int mars_set_rows(mars_ctx* ctx, int64_t n_rows);                 /* live row count */
int mars_upsert_rows(mars_ctx* ctx, int64_t n, const int64_t* rows, const mars_cols* cols);
int mars_read_rows(mars_ctx* ctx, int64_t n, const int64_t* rows, mars_cols* out);   /* sync */
/* Zero-copy input staging for whole-table uploads: a pinned host arena laid
 * out like the device table (one slab, columns grouped by element size).
 * *base / *bytes describe it; cols (optional) receives each column's host
 * address (max_rows rows).  Allocated on the first call, owned by the context. */
int mars_input_arena(mars_ctx* ctx, void** base, int64_t* bytes, mars_cols* cols);
/* rows [0, n) of the columns in `mask` (bit i = the i-th mars_cols field)
 * from the input arena to the table: n == max_rows and slab-contiguous
 * columns (a default step's 17 are) -> ONE linear copy; else one pitched
 * copy per run of adjacent columns of one element size; sync (the arena may
 * be rewritten after the return) */
int mars_upsert_arena(mars_ctx* ctx, int64_t n, uint64_t mask);
/* admission list (sim.py:132 admission_queue; control.py:190 persistent order) */
int mars_set_queue(mars_ctx* ctx, int64_t n, const uint32_t* rows, const int32_t* req_blocks,
                   const uint8_t* is_long);
int mars_get_queue(mars_ctx* ctx, int64_t cap, uint32_t* rows, int64_t* n);          /* sync */
/* arrivals appended to the end of the device admission list (sim.py:289-301
 * + control.py:76-93 make_queue_entry), without a host round trip of the list */
int mars_queue_append(mars_ctx* ctx, int64_t n, const uint32_t* rows, const int32_t* req,
                      const uint8_t* lng);
/* The drop-in's per-session MLFQ hooks, batched (rows distinct): on_admit
 * (baselines.py:351-360, initial_level scheduler.py:87-97 of the first
 * round's new prefill) and on_service (baselines.py:362-367, charge_service
 * scheduler.py:100-108) from the device state, or -- pre_charge non-null --
 * from the given (served << 8) | level (undoing a predicted charge).
 * MARS_ERR_CONTRACT for a prefill < 1 or negative tokens. */
int mars_on_admit(mars_ctx* ctx, int64_t n, const int64_t* rows, const int32_t* r0_prefill,
                  const double* now);
/* MarsPolicy.expired_pins (baselines.py:396-399): the pinned rows whose
 * deadline is before now, in no particular order (*n = how many) */
int mars_expired_pins(mars_ctx* ctx, double now, int64_t cap, uint32_t* rows, int64_t* n);
int mars_on_service(mars_ctx* ctx, int64_t n, const int64_t* rows, const int64_t* tokens,
                    const double* now, const int64_t* pre_charge);
int mars_set_scalars(mars_ctx* ctx, const mars_scalars* s);
int mars_get_scalars(mars_ctx* ctx, mars_scalars* s);                               /* sync */

/* ---- the step (S1-S5): replaces one tick's sim.py:324-342 scheduling half:
 *      MarsPolicy.expired_pins + evictions, Telemetry.probe, refresh_pressure,
 *      balance_and_admit + admit, decide_retention for BOUNDARY rows,
 *      MarsPolicy.plan_tick (promote_waiting + build_plan + reclaim). */
int mars_step(mars_ctx* ctx, const mars_step_in* in, mars_step_out* out);          /* sync */
int mars_step_enqueue(mars_ctx* ctx, const mars_step_in* in);   /* async, device-resident */
int mars_step_fetch(mars_ctx* ctx, mars_step_out* out);          /* sync, after enqueue */
/* the pinned host arena every mars_step_out array points into (valid for the
 * context's lifetime; contents valid until the next fetch) */
int mars_output_arena(mars_ctx* ctx, void** base, int64_t* bytes);
/* capture the whole step (both streams) as one CUDA graph; re-captured only
 * when the launch shape (rows, queue bucket, mode) changes */
int mars_set_graph(mars_ctx* ctx, int on);
/* replace the context's configuration (same policy): the reference builds its
 * engine parameters per run (sim.py:90-110, GpuModel token_budget_per_tick /
 * tick_duration_s, engine.py:24-29); drops the captured step graphs */
int mars_set_config(mars_ctx* ctx, const mars_config* cfg);

/* decide_retention (scheduler.py:190-213) for explicit inputs; elementwise f64
 * on the device, bit-exact (no FMA contraction). */
/* resume_from_tool (sim.py:190-231) for sessions whose tools finished, in
 * the tool plane's finish order: the tool-duration EMA fold (tool_end,
 * telemetry.py:96-120), round_index + 1, warm resume (the pin still covers
 * the finish time: unpin, KV kept) or cold (an expired pin is evicted),
 * submit_round with the next round's new prefill / decode lengths, and
 * on_resume.  Synchronous; counts out (warm, cold, pins evicted). */
int mars_resume(mars_ctx* ctx, int64_t n, const int64_t* rows, const double* finish_time,
                const double* duration, const int32_t* new_prefill, const int32_t* decode_tokens,
                double now, int32_t* counts /* [3] */);
/* per row of the last mars_resume, in its order (sync; ABI v4): kind 0 warm
 * (unpinned), 1 cold, 2 cold after the return-time release of an expired pin
 * (sim.py:193-205); blocks unpinned or released; and gpu_submit's payload
 * (sim.py:224-230): context_tokens, required_prefill, projected_blocks */
int mars_resume_rows(mars_ctx* ctx, int64_t n, uint8_t* kind, int32_t* blocks, int32_t* context,
                     int32_t* need, int32_t* projected);
int mars_retention_batch(mars_ctx* ctx, int64_t n, const int32_t* context, const int32_t* kv,
                         int64_t total_blocks, double kv_usage_ratio, double ema_tool,
                         double now, uint8_t* pin, double* benefit, double* cost,
                         double* deadline);                                         /* sync */

/* ---- checkpoint / resume of the whole device state (for replay and bench) */
int mars_checkpoint(mars_ctx* ctx);
int mars_restore(mars_ctx* ctx);
/* write `bytes` of scratch to evict L2 between timed steps */
int mars_flush_l2(mars_ctx* ctx, int64_t bytes);

/* ---- S5: paged KV block manager + HBM <-> pinned-host tier ----------------
 * Block IDs follow the LIFO policy written down in oracle/block_ids.py (the
 * reference KvPool counts only: engine.py:116-221).  Once enabled, every
 * mars_step also applies its own journal (expired pins in rank order, then
 * the plan's alloc/evict ops) to the block tables; mars_kv_apply replays any
 * other pool op stream (the KvPool.observer callbacks, engine.py:129-143). */
#define MARS_KV_ALLOC 1     /* pop n IDs onto the row's table */
#define MARS_KV_FREE 2      /* push the last n IDs back (n = -1: the whole table) */
#define MARS_KV_PIN 3       /* ownership only (no table change) */
#define MARS_KV_UNPIN 4

typedef struct mars_kv_config {
  int64_t total_blocks;        /* KvPool.total_blocks */
  int32_t max_blocks_per_row;  /* table capacity per session */
  int64_t block_bytes;         /* KV bytes per block (0 = block IDs only, no data) */
  int32_t layers;              /* >1: layer-major device layout, `layers` pieces per block */
  int64_t host_blocks;         /* pinned host-tier capacity in blocks */
} mars_kv_config;

int mars_kv_init(mars_ctx* ctx, const mars_kv_config* cfg);
int mars_kv_apply(mars_ctx* ctx, int64_t n_ops, const uint8_t* op, const uint32_t* row,
                  const int32_t* n);                                              /* sync */
/* initial tables from a fresh pool (no free segment yet): row[i] (distinct)
 * gets the next cnt[i] never-used IDs, as cnt[i] sequential allocs in list
 * order would (the bench's 1M-session tables) */
int mars_kv_bulk_alloc(mars_ctx* ctx, int64_t n, const uint32_t* row, const int32_t* cnt); /* sync */
int mars_kv_table(mars_ctx* ctx, uint32_t row, int64_t cap, uint32_t* ids, int64_t* n); /* sync */
/* next `k` IDs the stack would pop (UINT32_MAX past the last free block),
 * plus its depth (IDs on the explicit stack, next fresh ID) */
int mars_kv_state(mars_ctx* ctx, int64_t k, uint32_t* top_ids, int64_t* explicit_depth,
                  int64_t* fresh, int32_t* status);                               /* sync */
/* evict (HBM -> host slots [slot0, slot0+n)) / restore (host -> HBM) block data.
 * method 0: copy engines (one cudaMemcpyAsync per block piece),
 * method 1: SM-driven zero-copy kernel over mapped pinned memory,
 * method 2: staged -- HBM gather/scatter kernel + one large DMA per 64 blocks. */
int mars_kv_evict(mars_ctx* ctx, int64_t n, const uint32_t* block_ids, int64_t slot0, int method);
int mars_kv_restore(mars_ctx* ctx, int64_t n, const uint32_t* block_ids, int64_t slot0,
                    int method);
int mars_kv_host_ptr(mars_ctx* ctx, void** host, void** device);

/* The host tier driven by the step's decisions (no host tier in the
 * reference; decision-neutral: the pool counts stay the
 * reference's).  With capture on, every step records the IDs of the tables
 * that a running session's eviction (scheduler.py:228-267 via sim.py:168-188)
 * or an unpinned tool boundary (sim.py:266-272) frees; offload_captured copies
 * those blocks to the next slots of the pinned host ring (returns the count,
 * the first slot, and optionally the IDs in slot order).  offload_rows copies
 * whole tables of rows (a pin at a tool boundary, sim.py:261-265) to the ring
 * (row i at slot0 + counts[0..i)); restore_rows copies them back into the
 * rows' current tables (a warm resume, sim.py:193-200).  counts[i] must be
 * row i's table length. */
int mars_kv_capture(mars_ctx* ctx, int on);
int mars_kv_offload_captured(mars_ctx* ctx, int64_t* n_blocks, int64_t* slot0, uint32_t* ids,
                             int64_t ids_cap);
int mars_kv_offload_rows(mars_ctx* ctx, int64_t n, const int64_t* rows, const int32_t* counts,
                         int64_t* slot0);
int mars_kv_restore_rows(mars_ctx* ctx, int64_t n, const int64_t* rows, const int32_t* counts,
                         const int64_t* slots);
/* pinned cudaMemcpyAsync peak of the host link: best of `reps` per direction */
int mars_host_link_peak(mars_ctx* ctx, int64_t bytes, int reps, double* d2h_gbs, double* h2d_gbs,
                        double* bidir_gbs);

/* ---- sharded engine: one context per GPU, sessions partitioned across
 * replicas; S1/S2/S4/S5 replica-local, the control plane global.
 * A step is mars_step_phase(1) -> all-reduce(sum) of the XC_N int64 counters
 * at `xc` -> all-gather of `send_words` uint64 from `xsend` into `xrecv`
 * (rank-major; word 0 the entry count, then one gpos<<32 | req<<1 | long
 * word per local admission entry) -> mars_step_phase(2) -> mars_step_fetch.
 * The collectives are the caller's (NCCL through torch.distributed), on the
 * same stream. */
int mars_shard_init(mars_ctx* ctx, int world, int rank);
int mars_shard_buffers(mars_ctx* ctx, void** xc, void** xsend, void** xrecv, int64_t* send_words);
/* global list positions of the local admission entries (dense over the union) */
int mars_set_queue_gpos(mars_ctx* ctx, int64_t n, const uint32_t* gpos);
int mars_get_queue_gpos(mars_ctx* ctx, int64_t cap, uint32_t* gpos, int64_t* n);  /* sync */
int mars_step_phase(mars_ctx* ctx, const mars_step_in* in, int phase);

/* drain the context's stream and report any pending CUDA error */
int mars_sync(mars_ctx* ctx);

/* number of kernel launches issued by the last step (incl. early-exit ones) */
int mars_last_launch_count(mars_ctx* ctx);

/* per-kernel device times of the last step, recorded with CUDA events on the
 * stream each kernel runs on: [scan, expired-sort, control, walk] in ms
 * (-1 = not launched).  Profiling must be enabled before the step. */
#define MARS_NUM_KTIMES 7  /* k_scan, expired sort, k_control, k_walk, k_pack,
                              S5 expired-pin frees (k_kv_exp_*), S5 journal (k_kv_apply_step) */
int mars_set_profiling(mars_ctx* ctx, int on);
int mars_kernel_times(mars_ctx* ctx, float* ms, int n);   /* sync */

#ifdef __cplusplus
}
#endif
#endif /* MARS_B200_H */
