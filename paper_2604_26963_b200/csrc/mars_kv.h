// Device layout of the paged KV block manager (mars_kv.cu).
#pragma once

#include "mars_internal.cuh"

#define KV_CH 64  // block IDs per table chunk
#define KV_STAGE_BLOCKS 64  // blocks per staged host-tier DMA (128 MiB at 2 MiB/block)

struct KvScal {
  i64 seg_top;  // free-stack segments
  i64 arena_top;  // loose IDs in the arena (arena segments live below it)
  i64 fs_ids;   // IDs those segments hold (the explicit stack depth)
  i64 fresh;    // next never-used block ID (implicit stack bottom)
  i64 cfs_top;  // free table chunks
  i32 status;   // contract-break bits
};

struct Kv {
  i64 total;      // KvPool.total_blocks
  i32 D;          // chunk-directory entries per row
  i64 rows;
  i64 nchunks;
  u64* seg;       // free-stack segments, top = seg[seg_top-1]: chunk (chunk << 16 |
                  // start << 8 | count) or arena (1 << 63 | base << 16 | count)
  i64 seg_cap;
  u32* arena;     // [total] loose free IDs (arena segments, LIFO)
  u32* chunks;    // [nchunks][KV_CH] block IDs
  u32* cfs;       // free chunk stack
  u32* dir;       // [rows][D] chunk indices
  i32* len;       // [rows] table length
  KvScal* s;
  i64* xoff;      // [rows] scratch: per-table segment offsets (expiry / bulk runs)
  i64* xaoff;     // [rows] scratch: arena offsets
  i64* xroff;     // [rows] scratch: returned-chunk offsets
  i32* xlen;      // [rows] scratch: table lengths
  i64* xbase;     // [4] scratch: segment base, count, arena base, chunk-pool base
  // data plane
  u8* data;       // HBM pool: layer-major [layers][total][block_bytes/layers]
  u8* host;       // pinned host tier: [host_blocks][layers][piece]
  i64 block_bytes;
  i32 layers;
  i64 host_blocks;
};

int mars_kv_enqueue_apply(const Kv& k, cudaStream_t s, i64 n_ops, const u8* op, const u32* row,
                          const i32* n);
int mars_kv_enqueue_apply_step(const Kv& k, cudaStream_t s, Work* w, const Bufs& b);
// the step's expired pins' frees; offsets_done: k_scan laid out the offsets
int mars_kv_enqueue_exp_free(const Kv& k, cudaStream_t s, Work* w, const Bufs& b, int grid,
                             bool offsets_done);
int mars_kv_enqueue_bulk(const Kv& k, cudaStream_t s, i64 n, const u32* rows, const i32* cnt,
                         int grid);
int mars_kv_enqueue_resume_free(const Kv& k, cudaStream_t s, i64 n, const i64* rows,
                                const u8* kind);
int mars_kv_enqueue_table(const Kv& k, cudaStream_t s, u32 row, i64 cap, u32* out);
int mars_kv_enqueue_top(const Kv& k, cudaStream_t s, i64 cnt, u32* out);
int mars_kv_enqueue_copy(const Kv& k, cudaStream_t s, const u32* ids, i64 n, i64 slot0, int dir,
                         int grid);
int mars_kv_enqueue_stage(const Kv& k, cudaStream_t s, const u32* ids, i64 n, u8* stage, int dir,
                          int grid);
