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
  i32 pad_;
  i64 cap_n;    // IDs captured for the host tier since the last offload
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
  // host tier driven by the step's decisions: the IDs of the tables that
  // running-session evictions and unpinned tool boundaries free are captured
  // here (any order), to be copied to host memory after the step
  u32* cap;       // [total] or null (capture off)
};


// ---- free-stack segments and table frees (device helpers shared by the KV
// kernels and k_scan's fused expiry) ----------------------------------------
#define SEG_ARENA (1ull << 63)

__device__ __forceinline__ u64 seg_chunk_make(u32 ch, u32 start, u32 cnt) {
  return ((u64)ch << 16) | ((u64)start << 8) | (u64)cnt;
}
__device__ __forceinline__ u64 seg_arena_make(i64 base, u32 cnt) {
  return SEG_ARENA | ((u64)base << 16) | (u64)cnt;
}
__device__ __forceinline__ bool seg_is_arena(u64 s) { return (s & SEG_ARENA) != 0; }
__device__ __forceinline__ u64 seg_index(u64 s) { return (s >> 16) & 0xffffffffffull; }
__device__ __forceinline__ u32 seg_start(u64 s) { return (u32)(s >> 8) & 0xffu; }
__device__ __forceinline__ u32 seg_count(u64 s) { return (u32)s & 0xffu; }

// Pieces of freeing table positions [keep, L) (bottom -> top of the pushes):
// the tail T = [tb, L) of a partial last chunk (to the arena, its chunk back
// to the pool), the whole chunks between (chunk segments), the head
// H = [keep, hb) of a kept boundary chunk (to the arena).
struct FreePlan {
  i64 keep, L, hb, tb, f0, f1;  // full chunks [f0, f1)
  i64 nh, nt;                   // |H|, |T|
  bool tail_chunk;              // T's chunk returns to the pool
};

__device__ __forceinline__ FreePlan free_plan(i64 L, i64 keep) {
  FreePlan f;
  f.keep = keep;
  f.L = L;
  const i64 up = (keep + KV_CH - 1) / KV_CH * KV_CH;  // keep rounded up
  const i64 dn = L / KV_CH * KV_CH;                   // L rounded down
  if (up >= L) {  // one chunk, or nothing: all of it to the arena
    f.hb = L;
    f.tb = L;
    f.nh = L - keep;
    f.nt = 0;
    f.f0 = f.f1 = 0;
    f.tail_chunk = (keep % KV_CH) == 0 && L > keep;  // the chunk leaves the row
  } else {
    f.hb = up;
    f.nh = up - keep;
    f.tb = dn > up ? dn : up;
    f.nt = L - f.tb;
    f.f0 = up / KV_CH;
    f.f1 = f.tb / KV_CH;
    f.tail_chunk = f.nt > 0;
  }
  return f;
}

// Freeing table positions [keep, L) of `row` (FreePlan f), on one warp: the
// segments go to seg[sp..] bottom -> top (T's arena segment, the whole chunks
// from the last one down, H's arena segment), the loose IDs of T and H to the
// arena at ap.. (each segment pops from its end), T's chunk back to the pool
// at cfs[cf] (cf < 0: none); the lanes copy IDs / write segments in parallel.
// (W lanes per free: a warp, or a half warp for the many small expired tables)
template <int W = 32>
__device__ __forceinline__ void kv_free_warp(const Kv& k, u32 row, const FreePlan& f, i64 sp,
                                             i64 ap, i64 cf, int lane, bool cap = false) {
  const u32* dr = k.dir + (i64)row * k.D;
  if (cap && k.cap != nullptr && f.L > f.keep) {
    // the freed IDs (table positions [keep, L)) to the capture list first
    const i64 n = f.L - f.keep;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd((unsigned long long*)&k.s->cap_n, (unsigned long long)n);
    base = __shfl_sync(0xffffffffu, base, 0, W);
    if ((i64)base + n > k.total) {
      if (lane == 0) atomicOr(&k.s->status, 128);
    } else {
      for (i64 j = lane; j < n; j += W) {
        const i64 p = f.keep + j;
        k.cap[base + j] = k.chunks[(i64)dr[p / KV_CH] * KV_CH + p % KV_CH];
      }
    }
  }
  if (f.nt > 0) {
    for (i64 j = lane; j < f.nt; j += W) {
      const i64 p = f.tb + j;
      k.arena[ap + f.nt - 1 - j] = k.chunks[(i64)dr[p / KV_CH] * KV_CH + p % KV_CH];
    }
    if (lane == 0) k.seg[sp] = seg_arena_make(ap, (u32)f.nt);
    ++sp;
    ap += f.nt;
  }
  const i64 nf = f.f1 - f.f0;
  for (i64 j = lane; j < nf; j += W) k.seg[sp + j] = seg_chunk_make(dr[f.f1 - 1 - j], 0, KV_CH);
  sp += nf;
  if (f.nh > 0) {
    for (i64 j = lane; j < f.nh; j += W) {
      const i64 p = f.keep + j;
      k.arena[ap + f.nh - 1 - j] = k.chunks[(i64)dr[p / KV_CH] * KV_CH + p % KV_CH];
    }
    if (lane == 0) k.seg[sp] = seg_arena_make(ap, (u32)f.nh);
  }
  if (lane == 0) {
    if (cf >= 0) k.cfs[cf] = dr[(f.L - 1) / KV_CH];
    k.len[row] = (i32)f.keep;
  }
}

// a whole table of L IDs (an expired pin's): T = its partial last chunk, then
// its full chunks from the last one down
template <int W = 32>
__device__ __forceinline__ void kv_free_table_warp(const Kv& k, u32 row, i64 L, i64 sp, i64 ap,
                                                   i64 cf, int lane) {
  const i64 tail = L % KV_CH, full = L / KV_CH;
  FreePlan f;
  f.keep = 0;
  f.L = L;
  f.nh = 0;
  f.f0 = 0;
  f.f1 = full;
  f.tb = full * KV_CH;
  f.nt = tail;
  f.hb = 0;
  f.tail_chunk = tail > 0;
  kv_free_warp<W>(k, row, f, sp, ap, tail > 0 ? cf : -1, lane);
}

int mars_kv_preload();
#ifdef MARS_PHASE_TIMING
void mars_kv_ptime_dump(cudaStream_t s);  // first start / last end of the S5 kernels
#endif
int mars_kv_enqueue_apply(const Kv& k, cudaStream_t s, i64 n_ops, const u8* op, const u32* row,
                          const i32* n);
// the step's journal (parts & 1) and the tick tail's frees (parts & 2)
int mars_kv_enqueue_apply_step(const Kv& k, cudaStream_t s, Work* w, const Bufs& b, int parts);
// the step's expired pins' frees; offsets_done: k_scan laid out the offsets;
// pdl: the push is a programmatic dependent of the kernel before it (k_scan)
int mars_kv_enqueue_exp_free(const Kv& k, cudaStream_t s, Work* w, const Bufs& b, int grid,
                             bool offsets_done, bool pdl);
int mars_kv_enqueue_bulk(const Kv& k, cudaStream_t s, i64 n, const u32* rows, const i32* cnt,
                         int grid);
int mars_kv_enqueue_resume_free(const Kv& k, cudaStream_t s, i64 n, const i64* rows,
                                const u8* kind);
int mars_kv_enqueue_table(const Kv& k, cudaStream_t s, u32 row, i64 cap, u32* out);
int mars_kv_enqueue_gather_ids(const Kv& k, cudaStream_t s, i64 n, const u32* rows, const i64* off,
                               u32* out, int grid);
int mars_kv_enqueue_top(const Kv& k, cudaStream_t s, i64 cnt, u32* out);
int mars_kv_enqueue_copy(const Kv& k, cudaStream_t s, const u32* ids, i64 n, i64 slot0, int dir,
                         int grid);
int mars_kv_enqueue_stage(const Kv& k, cudaStream_t s, const u32* ids, i64 n, u8* stage, int dir,
                          int grid);
