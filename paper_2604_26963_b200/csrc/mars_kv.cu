// Paged KV block manager (S5) and the HBM <-> pinned-host KV tier.
//
// Block IDs follow the written-down policy of oracle/block_ids.py (the
// reference KvPool only counts, engine.py:116-221): a LIFO free stack whose
// pops first yield 0,1,2,..., alloc appends pops to the session's table,
// free pushes the table tail back in reverse.  The stack is an explicit
// array on top of an implicit "fresh" range, and tables are chunked (64 IDs
// per chunk, per-row chunk directory), so the pool can hold millions of
// blocks without materialising them up front.
//
// Ops of one journal are applied in order by one CTA; every op is parallel
// over its IDs (coalesced pushes/pops).
#include <cuda_runtime.h>

#include "mars_internal.cuh"
#include "mars_kv.h"

#define KV_TPB 1024

__device__ __forceinline__ u32 kv_slot(const Kv& k, u32 row, i64 pos) {
  u32 ch = k.dir[(i64)row * k.D + pos / KV_CH];
  return k.chunks[(i64)ch * KV_CH + pos % KV_CH];
}

// one pool op, executed by the whole CTA.  op: MARS_KV_ALLOC / MARS_KV_FREE
// (n = -1: the whole table).  Returns false on a contract break.
__device__ bool kv_op(Kv& k, int op, u32 row, i64 n) {
  __shared__ i64 s_top, s_fresh, s_ctop, s_len;
  if (threadIdx.x == 0) {
    s_top = k.s->fs_top;
    s_fresh = k.s->fresh;
    s_ctop = k.s->cfs_top;
    s_len = k.len[row];
  }
  __syncthreads();
  const i64 top = s_top, fresh = s_fresh, ctop = s_ctop, len = s_len;
  if (op == MARS_KV_ALLOC) {
    if (n <= 0) return true;
    if (len + n > (i64)k.D * KV_CH || n > top + (k.total - fresh)) {
      if (threadIdx.x == 0) k.s->status |= 1;
      __syncthreads();
      return false;
    }
    const i64 c0 = (len + KV_CH - 1) / KV_CH, c1 = (len + n + KV_CH - 1) / KV_CH;
    const i64 nc = c1 - c0;
    if (nc > ctop) {
      if (threadIdx.x == 0) k.s->status |= 2;
      __syncthreads();
      return false;
    }
    for (i64 j = threadIdx.x; j < nc; j += blockDim.x)
      k.dir[(i64)row * k.D + c0 + j] = k.cfs[ctop - 1 - j];
    __syncthreads();
    for (i64 q = threadIdx.x; q < n; q += blockDim.x) {
      u32 id = (q < top) ? k.fs[top - 1 - q] : (u32)(fresh + (q - top));
      i64 p = len + q;
      u32 ch = k.dir[(i64)row * k.D + p / KV_CH];
      k.chunks[(i64)ch * KV_CH + p % KV_CH] = id;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      i64 from_stack = n < top ? n : top;
      k.s->fs_top = top - from_stack;
      k.s->fresh = fresh + (n - from_stack);
      k.s->cfs_top = ctop - nc;
      k.len[row] = (i32)(len + n);
    }
    __syncthreads();
    return true;
  }
  // free: the last n IDs, pushed in reverse table order
  if (n < 0) n = len;
  if (n > len) {
    if (threadIdx.x == 0) k.s->status |= 4;
    __syncthreads();
    return false;
  }
  if (n == 0) return true;
  for (i64 q = threadIdx.x; q < n; q += blockDim.x) k.fs[top + q] = kv_slot(k, row, len - 1 - q);
  const i64 c_keep = (len - n + KV_CH - 1) / KV_CH, c_all = (len + KV_CH - 1) / KV_CH;
  __syncthreads();
  for (i64 j = threadIdx.x; j < c_all - c_keep; j += blockDim.x)
    k.cfs[ctop + j] = k.dir[(i64)row * k.D + c_all - 1 - j];
  __syncthreads();
  if (threadIdx.x == 0) {
    k.s->fs_top = top + n;
    k.s->cfs_top = ctop + (c_all - c_keep);
    k.len[row] = (i32)(len - n);
  }
  __syncthreads();
  return true;
}

// host journal: ordered (op, row, n)
__global__ void __launch_bounds__(KV_TPB) k_kv_apply(Kv k, i64 n_ops, const u8* op, const u32* row,
                                                     const i32* n) {
  for (i64 i = 0; i < n_ops; ++i) {
    int o = op[i];
    if (o == MARS_KV_ALLOC || o == MARS_KV_FREE) {
      if (!kv_op(k, o, row[i], o == MARS_KV_FREE && n[i] < 0 ? -1 : n[i])) return;
    }
  }
}

// the step's own journal: expired pins (rank order) then k_walk's journal,
// then (MARS_MODE_ADVANCE) the tick tail's frees in decode order -- a finished
// session's blocks (sim.py:243) and an unpinned boundary's (sim.py:269); a
// pin keeps the table (ownership moves, the IDs stay)
__global__ void __launch_bounds__(KV_TPB) k_kv_apply_step(Kv k, Work* w, Bufs b) {
  const int ne = w->n_exp;
  for (int i = 0; i < ne; ++i)
    if (!kv_op(k, MARS_KV_FREE, b.exp_row_sorted[i], -1)) return;
  const int nj = w->n_journal;
  for (int i = 0; i < nj; ++i) {
    int o = b.j_op[i];
    if (o == MARS_J_ALLOC) {
      if (!kv_op(k, MARS_KV_ALLOC, b.j_row[i], b.j_n[i])) return;
    } else {
      if (!kv_op(k, MARS_KV_FREE, b.j_row[i], -1)) return;
    }
  }
  if (w->in.mode & MARS_MODE_ADVANCE) {
    const int nr = w->n_round_end;
    for (int i = 0; i < nr; ++i)
      if (b.end_kind[i] != 1 && !kv_op(k, MARS_KV_FREE, b.end_row[i], -1)) return;
  }
}

// resume_from_tool's return-time release of an expired pin (sim.py:203-205),
// in the tool plane's finish order (kind 2 of mars_resume_rows)
__global__ void __launch_bounds__(KV_TPB) k_kv_resume_free(Kv k, i64 n, const i64* rows,
                                                           const u8* kind) {
  for (i64 i = 0; i < n; ++i)
    if (kind[i] == 2 && !kv_op(k, MARS_KV_FREE, (u32)rows[i], -1)) return;
}

int mars_kv_enqueue_resume_free(const Kv& k, cudaStream_t s, i64 n, const i64* rows,
                                const u8* kind) {
  k_kv_resume_free<<<1, KV_TPB, 0, s>>>(k, n, rows, kind);
  return (int)cudaGetLastError();
}

__global__ void k_kv_table(Kv k, u32 row, i64 cap, u32* out) {
  i64 len = k.len[row];
  if (len > cap) len = cap;
  for (i64 p = blockIdx.x * blockDim.x + threadIdx.x; p < len; p += gridDim.x * blockDim.x)
    out[p] = kv_slot(k, row, p);
}

__global__ void k_kv_top(Kv k, i64 cnt, u32* out) {
  i64 top = k.s->fs_top, fresh = k.s->fresh;
  for (i64 q = blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += gridDim.x * blockDim.x)
    out[q] = (q < top) ? k.fs[top - 1 - q] : (u32)(fresh + (q - top));
}

// SM-driven block copy (zero-copy pinned host memory): one CTA per block piece,
// 16-byte vector loads/stores.  dir 0: device -> host, 1: host -> device.
__global__ void __launch_bounds__(512) k_kv_copy(const Kv k, const u32* ids, i64 n, i64 slot0,
                                                 int dir) {
  const i64 piece = k.block_bytes / k.layers;
  const i64 pieces = n * k.layers;
  for (i64 pc = blockIdx.x; pc < pieces; pc += gridDim.x) {
    i64 bi = pc / k.layers, layer = pc % k.layers;
    i64 id = ids[bi];
    // device layout: layer-major [layer][block][piece] (vLLM-style) when layers > 1
    const u8* dsrc = k.data + (layer * k.total + id) * piece;
    u8* hdst = k.host + ((slot0 + bi) * k.layers + layer) * piece;
    const int4* s4 = (const int4*)(dir == 0 ? dsrc : hdst);
    int4* d4 = (int4*)(dir == 0 ? hdst : (u8*)dsrc);
    const i64 m = piece / 16;
    for (i64 j = threadIdx.x; j < m; j += blockDim.x) d4[j] = s4[j];
  }
}

int mars_kv_enqueue_apply(const Kv& k, cudaStream_t s, i64 n_ops, const u8* op, const u32* row,
                          const i32* n) {
  k_kv_apply<<<1, KV_TPB, 0, s>>>(k, n_ops, op, row, n);
  return (int)cudaGetLastError();
}

int mars_kv_enqueue_apply_step(const Kv& k, cudaStream_t s, Work* w, const Bufs& b) {
  k_kv_apply_step<<<1, KV_TPB, 0, s>>>(k, w, b);
  return (int)cudaGetLastError();
}

int mars_kv_enqueue_table(const Kv& k, cudaStream_t s, u32 row, i64 cap, u32* out) {
  k_kv_table<<<16, 256, 0, s>>>(k, row, cap, out);
  return (int)cudaGetLastError();
}

int mars_kv_enqueue_top(const Kv& k, cudaStream_t s, i64 cnt, u32* out) {
  k_kv_top<<<16, 256, 0, s>>>(k, cnt, out);
  return (int)cudaGetLastError();
}

int mars_kv_enqueue_copy(const Kv& k, cudaStream_t s, const u32* ids, i64 n, i64 slot0, int dir,
                         int grid) {
  k_kv_copy<<<grid, 512, 0, s>>>(k, ids, n, slot0, dir);
  return (int)cudaGetLastError();
}

// staged path: gather scattered blocks (layer-major pool) into a contiguous
// HBM staging buffer [n][layers][piece] -- or scatter back -- so the PCIe
// transfer is one large copy-engine DMA.  dir 0: pool -> staging, 1: back.
__global__ void __launch_bounds__(512) k_kv_stage(const Kv k, const u32* ids, i64 n, u8* stage,
                                                  int dir) {
  const i64 piece = k.block_bytes / k.layers;
  const i64 pieces = n * k.layers;
  for (i64 pc = blockIdx.x; pc < pieces; pc += gridDim.x) {
    i64 bi = pc / k.layers, layer = pc % k.layers;
    u8* pool = k.data + (layer * k.total + (i64)ids[bi]) * piece;
    u8* st = stage + (bi * k.layers + layer) * piece;
    const int4* s4 = (const int4*)(dir == 0 ? pool : st);
    int4* d4 = (int4*)(dir == 0 ? st : pool);
    const i64 m = piece / 16;
    for (i64 j = threadIdx.x; j < m; j += blockDim.x) d4[j] = s4[j];
  }
}

int mars_kv_enqueue_stage(const Kv& k, cudaStream_t s, const u32* ids, i64 n, u8* stage, int dir,
                          int grid) {
  k_kv_stage<<<grid, 512, 0, s>>>(k, ids, n, stage, dir);
  return (int)cudaGetLastError();
}
