// Paged KV block manager (S5) and the HBM <-> pinned-host KV tier.
//
// Block IDs follow the written-down policy of oracle/block_ids.py (the
// reference KvPool only counts, engine.py:116-221): a LIFO free stack whose
// pops first yield 0,1,2,..., alloc appends pops to the session's table,
// free pushes the table tail back in reverse (so the first freed ID is on
// top and an immediate re-allocation returns the same IDs in order).
//
// Layout: a session's table is a directory of 64-ID chunks.  The free stack
// is a stack of *segments* over an implicit "fresh" range of never-used IDs.
// A chunk segment is a whole 64-ID chunk handed over by a freed table (IDs
// pop forward from `start`); an arena segment holds < 64 loose IDs (a table's
// partial last chunk, a partial free's boundary part, the rest of a chunk a
// run popped partly) copied to the top of a LIFO ID arena (they pop from the
// segment's end).  Freeing a table is O(its chunks), not O(its IDs): the
// 1M-session step frees ~7K expired pins holding ~11M blocks by ~180K
// segment pushes and < 64 copied IDs per table.  Chunk segments are always
// full, so chunks in use stay below 2 * total/64 + rows.
//
// Ops apply in runs of one kind (frees or allocs, distinct rows within a
// run): a run is parallel over its ops via prefix sums (one CTA for the
// step's journal, the whole grid for the expired pins).
#include <cuda_runtime.h>

#include "mars_internal.cuh"
#include "mars_kv.h"

#define KV_TPB 1024
#define FULL32 0xffffffffu

// the q-th ID a segment pops
__device__ __forceinline__ u32 seg_id(const Kv& k, u64 sg, i64 q) {
  if (seg_is_arena(sg)) return k.arena[(i64)seg_index(sg) + seg_count(sg) - 1 - q];
  return k.chunks[(i64)seg_index(sg) * KV_CH + seg_start(sg) + q];
}

__device__ __forceinline__ u32* kv_slot_ptr(const Kv& k, u32 row, i64 pos) {
  const u32 ch = k.dir[(i64)row * k.D + pos / KV_CH];
  return &k.chunks[(i64)ch * KV_CH + pos % KV_CH];
}

// block-wide exclusive scan of one i64 per thread (blockDim.x == KV_TPB);
// returns the exclusive prefix, *total the sum
__device__ i64 kv_scan(i64 v, i64* total) {
  __shared__ i64 s_w[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  i64 incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const i64 x = __shfl_up_sync(FULL32, incl, o);
    if (lane >= o) incl += x;
  }
  __syncthreads();
  if (lane == 31) s_w[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    i64 t = s_w[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const i64 x = __shfl_up_sync(FULL32, t, o);
      if (lane >= o) t += x;
    }
    s_w[lane] = t;
  }
  __syncthreads();
  const i64 before = wid ? s_w[wid - 1] : 0;
  *total = s_w[31];
  __syncthreads();
  return before + incl - v;
}


// one per-block scratch area shared by the run kernels (a static __shared__
// inside a device function is one allocation per CTA, whatever the call site)
#define KV_SCRATCH (KV_TPB * 32)
__device__ __forceinline__ unsigned char* kv_scratch() {
  __shared__ __align__(16) unsigned char buf[KV_SCRATCH];
  return buf;
}


// One run of frees (distinct rows; n < 0: the whole table), <= KV_TPB ops, on
// the whole CTA.  Free i pushes its segments above those of frees 0..i-1; its
// first freed ID ends on top.  Thread i plans op i (prefix sums give every
// op's segment / arena / chunk-pool offsets), then one warp per op writes it.
// capm (nullable): per op, 1 if the freed IDs go to the host-tier capture
__device__ bool kv_free_run(Kv& k, int m, const u32* rows, const i32* ns,
                            const u8* capm = nullptr) {
  u32* o_row = (u32*)kv_scratch();
  i32* o_L = (i32*)(o_row + KV_TPB);
  i32* o_keep = o_L + KV_TPB;
  u32* o_so = (u32*)(o_keep + KV_TPB);
  u32* o_ao = o_so + KV_TPB;
  i32* o_ro = (i32*)(o_ao + KV_TPB);
  const int i = threadIdx.x;
  u32 row = 0;
  i64 L = 0, n = 0;
  if (i < m) {
    row = rows[i];
    L = k.len[row];
    n = (ns == nullptr || ns[i] < 0) ? L : ns[i];
  }
  const bool bad = i < m && n > L;
  if (__syncthreads_or(bad)) {
    if (threadIdx.x == 0) k.s->status |= 4;
    return false;
  }
  FreePlan f = free_plan(L, L - n);
  if (n == 0) f.nh = f.nt = f.f0 = f.f1 = 0, f.tail_chunk = false;
  const i64 nseg = (f.nt > 0) + (f.f1 - f.f0) + (f.nh > 0);
  i64 S, A, R, N;
  const i64 soff = kv_scan(nseg, &S);
  const i64 aoff = kv_scan(f.nh + f.nt, &A);
  const i64 roff = kv_scan(f.tail_chunk ? 1 : 0, &R);
  kv_scan(n, &N);
  const i64 s0 = k.s->seg_top, a0 = k.s->arena_top, c0 = k.s->cfs_top;
  if (s0 + S > k.seg_cap) {
    if (threadIdx.x == 0) k.s->status |= 32;
    return false;
  }
  if (i < m) {
    o_row[i] = row;
    o_L[i] = (i32)L;
    o_keep[i] = (i32)(n > 0 ? L - n : L);
    o_so[i] = (u32)soff;
    o_ao[i] = (u32)aoff;
    o_ro[i] = f.tail_chunk ? (i32)roff : -1;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int o = threadIdx.x >> 5; o < m; o += KV_TPB / 32) {
    const i64 Lo = o_L[o], ko = o_keep[o];
    if (ko == Lo) continue;  // nothing freed
    FreePlan g = free_plan(Lo, ko);
    kv_free_warp(k, o_row[o], g, s0 + o_so[o], a0 + o_ao[o], o_ro[o] < 0 ? -1 : c0 + o_ro[o],
                 lane, capm != nullptr && capm[o] != 0);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    k.s->seg_top = s0 + S;
    k.s->arena_top = a0 + A;
    k.s->fs_ids += N;
    k.s->cfs_top = c0 + R;
  }
  __syncthreads();
  return true;
}

// After a run popped F IDs from the touched top segments (top first, `cum`
// their prefix counts): emptied chunks return to the pool, an emptied arena
// segment lowers the arena top, and a partly popped chunk segment leaves its
// rest in the arena (chunk segments stay whole).  Thread 0; that rest's copy
// (< 64 IDs from chunk position cp[0] to arena position cp[1], cp[2] of them,
// in reverse) is left to the caller's threads.
__device__ void kv_settle(Kv& k, const u64* segs, const i64* cum, int nseg, i64 F, i64 top,
                          i64 ctop, i64* cp) {
  cp[2] = 0;
  i64 a = k.s->arena_top, cf = ctop;
  int full = 0;
  u64 last = 0;
  bool keep_last = false;
  for (int j = 0; j < nseg; ++j) {
    const u64 sg = segs[j];
    const i64 c = seg_count(sg), used = F - cum[j] < c ? F - cum[j] : c;
    if (used == c) {  // emptied
      ++full;
      if (seg_is_arena(sg)) a = (i64)seg_index(sg);
      else k.cfs[cf++] = (u32)seg_index(sg);
    } else if (seg_is_arena(sg)) {
      last = seg_arena_make((i64)seg_index(sg), (u32)(c - used));
      a = (i64)seg_index(sg) + (c - used);
      keep_last = true;
    } else {  // partly popped chunk: its rest to the arena, the chunk back
      const i64 r = c - used;
      cp[0] = (i64)seg_index(sg) * KV_CH + seg_start(sg) + used;
      cp[1] = a;
      cp[2] = r;
      last = seg_arena_make(a, (u32)r);
      a += r;
      k.cfs[cf++] = (u32)seg_index(sg);
      keep_last = true;
    }
  }
  i64 nt = top - full - (keep_last ? 1 : 0);
  if (keep_last) k.seg[nt++] = last;
  k.s->seg_top = nt;
  k.s->arena_top = a;
  k.s->cfs_top = cf;
}

// One run of allocs (distinct rows), <= KV_TPB ops, on the whole CTA: the
// run's N IDs are the next N pops (segments from the top, then fresh IDs),
// alloc i taking pops [off_i, off_i + n_i) onto its table's tail.  The top
// KV_TPB segments are staged in shared memory with their prefix counts; a run
// reaching deeper (only a host replay popping > KV_TPB small segments at
// once) pops one ID at a time on thread 0.
__device__ bool kv_alloc_run(Kv& k, int m, const u32* rows, const i32* ns) {
  i64* s_cum = (i64*)kv_scratch();
  u64* s_seg = (u64*)(s_cum + KV_TPB);
  i64* s_noff = (i64*)(s_seg + KV_TPB);
  u32* s_orow = (u32*)(s_noff + KV_TPB);
  i32* s_oL = (i32*)(s_orow + KV_TPB);
  const int i = threadIdx.x;
  u32 row = 0;
  i64 L = 0, n = 0;
  if (i < m) {
    row = rows[i];
    L = k.len[row];
    n = ns[i] > 0 ? ns[i] : 0;
  }
  const i64 cnew = n > 0 ? (L + n + KV_CH - 1) / KV_CH - (L + KV_CH - 1) / KV_CH : 0;
  const bool bad = i < m && (L + n > (i64)k.D * KV_CH);
  i64 N, Cn;
  const i64 noff = kv_scan(n, &N);
  const i64 coff = kv_scan(cnew, &Cn);
  const i64 top = k.s->seg_top, ids = k.s->fs_ids, fresh = k.s->fresh, ctop = k.s->cfs_top;
  if (__syncthreads_or(bad) || N > ids + (k.total - fresh) || Cn > ctop) {
    if (threadIdx.x == 0) k.s->status |= 1;
    return false;
  }
  if (N == 0) return true;
  const i64 F = N < ids ? N : ids;  // pops served by segments
  // new table chunks for the allocating rows (popped before any release)
  if (n > 0) {
    const i64 c0 = (L + KV_CH - 1) / KV_CH;
    for (i64 j = 0; j < cnew; ++j)
      k.dir[(i64)row * k.D + c0 + j] = k.cfs[ctop - 1 - (coff + j)];
  }
  // the top segments and the IDs before each
  const u64 sg = (i < top) ? k.seg[top - 1 - i] : 0ull;
  i64 staged;
  const i64 ex = kv_scan((i < top) ? (i64)seg_count(sg) : 0, &staged);
  s_seg[i] = sg;
  s_cum[i] = ex;
  __syncthreads();
  if (staged >= F) {
    i64 t;
    kv_scan((i < top && ex < F) ? 1 : 0, &t);
    const int nseg = (int)t;  // segments touched: those starting before F
    if (i < m) {
      s_noff[i] = noff;
      s_orow[i] = row;
      s_oL[i] = (i32)L;
    }
    __syncthreads();  // (the new chunks' directory entries are written too)
    // pop p of the run -> alloc op (last op starting at or before p; ops
    // with n = 0 start where the next one does) -> its table slot
    for (i64 p = threadIdx.x; p < N; p += KV_TPB) {
      int lo = 0, hi = m - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_noff[mid] <= p) lo = mid; else hi = mid - 1;
      }
      u32 id;
      if (p < F) {
        int a = 0, b2 = nseg - 1;
        while (a < b2) {
          const int mid = (a + b2 + 1) >> 1;
          if (s_cum[mid] <= p) a = mid; else b2 = mid - 1;
        }
        id = seg_id(k, s_seg[a], p - s_cum[a]);
      } else {
        id = (u32)(fresh + (p - F));
      }
      *kv_slot_ptr(k, s_orow[lo], (i64)s_oL[lo] + (p - s_noff[lo])) = id;
    }
    if (n > 0) k.len[row] = (i32)(L + n);
    __syncthreads();
    __shared__ i64 s_cp[3];
    if (threadIdx.x == 0) {
      kv_settle(k, s_seg, s_cum, nseg, F, top, ctop - Cn, s_cp);
      k.s->fs_ids = ids - F;
      k.s->fresh = fresh + (N - F);
    }
    __syncthreads();
    for (i64 q = threadIdx.x; q < s_cp[2]; q += KV_TPB)
      k.arena[s_cp[1] + s_cp[2] - 1 - q] = k.chunks[s_cp[0] + q];
  } else {
    // deep run: sequential pops (thread 0), in the run's order
    __syncthreads();
    s_cum[i] = (i < m) ? n : 0;  // reuse: per-op counts / rows
    s_seg[i] = row;
    __syncthreads();
    if (threadIdx.x == 0) {
      i64 st = top, cf = ctop - Cn, fr = fresh, left = ids, a = k.s->arena_top;
      for (int o = 0; o < m; ++o) {
        const u32 r = (u32)s_seg[o];
        const i64 la = k.len[r], na = s_cum[o];
        for (i64 q = 0; q < na; ++q) {
          u32 id;
          if (left > 0) {
            const u64 g = k.seg[st - 1];
            id = seg_id(k, g, 0);
            const u32 c = seg_count(g);
            if (c == 1) {
              if (seg_is_arena(g)) a = (i64)seg_index(g);
              else k.cfs[cf++] = (u32)seg_index(g);
              --st;
            } else if (seg_is_arena(g)) {
              k.seg[st - 1] = seg_arena_make((i64)seg_index(g), c - 1);
              a = (i64)seg_index(g) + c - 1;
            } else {
              k.seg[st - 1] = seg_chunk_make((u32)seg_index(g), seg_start(g) + 1, c - 1);
            }
            --left;
          } else {
            id = (u32)(fr++);
          }
          *kv_slot_ptr(k, r, la + q) = id;
        }
        k.len[r] = (i32)(la + na);
      }
      // a partly popped chunk on top leaves its rest in the arena
      if (st > 0 && !seg_is_arena(k.seg[st - 1]) && seg_count(k.seg[st - 1]) < KV_CH) {
        const u64 g = k.seg[st - 1];
        const i64 r = seg_count(g);
        for (i64 q = 0; q < r; ++q)
          k.arena[a + r - 1 - q] = k.chunks[(i64)seg_index(g) * KV_CH + seg_start(g) + q];
        k.seg[st - 1] = seg_arena_make(a, (u32)r);
        a += r;
        k.cfs[cf++] = (u32)seg_index(g);
      }
      k.s->seg_top = st;
      k.s->fs_ids = left;
      k.s->fresh = fr;
      k.s->cfs_top = cf;
      k.s->arena_top = a;
    }
  }
  __syncthreads();
  return true;
}

// An ordered op list (op, row, n) on one CTA: maximal runs of frees or of
// allocs with distinct rows, <= KV_TPB ops each, applied run by run.  PIN /
// UNPIN move ownership only (no table change).  `journal`: the ops are the
// step journal's codes (MARS_J_ALLOC, or a whole-table free).
__device__ void kv_apply_list(Kv& k, i64 n_ops, const u8* op, const u32* row, const i32* n,
                              bool journal) {
  __shared__ u32 s_row[KV_TPB];
  __shared__ i32 s_n[KV_TPB];
  __shared__ u8 s_kd[KV_TPB];
  __shared__ u8 s_cap[KV_TPB];  // host-tier capture: a running session's eviction
  __shared__ int s_m;
  const int t = threadIdx.x;
  // the window's rows -> their first position (open addressing in the run
  // scratch, which is free between runs): a repeated row ends the run
  constexpr int HS = 2 * KV_TPB;
  u32* h_key = (u32*)kv_scratch();
  int* h_first = (int*)(h_key + HS);
  static_assert(HS * 8 <= KV_SCRATCH, "row hash fits the run scratch");
  i64 i = 0;
  while (i < n_ops) {
    // the next window of ops, one per thread
    const bool valid = i + t < n_ops;
    int kd = 3;  // past the end
    u32 r = 0;
    if (valid) {
      const int o = op[i + t];
      if (journal) kd = (o == MARS_J_ALLOC) ? 1 : 2;
      else kd = (o == MARS_KV_ALLOC) ? 1 : (o == MARS_KV_FREE ? 2 : 0);
      r = row[i + t];
      s_row[t] = r;
      s_n[t] = (journal && kd == 2) ? -1 : n[i + t];
      s_cap[t] = (journal && o == MARS_J_EVICT_RUNNING) ? 1 : 0;
    }
    s_kd[t] = (u8)kd;
    for (int q = t; q < HS; q += KV_TPB) {
      h_key[q] = 0xffffffffu;
      h_first[q] = 0x7fffffff;
    }
    if (t == 0) s_m = KV_TPB;
    __syncthreads();
    int slot = 0;
    if (valid) {
      slot = (int)((r * 2654435761u) >> 21) & (HS - 1);
      for (;;) {
        const u32 prev = atomicCAS(&h_key[slot], 0xffffffffu, r);
        if (prev == 0xffffffffu || prev == r) break;
        slot = (slot + 1) & (HS - 1);
      }
      atomicMin(&h_first[slot], t);
    }
    __syncthreads();
    // the run is the longest prefix of one kind (alloc or free) with distinct
    // rows; a pin / unpin (no table change) is a run of its own, skipped.
    // Every thread tests whether its op ends the run (in parallel).
    const int kind = s_kd[0];
    if (t > 0) {
      const bool stop = kind == 0 || kd != kind || h_first[slot] < t;
      if (stop) atomicMin(&s_m, t);
    }
    __syncthreads();
    const int m = s_m;
    bool ok = true;
    if (kind == 1) ok = kv_alloc_run(k, m, s_row, s_n);
    else if (kind == 2) ok = kv_free_run(k, m, s_row, s_n, s_cap);
    if (!ok) return;
    i += m;
    __syncthreads();
  }
}

// host journal: ordered (op, row, n)
#ifdef MARS_PHASE_TIMING
#include <cstdio>
// debug builds only: first CTA start (even slots) / last CTA end (odd slots)
__device__ unsigned long long g_kvt[8];
__device__ __forceinline__ unsigned long long kvt_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define KVT_BEGIN(k) \
  if (threadIdx.x == 0) atomicMin(&g_kvt[2 * (k)], kvt_now())
#define KVT_END(k) \
  if (threadIdx.x == 0) atomicMax(&g_kvt[2 * (k) + 1], kvt_now())
__global__ void k_kvt_dump() {
  for (int k = 0; k < 4; ++k) {
    if (g_kvt[2 * k + 1]) printf("kvt %d %llu %llu\n", k, g_kvt[2 * k], g_kvt[2 * k + 1]);
    g_kvt[2 * k] = ~0ull;
    g_kvt[2 * k + 1] = 0;
  }
}
void mars_kv_ptime_dump(cudaStream_t s) { k_kvt_dump<<<1, 1, 0, s>>>(); }
#else
#define KVT_BEGIN(k)
#define KVT_END(k)
#endif

__global__ void __launch_bounds__(KV_TPB) k_kv_apply(Kv k, i64 n_ops, const u8* op, const u32* row,
                                                     const i32* n) {
  kv_apply_list(k, n_ops, op, row, n, false);
}

// The step's expired pins (rank order), freed as one run by the whole grid:
// k_kv_exp_scan (one CTA) computes every table's segment / arena / chunk
// offsets and moves the scalars, k_kv_exp_push writes each table's segments
// and loose IDs with one warp per table.
__global__ void __launch_bounds__(KV_TPB) k_kv_exp_scan(Kv k, const Work* w, Bufs b) {
  const int ne = w->n_exp;
  const int per = (ne + KV_TPB - 1) / KV_TPB;
  const int i0 = threadIdx.x * per, i1 = min(ne, i0 + per);
  // a pinned session's table is exactly its pinned blocks (a pin moves the
  // whole table, engine.py:190-200): the lengths come with the expired list,
  // all in flight at once (k_kv_exp_push checks them against the tables)
  constexpr int PR = 8;  // entries per thread held in registers (ne <= 8K; then loads)
  i32 Lr[PR];
#pragma unroll
  for (int q = 0; q < PR; ++q) Lr[q] = (i0 + q < i1) ? __ldcg(&b.exp_blk_sorted[i0 + q]) : 0;
  i64 segs = 0, ids = 0, ar = 0, rc = 0;
  auto add = [&](i64 L) {
    segs += L / KV_CH + ((L % KV_CH) ? 1 : 0);
    ar += L % KV_CH;
    rc += (L % KV_CH) ? 1 : 0;
    ids += L;
  };
#pragma unroll
  for (int q = 0; q < PR; ++q) add(Lr[q]);  // (0 past the run)
  for (int i = i0 + PR; i < i1; ++i) add(__ldcg(&b.exp_blk_sorted[i]));
  i64 S, N, A, R;
  i64 so = kv_scan(segs, &S);
  i64 ao = kv_scan(ar, &A);
  i64 ro = kv_scan(rc, &R);
  kv_scan(ids, &N);
  auto put = [&](int i, i64 L) {
    k.xoff[i] = so;
    k.xaoff[i] = ao;
    k.xroff[i] = ro;
    so += L / KV_CH + ((L % KV_CH) ? 1 : 0);
    ao += L % KV_CH;
    ro += (L % KV_CH) ? 1 : 0;
  };
#pragma unroll
  for (int q = 0; q < PR; ++q)
    if (i0 + q < i1) put(i0 + q, Lr[q]);
  for (int i = i0 + PR; i < i1; ++i) put(i, __ldcg(&b.exp_blk_sorted[i]));
  __syncthreads();
  if (threadIdx.x == 0) {
    const i64 s0 = k.s->seg_top;
    if (s0 + S > k.seg_cap) {
      k.s->status |= 32;
      k.xbase[1] = -1;
      return;
    }
    k.xbase[0] = s0;
    k.xbase[1] = S;
    k.xbase[2] = k.s->arena_top;
    k.xbase[3] = k.s->cfs_top;
    k.s->seg_top = s0 + S;
    k.s->arena_top += A;
    k.s->cfs_top += R;
    k.s->fs_ids += N;
  }
}

// a whole table: T = its partial last chunk (loose IDs to the arena, the
// chunk back to the pool), then its full chunks from the last one down
__global__ void k_kv_exp_push(Kv k, const Work* w, Bufs b) {
  // (a programmatic dependent of k_scan when the scan laid out the offsets:
  // resident early, it waits here for the scan's completion; a no-op else)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // the scan is complete: the control plane behind (a programmatic dependent
  // that shares no data with the push) may take SMs as they free up
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  KVT_BEGIN(0);
  const int ne = w->n_exp;
  if (__ldcg(&k.xbase[1]) < 0) return;  // the stack overflowed (status set)
  const i64 base = k.xbase[0], a0 = k.xbase[2], c0 = k.xbase[3];
  // one warp per table (a half warp per table measured the same, r2)
  const int lane = threadIdx.x & 31;
  for (int e = (int)(((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5); e < ne;
       e += (int)(((i64)gridDim.x * blockDim.x) >> 5)) {
    const u32 row = b.exp_row_sorted[e];
    const i64 L = b.exp_blk_sorted[e];
    if (lane == 0 && k.len[row] != L) atomicOr(&k.s->status, 64);  // table != pinned blocks
    kv_free_table_warp(k, row, L, base + k.xoff[e], a0 + k.xaoff[e], c0 + k.xroff[e], lane);
  }
  KVT_END(0);
}

// the rest of the step's journal on one CTA: k_walk's alloc / evict ops in
// plan order, then (MARS_MODE_ADVANCE) the tick tail's frees in decode order
// -- a finished session's blocks (sim.py:243) and an unpinned boundary's
// (sim.py:269); a pin keeps the table (ownership moves, the IDs stay)
// parts: 1 the journal, 2 the tick tail's frees, 3 both
__global__ void __launch_bounds__(KV_TPB) k_kv_apply_step(Kv k, Work* w, Bufs b, int parts) {
  KVT_BEGIN(1);
  if (k.s->status) return;
  if (parts & 1) kv_apply_list(k, w->n_journal, b.j_op, b.j_row, b.j_n, true);
  KVT_END(1);
  if ((parts & 2) && (w->in.mode & MARS_MODE_ADVANCE) && k.s->status == 0) {
    __shared__ u32 s_r[KV_TPB];
    __shared__ u8 s_c[KV_TPB];
    __shared__ int s_m;
    const int nr = w->n_round_end;
    for (int i0 = 0; i0 < nr; i0 += KV_TPB) {
      if (threadIdx.x == 0) {
        int m = 0;
        for (int i = i0; i < nr && i < i0 + KV_TPB; ++i)
          if (b.end_kind[i] != 1) {
            s_c[m] = b.end_kind[i] == 2 ? 1 : 0;  // an unpinned boundary (not a finished session)
            s_r[m++] = b.end_row[i];
          }
        s_m = m;
      }
      __syncthreads();
      if (!kv_free_run(k, s_m, s_r, nullptr, s_c)) return;
    }
  }
}

// resume_from_tool's return-time release of an expired pin (sim.py:203-205),
// in the tool plane's finish order (kind 2 of mars_resume_rows)
__global__ void __launch_bounds__(KV_TPB) k_kv_resume_free(Kv k, i64 n, const i64* rows,
                                                           const u8* kind) {
  __shared__ u32 s_r[KV_TPB];
  __shared__ int s_m;
  for (i64 i0 = 0; i0 < n; i0 += KV_TPB) {
    if (threadIdx.x == 0) {
      int m = 0;
      for (i64 i = i0; i < n && i < i0 + KV_TPB; ++i)
        if (kind[i] == 2) s_r[m++] = (u32)rows[i];
      s_m = m;
    }
    __syncthreads();
    if (!kv_free_run(k, s_m, s_r, nullptr)) return;
  }
}

// bulk table initialisation from a fresh pool (no free segment): row i of the
// list gets the next n_i IDs of the fresh range, exactly as n_i sequential
// allocs in list order would.  k_kv_bulk_scan (one CTA) + k_kv_bulk_fill.
__global__ void __launch_bounds__(KV_TPB) k_kv_bulk_scan(Kv k, i64 n, const u32* rows,
                                                         const i32* cnt) {
  const i64 per = (n + KV_TPB - 1) / KV_TPB;
  const i64 i0 = threadIdx.x * per, i1 = (i0 + per < n) ? i0 + per : n;
  i64 ids = 0, chs = 0;
  for (i64 i = i0; i < i1; ++i) {
    const i64 L = k.len[rows[i]], c = cnt[i];
    ids += c;
    chs += (L + c + KV_CH - 1) / KV_CH - (L + KV_CH - 1) / KV_CH;
  }
  i64 N, C;
  i64 io = kv_scan(ids, &N);
  i64 co = kv_scan(chs, &C);
  const i64 fresh = k.s->fresh, ctop = k.s->cfs_top;
  if (k.s->fs_ids != 0 || N > k.total - fresh || C > ctop) {
    if (threadIdx.x == 0) k.s->status |= 16;
    return;
  }
  for (i64 i = i0; i < i1; ++i) {
    const i64 L = k.len[rows[i]], c = cnt[i];
    const i64 c0 = (L + KV_CH - 1) / KV_CH, cn = (L + c + KV_CH - 1) / KV_CH - c0;
    for (i64 j = 0; j < cn; ++j) k.dir[(i64)rows[i] * k.D + c0 + j] = k.cfs[ctop - 1 - (co + j)];
    k.xoff[i] = fresh + io;  // first ID of this row
    io += c;
    co += cn;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    k.s->fresh = fresh + N;
    k.s->cfs_top = ctop - C;
  }
}

__global__ void k_kv_bulk_fill(Kv k, i64 n, const u32* rows, const i32* cnt) {
  // one warp per row: consecutive IDs onto its table tail, then the length
  const int lane = threadIdx.x & 31;
  for (i64 i = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((i64)gridDim.x * blockDim.x) >> 5) {
    const u32 r = rows[i];
    const i64 L = k.len[r], c = cnt[i], id0 = k.xoff[i];
    for (i64 q = lane; q < c; q += 32) *kv_slot_ptr(k, r, L + q) = (u32)(id0 + q);
    __syncwarp();
    if (lane == 0) k.len[r] = (i32)(L + c);
  }
}

__global__ void k_kv_table(Kv k, u32 row, i64 cap, u32* out) {
  i64 len = k.len[row];
  if (len > cap) len = cap;
  for (i64 p = blockIdx.x * blockDim.x + threadIdx.x; p < len; p += gridDim.x * blockDim.x)
    out[p] = *kv_slot_ptr(k, row, p);
}

// the next `cnt` IDs pops would return (segments from the top, then fresh)
__global__ void k_kv_top(Kv k, i64 cnt, u32* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  i64 q = 0;
  for (i64 j = k.s->seg_top - 1; j >= 0 && q < cnt; --j) {
    const u64 sg = k.seg[j];
    for (u32 t = 0; t < seg_count(sg) && q < cnt; ++t) out[q++] = seg_id(k, sg, t);
  }
  for (i64 f = k.s->fresh; q < cnt; ++f) out[q++] = f < k.total ? (u32)f : 0xffffffffu;
}

int mars_kv_enqueue_apply(const Kv& k, cudaStream_t s, i64 n_ops, const u8* op, const u32* row,
                          const i32* n) {
  k_kv_apply<<<1, KV_TPB, 0, s>>>(k, n_ops, op, row, n);
  return (int)cudaGetLastError();
}

int mars_kv_enqueue_exp_free(const Kv& k, cudaStream_t s, Work* w, const Bufs& b, int grid,
                             bool offsets_done, bool pdl) {
  if (!offsets_done) k_kv_exp_scan<<<1, KV_TPB, 0, s>>>(k, w, b);
  // small CTAs, one wave of at most 1024 threads per SM: resident beside
  // k_scan's CTA while they wait for it (programmatic launch), they leave
  // the scan's slot to the walk, which launches when the scan ends (8 per SM
  // queued CTAs ahead of the walk and delayed its start by ~7 us at 1M, r2)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(4 * grid);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k_kv_exp_push, k, (const Work*)w, b);
  return (int)cudaGetLastError();
}

int mars_kv_enqueue_apply_step(const Kv& k, cudaStream_t s, Work* w, const Bufs& b, int parts) {
  k_kv_apply_step<<<1, KV_TPB, 0, s>>>(k, w, b, parts);
  return (int)cudaGetLastError();
}

int mars_kv_enqueue_resume_free(const Kv& k, cudaStream_t s, i64 n, const i64* rows,
                                const u8* kind) {
  k_kv_resume_free<<<1, KV_TPB, 0, s>>>(k, n, rows, kind);
  return (int)cudaGetLastError();
}

int mars_kv_enqueue_bulk(const Kv& k, cudaStream_t s, i64 n, const u32* rows, const i32* cnt,
                         int grid) {
  k_kv_bulk_scan<<<1, KV_TPB, 0, s>>>(k, n, rows, cnt);
  k_kv_bulk_fill<<<grid, 256, 0, s>>>(k, n, rows, cnt);
  return (int)cudaGetLastError();
}

// the tables of n rows into one list (row i's IDs at out[off[i]..off[i+1]),
// one warp per row; a table whose length is not off[i+1] - off[i] sets
// status bit 256
__global__ void k_kv_gather_ids(Kv k, i64 n, const u32* rows, const i64* off, u32* out) {
  const int lane = threadIdx.x & 31;
  for (i64 i = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((i64)gridDim.x * blockDim.x) >> 5) {
    const u32 r = rows[i];
    const i64 o = off[i], c = off[i + 1] - o;
    if (lane == 0 && (i64)k.len[r] != c) atomicOr(&k.s->status, 256);
    const u32* dr = k.dir + (i64)r * k.D;
    for (i64 p = lane; p < c; p += 32) out[o + p] = k.chunks[(i64)dr[p / KV_CH] * KV_CH + p % KV_CH];
  }
}

int mars_kv_enqueue_gather_ids(const Kv& k, cudaStream_t s, i64 n, const u32* rows, const i64* off,
                               u32* out, int grid) {
  k_kv_gather_ids<<<grid, 256, 0, s>>>(k, n, rows, off, out);
  return (int)cudaGetLastError();
}

int mars_kv_enqueue_table(const Kv& k, cudaStream_t s, u32 row, i64 cap, u32* out) {
  k_kv_table<<<16, 256, 0, s>>>(k, row, cap, out);
  return (int)cudaGetLastError();
}

int mars_kv_enqueue_top(const Kv& k, cudaStream_t s, i64 cnt, u32* out) {
  k_kv_top<<<1, 32, 0, s>>>(k, cnt, out);
  return (int)cudaGetLastError();
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

// every kernel of this file loaded now (see mars_kernels_preload)
int mars_kv_preload() {
  cudaFuncAttributes fa;
  const void* fns[] = {(const void*)k_kv_apply, (const void*)k_kv_apply_step,
                       (const void*)k_kv_bulk_fill, (const void*)k_kv_bulk_scan,
                       (const void*)k_kv_copy, (const void*)k_kv_exp_push,
                       (const void*)k_kv_exp_scan, (const void*)k_kv_gather_ids,
                       (const void*)k_kv_resume_free, (const void*)k_kv_stage,
                       (const void*)k_kv_table, (const void*)k_kv_top};
  for (const void* f : fns) {
    cudaError_t e = cudaFuncGetAttributes(&fa, f);
    if (e != cudaSuccess) return (int)e;
  }
  return 0;
}
