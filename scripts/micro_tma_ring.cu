// Micro-benchmark: how fast can one persistent 148-CTA grid stream k_scan's
// 11 session-table columns (41 B/row) through a TMA bulk-copy ring, with no
// row processing?  Compares ring depth / round size and plain vector loads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mt scripts/micro_tma_ring.cu
#include <cstdio>
#include <cstdint>

typedef unsigned long long u64;
typedef uint32_t u32;

__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n"
               ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

struct Cols { const unsigned char* c[11]; };
__constant__ int kW[11] = {8, 8, 8, 4, 4, 4, 1, 1, 1, 1, 1};

// ring of NB buffers of R rows; every thread touches one byte of its row per
// round (so the data is "consumed"), then the CTA refills the buffer
__global__ void __launch_bounds__(1024, 1) k_ring(Cols C, long long n, long long chunk, int R, int NB,
                                                  unsigned* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) u64 bars[8];
  const int rowb = 41;
  const long long cs = (long long)blockIdx.x * chunk;
  const long long ce = cs + chunk < n ? cs + chunk : n;
  const int nr = ce > cs ? (int)((ce - cs + R - 1) / R) : 0;
  auto issue = [&](int rd) {
    const long long rb = cs + (long long)rd * R;
    const int k = (int)((ce - rb) < R ? (ce - rb) : R);
    const u32 k16 = (u32)((k + 15) & ~15);
    unsigned char* B = sm + (size_t)(rd % NB) * R * rowb;
    u64* bar = &bars[rd % NB];
    mbar_expect_tx(bar, k16 * rowb);
    size_t off = 0;
    for (int q = 0; q < 11; ++q) {
      bulk_g2s(B + off, C.c[q] + rb * kW[q], k16 * kW[q], bar);
      off += (size_t)R * kW[q];
    }
  };
  if (threadIdx.x == 0) {
    for (int q = 0; q < NB; ++q) mbar_init(&bars[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int rd = 0; rd < nr && rd < NB; ++rd) issue(rd);
  }
  __syncthreads();
  unsigned acc = 0;
  for (int rd = 0; rd < nr; ++rd) {
    mbar_wait(&bars[rd % NB], (u32)((rd / NB) & 1));
    const unsigned char* B = sm + (size_t)(rd % NB) * R * rowb;
    for (int i = threadIdx.x; i < R; i += blockDim.x) acc += B[(size_t)R * 36 + i];  // flags column
    __syncthreads();
    if (threadIdx.x == 0 && rd + NB < nr) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(rd + NB);
    }
  }
  if (acc == 0xdeadbeef) sink[0] = acc;
}

// plain coalesced 16-byte loads of the same columns (no shared memory)
__global__ void __launch_bounds__(1024, 1) k_plain(Cols C, long long n, unsigned* sink) {
  unsigned acc = 0;
  for (int q = 0; q < 11; ++q) {
    const uint4* p = (const uint4*)C.c[q];
    const long long m = n * kW[q] / 16;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (long long)gridDim.x * blockDim.x) {
      uint4 v = __ldcs(p + i);
      acc += v.x ^ v.w;
    }
  }
  if (acc == 0xdeadbeef) sink[0] = acc;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int widths[11] = {8, 8, 8, 4, 4, 4, 1, 1, 1, 1, 1};
  unsigned* sink;
  cudaMalloc(&sink, 4);
  cudaFuncSetAttribute(k_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (long long n : {1000000LL, 16000000LL, 64000000LL}) {
    Cols C;
    for (int q = 0; q < 11; ++q) {
      void* p;
      cudaMalloc(&p, (size_t)(n + 4096) * widths[q]);
      cudaMemset(p, q + 1, (size_t)(n + 4096) * widths[q]);
      C.c[q] = (const unsigned char*)p;
    }
    void* flush;
    const size_t fl = 512u << 20;
    cudaMalloc(&flush, fl);
    const double bytes = 41.0 * n;
    struct V { int R, NB; } vs[] = {{1024, 3}, {1024, 4}, {512, 6}, {512, 4}, {2048, 2}};
    for (V v : vs) {
      const size_t smem = (size_t)v.R * 41 * v.NB;
      if (smem > 200 * 1024) continue;
      long long units = (n + 15) / 16;
      long long chunk = ((units + nsm - 1) / nsm) * 16;
      float best = 1e30f;
      for (int it = 0; it < 5; ++it) {
        cudaMemsetAsync(flush, it, fl);
        cudaEventRecord(a);
        k_ring<<<nsm, 1024, smem>>>(C, n, chunk, v.R, v.NB, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (it > 0 && ms < best) best = ms;
      }
      printf("n=%lld ring R=%d NB=%d: %.3f ms  %.0f GB/s\n", n, v.R, v.NB, best, bytes / (best * 1e-3) / 1e9);
    }
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
      cudaMemsetAsync(flush, it, fl);
      cudaEventRecord(a);
      k_plain<<<nsm * 2, 1024>>>(C, n, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (it > 0 && ms < best) best = ms;
    }
    printf("n=%lld plain ld.v4: %.3f ms  %.0f GB/s\n", n, best, bytes / (best * 1e-3) / 1e9);
    for (int q = 0; q < 11; ++q) cudaFree((void*)C.c[q]);
    cudaFree(flush);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
