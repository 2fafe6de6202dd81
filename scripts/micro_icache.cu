// Micro-benchmark: cost of executing a cold straight-line code region once on
// B200 (instruction-cache misses), the pattern of the step's one-shot phases.
//  cold:   code in DRAM (first launch after an L2 flush) -- CTA 0's first run
//  l2warm: code already fetched into L2 by CTA 0, this SM's L1i cold -- the
//          other CTAs' first run after CTA 0 finished
//  hot:    second run on the same SM
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mi scripts/micro_icache.cu
#include <cstdio>

template <int R>
__device__ __noinline__ unsigned region(unsigned x) {
#pragma unroll
  for (int i = 0; i < R; ++i) x = ((x ^ (x >> 7)) * 0x9E3779B1u) + (unsigned)i;  // no folding
  return x;
}

__device__ __forceinline__ long long clk(unsigned dep) {
  long long t;
  asm volatile("add.u32 %1, %1, 0;\n\tmov.u64 %0, %%clock64;" : "=l"(t), "+r"(dep) :: "memory");
  return t;
}

template <int R>
__global__ void k_ic(unsigned long long* out, unsigned* sink, volatile unsigned* flag) {
  unsigned x = threadIdx.x;
  if (blockIdx.x > 0) {
    if (threadIdx.x == 0)
      while (*flag == 0) {
      }
    __syncthreads();
  }
  __shared__ unsigned sx[1024];
  const long long t0 = clk(x);
  x = region<R>(x);
  sx[threadIdx.x] = x;
  __syncthreads();
  const long long t1 = clk(sx[threadIdx.x ^ 1]);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence();
    *flag = 1;
  }
  x = region<R>(x + 1);
  sx[threadIdx.x] = x;
  __syncthreads();
  const long long t2 = clk(sx[threadIdx.x ^ 1]);
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = (unsigned long long)(t1 - t0);
    out[2 * blockIdx.x + 1] = (unsigned long long)(t2 - t1);
  }
  if (x == 0xdeadbeef) sink[0] = x;
}

template <int R>
void run(int blocks, int threads, void* flush, size_t fl) {
  unsigned long long* d;
  unsigned *s, *f;
  cudaMalloc(&d, 2 * blocks * 8);
  cudaMalloc(&s, 4);
  cudaMalloc(&f, 4);
  cudaMemset(f, 0, 4);
  cudaMemset(flush, 1, fl);  // evict the code from L2
  k_ic<R><<<blocks, threads>>>(d, s, f);
  cudaDeviceSynchronize();
  unsigned long long h[2 * 148];
  cudaMemcpy(h, d, 2 * blocks * 8, cudaMemcpyDeviceToHost);
  double b = 0, c = 0;
  for (int i = 1; i < blocks; ++i) {
    b += h[2 * i];
    c += h[2 * i + 1];
  }
  const double ins = 3.0 * R;  // SHF + LOP3 + IMAD per op
  printf("R=%5d (%5.0f SASS), %4d thr: cold %7llu cyc (%.1f/ins)  l2warm %7.0f cyc (%.1f/ins)  hot %5.0f\n",
         R, ins, threads, h[0], h[0] / ins, b / (blocks - 1), b / (blocks - 1) / ins, c / (blocks - 1));
  cudaFree(d);
  cudaFree(s);
  cudaFree(f);
}

int main() {
  void* flush;
  const size_t fl = 512u << 20;
  cudaMalloc(&flush, fl);
  run<512>(148, 1024, flush, fl);
  run<2048>(148, 1024, flush, fl);
  run<8192>(148, 1024, flush, fl);
  run<2048>(148, 32, flush, fl);
  run<8192>(148, 32, flush, fl);
  return 0;
}
