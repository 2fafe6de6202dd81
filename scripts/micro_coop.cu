// Micro-benchmark: cost of a cooperative launch and of cg grid.sync() on this
// GPU (148 x 1024-thread CTAs), event-timed over many back-to-back launches.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mc scripts/micro_coop.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(1024, 1) k_sync(int nsync, unsigned* out) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < nsync; ++i) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = nsync;
}

// hand-rolled sense-reversing barrier (one arrival atomic per CTA)
__device__ __forceinline__ void bar_grid(unsigned* cnt, volatile unsigned* gen, unsigned nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g0 = *gen;
    __threadfence();
    if (atomicAdd(cnt, 1u) == nb - 1) {
      *cnt = 0;
      __threadfence();
      atomicAdd((unsigned*)gen, 1u);
    } else {
      while (*gen == g0) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(1024, 1) k_bar(int nsync, unsigned* cnt, unsigned* gen) {
  for (int i = 0; i < nsync; ++i) bar_grid(cnt, gen, gridDim.x);
}

__global__ void __launch_bounds__(1024, 1) k_plain(unsigned* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = 1;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned *out, *cnt, *gen;
  cudaMalloc(&out, 16);
  cudaMalloc(&cnt, 4);
  cudaMalloc(&gen, 4);
  cudaMemset(cnt, 0, 4);
  cudaMemset(gen, 0, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int R = 200;
  for (int ns : {0, 1, 2, 4, 8}) {
    void* args[] = {&ns, &out};
    for (int w = 0; w < 10; ++w)
      cudaLaunchCooperativeKernel((void*)k_sync, nsm, 1024, args, 0, 0);
    cudaEventRecord(a);
    for (int r = 0; r < R; ++r) cudaLaunchCooperativeKernel((void*)k_sync, nsm, 1024, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("coop launch, %d grid.sync: %.2f us/launch\n", ns, 1000 * ms / R);
  }
  for (int ns : {0, 1, 2, 4, 8}) {
    for (int w = 0; w < 10; ++w) k_bar<<<nsm, 1024>>>(ns, cnt, gen);
    cudaEventRecord(a);
    for (int r = 0; r < R; ++r) k_bar<<<nsm, 1024>>>(ns, cnt, gen);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("plain launch, %d hand barriers: %.2f us/launch\n", ns, 1000 * ms / R);
  }
  for (int w = 0; w < 10; ++w) k_plain<<<nsm, 1024>>>(out);
  cudaEventRecord(a);
  for (int r = 0; r < R; ++r) k_plain<<<nsm, 1024>>>(out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("plain empty launch: %.2f us/launch\n", 1000 * ms / R);
  // single launch bracketed by events (what the step profiler sees)
  {
    int ns = 1;
    void* args[] = {&ns, &out};
    float tot = 0;
    for (int r = 0; r < 20; ++r) {
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_sync, nsm, 1024, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      tot += ms;
    }
    printf("isolated coop launch (1 sync), event-bracketed: %.2f us\n", 1000 * tot / 20);
    tot = 0;
    for (int r = 0; r < 20; ++r) {
      cudaEventRecord(a);
      k_bar<<<nsm, 1024>>>(1, cnt, gen);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      tot += ms;
    }
    printf("isolated plain launch (1 hand barrier), event-bracketed: %.2f us\n", 1000 * tot / 20);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
