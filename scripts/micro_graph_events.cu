// Do CUDA events recorded inside a captured graph time the kernels between
// them (cudaEventElapsedTime after a replay)?  Prints both timings.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_spin(long long cycles) {
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
}
int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  k_spin<<<1, 32, 0, s>>>(100000);
  cudaEventRecord(a, s);
  k_spin<<<1, 32, 0, s>>>(2000000);  // ~1 ms at ~2 GHz
  cudaEventRecord(b, s);
  cudaError_t e = cudaStreamEndCapture(s, &g);
  printf("capture: %s\n", cudaGetErrorString(e));
  e = cudaGraphInstantiate(&ge, g, 0);
  printf("instantiate: %s\n", cudaGetErrorString(e));
  for (int i = 0; i < 3; ++i) {
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    float ms = -1;
    e = cudaEventElapsedTime(&ms, a, b);
    printf("replay %d: elapsed %s %.4f ms\n", i, cudaGetErrorString(e), ms);
  }
  return 0;
}
