// Measures FFMA / DFMA throughput on the device (development aid): 8 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void k(T* out, int iters, T a, T b) {
  T x[8];
  for (int i = 0; i < 8; ++i) x[i] = T(threadIdx.x + i);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  T s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <typename T>
void run(const char* name) {
  T* d;
  cudaMalloc(&d, sizeof(T) * 148 * 8 * 1024);
  const int iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<T><<<148 * 8, 1024>>>(d, 10, T(1.0000001), T(1e-7));
  cudaEventRecord(e0);
  k<T><<<148 * 8, 1024>>>(d, iters, T(1.0000001), T(1e-7));
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fmas = double(148 * 8) * 1024 * iters * 8;
  int dev;
  cudaGetDevice(&dev);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("%s: %.2f TFMA/s = %.1f FMA/clk/SM (%.3f ms)\n", name, fmas / ms / 1e9, fmas / (ms * 1e-3) / 148 / (clk * 1e3), ms);
  cudaFree(d);
}
int main() {
  run<float>("FFMA");
  run<double>("DFMA");
  return 0;
}
