// Probe: host round-trip latency of launch + cudaStreamSynchronize on a B200.
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
__global__ void tiny(double* x) { if (threadIdx.x == 0) x[0] += 1.0; }
__global__ void spin(double* x, int iters) { double a = x[threadIdx.x]; for (int i = 0; i < iters; ++i) a = a * 0.999 + 1.0; x[threadIdx.x] = a; }
int main(int argc, char** argv) {
  if (argc > 1) cudaSetDeviceFlags(cudaDeviceScheduleSpin);
  double* x; cudaMalloc(&x, 1 << 20); cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  double *h; cudaMallocHost(&h, 64);
  for (int w = 0; w < 100; ++w) { tiny<<<1, 32, 0, s>>>(x); cudaStreamSynchronize(s); }
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < 1000; ++i) { tiny<<<1, 32, 0, s>>>(x); cudaMemcpyAsync(h, x, 8, cudaMemcpyDeviceToHost, s); cudaStreamSynchronize(s); }
  auto t1 = std::chrono::steady_clock::now();
  printf("launch+d2h+sync round trip: %.2f us\n", std::chrono::duration<double>(t1 - t0).count() * 1e3);
  // chain of 10 launches of ~20us kernels then sync
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < 100; ++i) { for (int k = 0; k < 10; ++k) spin<<<148, 256, 0, s>>>(x, 20000); cudaStreamSynchronize(s); }
  t1 = std::chrono::steady_clock::now();
  cudaEventRecord(e0, s); for (int k = 0; k < 10; ++k) spin<<<148, 256, 0, s>>>(x, 20000); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("10 x spin kernels + sync: wall %.1f us per group, device %.1f us per group\n", std::chrono::duration<double>(t1 - t0).count() * 1e4, ms * 1e3);
  return 0;
}
