// Raw DMMA throughput probe: mma.sync f64 shapes on sm_100a. Not product code.
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>
__global__ void k(double* out, int iters) {
  double a[4], b[2], c[8][4];
  for (int i = 0; i < 4; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 2; ++i) b[i] = threadIdx.x * 2e-3 + i;
  for (int j = 0; j < 8; ++j) for (int i = 0; i < 4; ++i) c[j][i] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (SHAPE == 0) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a[0]), "d"(b[0]));
      } else if (SHAPE == 1) {
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      } else {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]),
                       "d"(b[0]), "d"(b[1]), "d"(b[0]), "d"(b[1]));
      }
    }
  }
  double s = 0;
  for (int j = 0; j < 8; ++j) for (int i = 0; i < 4; ++i) s += c[j][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out; cudaMalloc(&out, 148 * 64 * 1024 * 8);
  const char* names[3] = {"m8n8k4", "m16n8k4", "m16n8k16"};
  const double flops_per[3] = {8 * 8 * 4 * 2, 16 * 8 * 4 * 2, 16 * 8 * 16 * 2};
  for (int shape = 0; shape < 3; ++shape)
    for (int warps : {4, 8, 16}) {
      int iters = 2000;
      int blocks = 148 * 2;
      auto launch = [&] {
        if (shape == 0) k<0><<<blocks, warps * 32>>>(out, iters);
        if (shape == 1) k<1><<<blocks, warps * 32>>>(out, iters);
        if (shape == 2) k<2><<<blocks, warps * 32>>>(out, iters);
      };
      launch(); cudaDeviceSynchronize();
      cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
      cudaEventRecord(s); launch(); cudaEventRecord(e); cudaEventSynchronize(e);
      float ms; cudaEventElapsedTime(&ms, s, e);
      double fl = flops_per[shape] * 8.0 * iters * (double)blocks * warps;
      printf("%s warps/blk=%d blocks=%d: %.2f TFLOP/s\n", names[shape], warps, blocks, fl / (ms * 1e-3) / 1e12);
    }
  cudaError_t err = cudaGetLastError();
  printf("err=%s\n", cudaGetErrorString(err));
  return 0;
}
