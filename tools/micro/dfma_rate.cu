// Throughput of DFMA, F2F.F64.F32 and the integer rebias per SM on this GPU:
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dfma_rate dfma_rate.cu && ./dfma_rate
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* out, float seed, int iters) {
  double a[8];
  float f[8];
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x + i; f[i] = seed + i; }
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = fma(a[i], b, c);                       // DFMA
      if (MODE == 1) { a[i] += (double)f[i]; f[i] += 1.0f; }        // F2F + DADD + FADD
      if (MODE == 2) { f[i] = fmaf(f[i], 1.0000001f, 1e-9f); }      // FFMA
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i] + f[i];
  if (s == 12345.678) out[0] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096, threads = 512, blocks = sms * 4;
  const char* names[3] = {"DFMA", "F2F.F64.F32 (+DADD +FADD)", "FFMA"};
  for (int m = 0; m < 3; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (m == 0) k<0><<<blocks, threads>>>(out, 1.f, iters);
      if (m == 1) k<1><<<blocks, threads>>>(out, 1.f, iters);
      if (m == 2) k<2><<<blocks, threads>>>(out, 1.f, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double ops = (double)blocks * threads * iters * 8;
      if (rep) printf("%-28s %.3f ms  %.1f G/s  = %.1f per clk per SM (at %d MHz)\n", names[m], ms, ops / ms / 1e6,
                      ops / (ms * 1e-3) / (sms * (double)clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
