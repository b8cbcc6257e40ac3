// L2-resident vs HBM streaming read bandwidth (decides the fused-pass design)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const double2* __restrict__ x, size_t n, int reps, double* out) {
  double s = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      double2 v = __ldcg(x + i);
      s += v.x + v.y;
    }
  if (s == 12345.678) out[0] = s;
}
int main() {
  size_t big = (size_t)4 << 30, small = (size_t)48 << 20;
  double2* d; double* o;
  cudaMalloc(&d, big); cudaMalloc(&o, 8); cudaMemset(d, 0, big);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int grid = 148 * 8;
  for (int pass = 0; pass < 2; ++pass) {
    size_t bytes = pass ? small : big; int reps = pass ? 80 : 1;
    rd<<<grid, 512>>>(d, bytes / 16, reps, o);
    cudaEventRecord(a);
    rd<<<grid, 512>>>(d, bytes / 16, reps, o);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%s: %.1f GB/s\n", pass ? "L2-resident 48MB x80" : "HBM 4GB", bytes * (double)reps / ms / 1e6);
  }
  return 0;
}
