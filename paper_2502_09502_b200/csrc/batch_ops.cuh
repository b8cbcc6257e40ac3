// Elementwise helpers of the batched engine: 3xTF32 operand splitting.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace l0 {

// x ~= hi + lo, hi exactly representable in TF32 (round to nearest on the
// magnitude), lo = fp32(x - hi).  Exact for fp32 x up to TF32's truncation of lo.
__device__ __forceinline__ void tf32_split(double x, float& hi, float& lo) {
  const float xf = (float)x;
  const float h = __uint_as_float((__float_as_uint(xf) + 0x1000u) & 0xFFFFE000u);
  hi = h;
  lo = (float)(x - (double)h);
}

// rows x cols (row pitch ld_in) fp32 or fp64 -> hi/lo fp32 with pitch ld_out,
// zero in the padding columns [cols, ld_out)
template <typename T>
__global__ void k_split_rows(const T* in, int64_t rows, int64_t cols, int64_t ld_in, float* hi,
                             float* lo, int64_t ld_out) {
  const int64_t total = rows * ld_out;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / ld_out, c = e - r * ld_out;
    float h = 0.f, l = 0.f;
    if (c < cols) tf32_split((double)in[r * ld_in + c], h, l);
    hi[e] = h;
    lo[e] = l;
  }
}

// transpose + split: in is rows x cols (pitch ld_in); out is cols x ld_out
// (ld_out >= rows), 32x32 tiles through shared memory
template <typename T>
__global__ void k_split_transpose(const T* in, int64_t rows, int64_t cols, int64_t ld_in, float* hi,
                                  float* lo, int64_t ld_out) {
  __shared__ double tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (r < rows && c < cols) ? (double)in[r * ld_in + c] : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;   // out[c][r]
    if (c < cols && r < ld_out) {
      float h, l;
      tf32_split(tile[threadIdx.x][i], h, l);
      hi[c * ld_out + r] = h;
      lo[c * ld_out + r] = l;
    }
  }
}

}  // namespace l0
