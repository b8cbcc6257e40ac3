// Elementwise helpers of the batched engine: 3xTF32 / 3xFP16 operand splitting.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math.h>
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

// xs (already scaled, |xs| < 2^14) ~= hi + lo in fp16: hi the nearest fp16,
// lo the nearest fp16 of the remainder (tc_gemm.cuh, 3xFP16)
__device__ __forceinline__ void f16_split(double xs, __half& hi, __half& lo) {
  hi = __double2half(xs);
  lo = __double2half(xs - (double)__half2float(hi));
}
__device__ __forceinline__ bool f16_nonzero(__half h) { return (__half_as_ushort(h) & 0x7fffu) != 0u; }

// power-of-two exponent s with amax * 2^s < 2^14 (0 for a zero / non-finite amax)
__host__ __device__ inline int f16_exp(double amax) {
  if (!(amax > 0.0) || !(amax < 1e300)) return 0;
  int e = 0;
  frexp(amax, &e);   // amax < 2^e
  int s = 14 - e;
  return s < -100 ? -100 : (s > 100 ? 100 : s);
}

// max |x| over a rows x cols matrix (pitch ld) -> *out (as float bits, atomicMax
// on the non-negative float's integer image; *out zeroed by the caller)
template <typename T>
__global__ void k_absmax(const T* in, int64_t rows, int64_t cols, int64_t ld, unsigned* out) {
  float m = 0.f;
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols, c = e - r * cols;
    m = fmaxf(m, (float)fabs((double)in[r * ld + c]));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

// scaled fp16 splits of a matrix: row-major (pitch ld_out, zero padding
// columns) and transposed (out is cols x ld_out), as the fp32 kernels below
template <typename T>
__global__ void k_split_rows_h(const T* in, int64_t rows, int64_t cols, int64_t ld_in, double sc, __half* hi,
                               __half* lo, int64_t ld_out) {
  const int64_t total = rows * ld_out;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / ld_out, c = e - r * ld_out;
    __half h = __ushort_as_half(0), l = __ushort_as_half(0);
    if (c < cols) f16_split((double)in[r * ld_in + c] * sc, h, l);
    hi[e] = h;
    lo[e] = l;
  }
}
template <typename T>
__global__ void k_split_transpose_h(const T* in, int64_t rows, int64_t cols, int64_t ld_in, double sc,
                                    __half* hi, __half* lo, int64_t ld_out) {
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
      __half h, l;
      f16_split(tile[threadIdx.x][i] * sc, h, l);
      hi[c * ld_out + r] = h;
      lo[c * ld_out + r] = l;
    }
  }
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
