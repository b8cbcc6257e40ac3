// Column standardisation on the device, bit-identical to the reference's numpy
// (data.py:224-242): numpy reduces a C-contiguous matrix over axis 0 row by
// row, so every column sum below is the same sequential sum over rows
// (x_0 + x_1) + x_2 + ..., with one IEEE rounding per operation (no FMA
// contraction):
//   mean_j  = (sum_i x_ij) / n                       X.mean(axis=0)
//   norm_j  = sqrt(sum_i (x_ij - mean_j)^2)          np.linalg.norm(X - mean, axis=0)
//   scale_j = max_i |x_ij|                           np.abs(X).max(axis=0)
//   out_ic  = (x_i,kept_c - mean) / norm             centered[:, kept] / norms[kept]
// One thread per column walks the rows (consecutive threads read consecutive
// columns: coalesced), eight rows of loads in flight per step.

#include "engine.cuh"

namespace l0 {

constexpr int kStdUnroll = 8;

__global__ void __launch_bounds__(128) k_std_stats(const double* __restrict__ X, int64_t n, int64_t p,
                                                   int64_t ld, double* __restrict__ mean,
                                                   double* __restrict__ norm, double* __restrict__ scale) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= p) return;
  const double* col = X + j;
  double s = 0.0, amax = 0.0;
  int64_t i = 0;
  for (; i + kStdUnroll <= n; i += kStdUnroll) {
    double v[kStdUnroll];
#pragma unroll
    for (int u = 0; u < kStdUnroll; ++u) v[u] = __ldg(col + (i + u) * ld);
#pragma unroll
    for (int u = 0; u < kStdUnroll; ++u) {
      s = dadd(s, v[u]);
      amax = fmax(amax, fabs(v[u]));
    }
  }
  for (; i < n; ++i) {
    const double v = __ldg(col + i * ld);
    s = dadd(s, v);
    amax = fmax(amax, fabs(v));
  }
  const double m = ddiv(s, (double)n);
  double ss = 0.0;
  for (i = 0; i + kStdUnroll <= n; i += kStdUnroll) {
    double v[kStdUnroll];
#pragma unroll
    for (int u = 0; u < kStdUnroll; ++u) v[u] = __ldg(col + (i + u) * ld);
#pragma unroll
    for (int u = 0; u < kStdUnroll; ++u) {
      const double c = dsub(v[u], m);
      ss = dadd(ss, dmul(c, c));
    }
  }
  for (; i < n; ++i) {
    const double c = dsub(__ldg(col + i * ld), m);
    ss = dadd(ss, dmul(c, c));
  }
  mean[j] = m;
  norm[j] = sqrt(ss);   // IEEE square root, as np.sqrt
  scale[j] = amax;
}

__global__ void k_std_apply(const double* __restrict__ X, int64_t n, int64_t ld, const int64_t* __restrict__ kept,
                            int64_t m, const double* __restrict__ mean, const double* __restrict__ norm,
                            double* __restrict__ out) {
  const int64_t total = n * m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / m, c = e % m;
    const int64_t j = kept[c];
    out[e] = ddiv(dsub(X[i * ld + j], mean[j]), norm[j]);
  }
}

}  // namespace l0

extern "C" {

// data.py:224-236: per-column mean, centred norm and max |x| (host decides `keep`)
int32_t l0_standardize_stats(const double* d_X, int64_t n, int64_t p, int64_t ld, double* d_mean,
                             double* d_norm, double* d_scale, void* stream) {
  if (!d_X || !d_mean || !d_norm || !d_scale || n < 1 || p < 1 || ld < p)
    return set_error(ST_INVALID, "bad arguments");
  k_std_stats<<<(unsigned)((p + 127) / 128), 128, 0, (cudaStream_t)stream>>>(d_X, n, p, ld, d_mean, d_norm,
                                                                               d_scale);
  OPS_CUDA(cudaGetLastError());
  return ST_OK;
}

// data.py:237-242: out (n x m, row-major) = (X[:, kept] - mean[kept]) / norm[kept]
int32_t l0_standardize_apply(const double* d_X, int64_t n, int64_t ld, const int64_t* d_kept, int64_t m,
                             const double* d_mean, const double* d_norm, double* d_out, void* stream) {
  if (!d_X || !d_kept || !d_mean || !d_norm || !d_out || n < 1 || m < 1)
    return set_error(ST_INVALID, "bad arguments");
  const int64_t blocks = std::min<int64_t>(148 * 16, (n * m + 255) / 256);
  k_std_apply<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(d_X, n, ld, d_kept, m, d_mean, d_norm, d_out);
  OPS_CUDA(cudaGetLastError());
  return ST_OK;
}

}  // extern "C"
