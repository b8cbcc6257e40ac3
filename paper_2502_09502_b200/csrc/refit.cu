// Batched exact ridge refits for the branch-and-bound driver (bnb.py _refit,
// squared error; SPEC.md:314-330 incumbents and node points): for C candidate
// supports S_c (|S_c| <= kRefitMaxS = 48) at once,
//
//   b_c = argmin ||y - X_S b||^2 + l2 ||b||^2 = (X_S^T X_S + l2 I)^{-1} X_S^T y
//   obj_c = y^T y - 2 b^T h + b^T (X_S^T X_S + l2 I) b
//
// One CTA per support: the support's columns are gathered 64 rows at a time
// into shared memory (X widened to fp64 once), every thread owns fixed entries
// of G = X_S^T X_S and h = X_S^T y and accumulates them in row order (fixed
// order: deterministic), then one warp factors G + l2 I (Cholesky) and solves.
// Replaces the eager einsum / linalg.solve of the round-1 driver (a cuBLAS /
// cuSOLVER call per refit batch and ~20 small launches around it).

#include "engine.cuh"

namespace l0 {

constexpr int kRefitMaxS = 48;   // static shared memory: G and the row chunk under 48 KB
constexpr int kRefitRows = 64;
constexpr int kRefitThreads = 256;

template <typename TX>
__global__ void __launch_bounds__(kRefitThreads) k_refit_ridge(const TX* __restrict__ X, int64_t n, int64_t ld,
                                                               const double* __restrict__ y, double yty,
                                                               const int* __restrict__ supp, int s, double l2,
                                                               double* __restrict__ beta, double* __restrict__ obj) {
  __shared__ int S[kRefitMaxS];
  __shared__ double xs[kRefitRows][kRefitMaxS + 1];
  __shared__ double ys[kRefitRows];
  __shared__ double G[kRefitMaxS][kRefitMaxS + 1];
  __shared__ double h[kRefitMaxS];
  __shared__ double b[kRefitMaxS];
  __shared__ int m_s;
  const int c = blockIdx.x, tid = threadIdx.x;
  if (tid == 0) {
    int m = 0;
    for (int j = 0; j < s; ++j) {
      const int v = supp[(int64_t)c * s + j];
      if (v >= 0) S[m++] = v;
    }
    m_s = m;
  }
  __syncthreads();
  const int m = m_s;
  // entries owned by this thread: e < m(m+1)/2 -> G[j][l] (j <= l), then h
  const int ng = m * (m + 1) / 2, ne = ng + m;
  constexpr int kOwn = (kRefitMaxS * (kRefitMaxS + 1) / 2 + kRefitMaxS + kRefitThreads - 1) / kRefitThreads;
  double acc[kOwn];
  int ej[kOwn], el[kOwn];
#pragma unroll
  for (int q = 0; q < kOwn; ++q) {
    acc[q] = 0.0;
    const int e = tid + q * kRefitThreads;
    int j = -1, l = -1;
    if (e < ng) {   // row-major upper triangle: j such that j*(2m-j+1)/2 <= e
      int jj = 0, base = 0;
      while (base + (m - jj) <= e) { base += m - jj; ++jj; }
      j = jj;
      l = jj + (e - base);
    } else if (e < ne) {
      j = e - ng;   // h[j]
      l = -2;
    }
    ej[q] = j;
    el[q] = l;
  }
  for (int64_t i0 = 0; i0 < n; i0 += kRefitRows) {
    const int rows = (int)min((int64_t)kRefitRows, n - i0);
    for (int e = tid; e < rows * m; e += kRefitThreads) {
      const int r = e / m, j = e % m;
      xs[r][j] = (double)X[(i0 + r) * ld + S[j]];
    }
    for (int r = tid; r < rows; r += kRefitThreads) ys[r] = y[i0 + r];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kOwn; ++q) {
      const int j = ej[q], l = el[q];
      if (j < 0) continue;
      double a = acc[q];
      if (l >= 0)
        for (int r = 0; r < rows; ++r) a = fma(xs[r][j], xs[r][l], a);
      else
        for (int r = 0; r < rows; ++r) a = fma(xs[r][j], ys[r], a);
      acc[q] = a;
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < kOwn; ++q) {
    const int j = ej[q], l = el[q];
    if (j < 0) continue;
    if (l >= 0) {
      G[j][l] = acc[q];
      G[l][j] = acc[q];
    } else {
      h[j] = acc[q];
    }
  }
  __syncthreads();
  if (tid < 32) {
    // Cholesky G + l2 I = L L^T in place (lower triangle), one warp
    const int lane = tid;
    for (int j = 0; j < m; ++j) {
      if (lane == 0) {
        double d = G[j][j] + l2;
        for (int k = 0; k < j; ++k) d -= G[j][k] * G[j][k];
        G[j][j] = sqrt(d);
      }
      __syncwarp();
      for (int i = j + 1 + lane; i < m; i += 32) {
        double v = G[i][j];
        for (int k = 0; k < j; ++k) v -= G[i][k] * G[j][k];
        G[i][j] = v / G[j][j];
      }
      __syncwarp();
    }
    if (lane == 0) {
      // L z = h, L^T b = z
      for (int i = 0; i < m; ++i) {
        double v = h[i];
        for (int k = 0; k < i; ++k) v -= G[i][k] * b[k];
        b[i] = v / G[i][i];
      }
      for (int i = m - 1; i >= 0; --i) {
        double v = b[i];
        for (int k = i + 1; k < m; ++k) v -= G[k][i] * b[k];
        b[i] = v / G[i][i];
      }
      // objective y^T y - 2 b^T h + b^T (L L^T) b = y^T y - 2 b^T h + |L^T b|^2
      double bh = 0.0, q2 = 0.0;
      for (int i = 0; i < m; ++i) bh += b[i] * h[i];
      for (int i = 0; i < m; ++i) {
        double v = 0.0;
        for (int k = i; k < m; ++k) v += G[k][i] * b[k];
        q2 += v * v;
      }
      obj[c] = yty - 2.0 * bh + q2;
    }
  }
  __syncthreads();
  // write b in the support's slot order (padding -> 0)
  if (tid == 0) {
    int q = 0;
    for (int j = 0; j < s; ++j) {
      const int v = supp[(int64_t)c * s + j];
      beta[(int64_t)c * s + j] = v >= 0 ? b[q++] : 0.0;
    }
  }
}

}  // namespace l0

extern "C" {

// bnb.py _refit (squared error): C supports of width s (int32, -1 = padding,
// device), exact ridge solutions d_beta (C x s) and objectives d_obj (C)
int32_t l0_refit_ridge(l0_problem* P, const int32_t* d_supports, int64_t C, int32_t s, double lambda2,
                       double yty, double* d_beta, double* d_obj, void* stream) {
  if (!P || !d_supports || !d_beta || !d_obj || C < 0 || s < 1 || s > kRefitMaxS || !(lambda2 > 0))
    return set_error(ST_INVALID, "bad arguments");
  if (C == 0) return ST_OK;
  const EngineArgs& a = P->a;
  cudaStream_t st = (cudaStream_t)stream;
  if (a.dtype == F64)
    k_refit_ridge<double><<<(unsigned)C, kRefitThreads, 0, st>>>(static_cast<const double*>(a.X), a.n, a.ld, a.y, yty,
                                                                 d_supports, s, lambda2, d_beta, d_obj);
  else
    k_refit_ridge<float><<<(unsigned)C, kRefitThreads, 0, st>>>(static_cast<const float*>(a.X), a.n, a.ld, a.y, yty,
                                                                d_supports, s, lambda2, d_beta, d_obj);
  OPS_CUDA(cudaGetLastError());
  return ST_OK;
}

}  // extern "C"
