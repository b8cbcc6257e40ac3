// Batched fp64 safe lower bound (reference
// perspective.py:162-190 per node):
//
//   U = X B^T            (n x nb, fp64 multi-right-hand-side pass)
//   zeta_j = -grad F(U_j),  F*(-zeta_j)        (one CTA per node)
//   V = X^T Z            (p x nb, fp64 multi-right-hand-side pass, split over rows)
//   g*_j = sum_{fixed-one} H + TopSum_{k_j}(H over free)(V_j / 2 l2)   (one CTA per node)
//   bound_j = -F*_j - 2 l2 g*_j
//
// One C-ABI call certifies a whole batch of branch-and-bound nodes in fp64:
// each X tile is read once for all nb nodes (the per-node call reads X twice
// per node and syncs the host each time).  The two passes are one tiled fp64
// kernel (k_mrhs): 128 x 64 output tiles, 16-deep k slices staged in shared
// memory (X widened to fp64 once per tile), 8 x 4 outputs per thread in
// registers, fixed-order split-K partials reduced by k_split_sum -- every
// bound is deterministic run to run and equals the per-node bound up to the
// summation order of the two matvecs.

#include "engine.cuh"
#include "prox.cuh"

namespace l0 {

constexpr int kMrBM = 128, kMrBN = 64, kMrBK = 16, kMrThreads = 256;
constexpr int kMrAs = kMrBM + 2;   // padded row (doubles) of the A slice
constexpr int kMrBs = kMrBN + 2;

// part[s][j][m] = sum_{k in slice s} A(m, k) * Bv(j, k)
//   TRANS = false: A(m, k) = X[m ld + k] (m < n rows, k < p), Bv(j, k) = V[j ldv + k]
//   TRANS = true:  A(m, k) = X[k ld + m] (m < p cols, k < n), Bv(j, k) = V[j ldv + k]
template <typename TX, bool TRANS>
__global__ void __launch_bounds__(kMrThreads) k_mrhs(const TX* __restrict__ X, int64_t ld, int64_t M,
                                                     int64_t K, const double* __restrict__ V, int64_t ldv,
                                                     int nb, int64_t kchunk, double* __restrict__ part) {
  __shared__ __align__(16) double As[kMrBK][kMrAs];
  __shared__ __align__(16) double Bs[kMrBK][kMrBs];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;       // 16 x 16 threads: 8 rows x 4 nodes each
  const int64_t m0 = (int64_t)blockIdx.x * kMrBM;
  const int j0 = blockIdx.y * kMrBN;
  const int s = blockIdx.z;
  const int64_t kb = (int64_t)s * kchunk, ke = min(K, kb + kchunk);
  double acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[i][c] = 0.0;
  for (int64_t k0 = kb; k0 < ke; k0 += kMrBK) {
    // A slice: kMrBK x kMrBM
    for (int e = tid; e < kMrBK * kMrBM; e += kMrThreads) {
      int kk, mm;
      if (TRANS) { kk = e / kMrBM; mm = e % kMrBM; }   // consecutive threads along m (a row of X)
      else { mm = e / kMrBK; kk = e % kMrBK; }         // consecutive threads along k (a row of X)
      const int64_t m = m0 + mm, k = k0 + kk;
      double v = 0.0;
      if (m < M && k < ke) v = (double)(TRANS ? X[k * ld + m] : X[m * ld + k]);
      As[kk][mm] = v;
    }
    // B slice: kMrBK x kMrBN (node rows of V are contiguous along k)
    for (int e = tid; e < kMrBK * kMrBN; e += kMrThreads) {
      const int jj = e / kMrBK, kk = e % kMrBK;
      const int j = j0 + jj;
      const int64_t k = k0 + kk;
      Bs[kk][jj] = (j < nb && k < ke) ? V[(int64_t)j * ldv + k] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < kMrBK; ++kk) {
      double a[8], b[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = As[kk][tx + 16 * i];
#pragma unroll
      for (int c = 0; c < 4; ++c) b[c] = Bs[kk][ty + 16 * c];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[i][c] = fma(a[i], b[c], acc[i][c]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int j = j0 + ty + 16 * c;
    if (j >= nb) continue;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t m = m0 + tx + 16 * i;
      if (m < M) part[((int64_t)s * nb + j) * M + m] = acc[i][c];
    }
  }
}

// out[j][m] = sum_s part[s][j][m]  (fixed order)
__global__ void k_split_sum(const double* __restrict__ part, int64_t M, int nb, int S, double* __restrict__ out) {
  const int64_t total = M * nb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int s = 0; s < S; ++s) v += part[(int64_t)s * total + e];
    out[e] = v;
  }
}

// zeta_j = -grad F(u_j) in place, F*(-zeta_j) -> out[j]   (block j)
__global__ void __launch_bounds__(1024) k_loss_conj_b(int loss, double* __restrict__ UZ,
                                                      const double* __restrict__ y, int64_t n,
                                                      double* __restrict__ out) {
  __shared__ double red[32];
  double* z = UZ + (int64_t)blockIdx.x * n;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double zi = -loss_grad(loss, z[i], y[i]);
    z[i] = zi;
    conj_accumulate(loss, zi, y[i], acc);
  }
  acc[0] = block_sum(acc[0], red);
  acc[1] = block_sum(acc[1], red);
  acc[2] = block_sum(acc[2], red);
  if (threadIdx.x == 0) out[blockIdx.x] = conj_finish(loss, acc);
}

// H_M(v / 2 l2) on free coordinates, -1 elsewhere   (all nodes)
__global__ void k_huber_free_b(const double* __restrict__ V, int64_t p, int nb, double div, double M,
                               const uint8_t* __restrict__ cls, double* __restrict__ vals) {
  const int64_t total = p * nb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = cls ? cls[e] : FREE;
    vals[e] = c == FREE ? huber(ddiv(V[e], div), M) : -1.0;
  }
}

// g*_j = sum_{fixed-one} H + TopSum_{k_j}(free H), bound_j = -F*_j - 2 l2 g*_j   (block j)
__global__ void __launch_bounds__(1024) k_bound_final_b(const double* __restrict__ V,
                                                        const double* __restrict__ vals, int64_t p,
                                                        const int64_t* __restrict__ kfree, double div,
                                                        double M, const uint8_t* __restrict__ cls,
                                                        const double* __restrict__ fstar,
                                                        double* __restrict__ out) {
  __shared__ SelectSmem sel;
  __shared__ double red[32];
  const int j = blockIdx.x;
  const double* v = V + (int64_t)j * p;
  const double* h = vals + (int64_t)j * p;
  const uint8_t* c = cls ? cls + (int64_t)j * p : nullptr;
  double fsum = 0.0, nfree = 0.0;
  for (int64_t i = threadIdx.x; i < p; i += blockDim.x) {
    const int ci = c ? c[i] : FREE;
    if (ci == FIXED_ONE) fsum += huber(ddiv(v[i], div), M);
    nfree += ci == FREE ? 1.0 : 0.0;
  }
  fsum = block_sum(fsum, red);
  const int64_t nf = (int64_t)block_sum(nfree, red);
  const double top = block_topk_sum(h, p, kfree[j], nf, sel, red);
  if (threadIdx.x == 0) {
    const double fs = fstar[j];
    const double gs = c ? dadd(fsum, top) : top;
    out[j] = isfinite(fs) ? dsub(-fs, dmul(div, gs)) : -CUDART_INF;   // host order of the per-node call
  }
}

// workspace: U/Z (nb n) | V (nb p) | split partials (S nb max(n, p)) | vals (nb p) | k (nb) | fstar, out (2 nb)
struct BbWs {
  double *uz, *v, *part, *vals, *fstar, *out;
  int64_t* kf;
};

static int bb_splits(int64_t M, int64_t K, int nb, int sms) {
  const int64_t tiles = ((M + kMrBM - 1) / kMrBM) * ((nb + kMrBN - 1) / kMrBN);
  int S = (int)std::max<int64_t>(1, (2 * sms + tiles - 1) / tiles);
  S = (int)std::min<int64_t>(S, std::max<int64_t>(1, K / (4 * kMrBK)));   // >= 4 slices per split
  return std::min(S, 64);
}

static uint64_t bb_carve(int64_t n, int64_t p, int nb, int S, char* base, BbWs* w) {
  uint64_t off = 0;
  auto take = [&](uint64_t bytes) -> char* {
    off = (off + 255) & ~uint64_t(255);
    char* r = base ? base + off : nullptr;
    off += bytes;
    return r;
  };
  BbWs t{};
  t.uz = (double*)take(8ull * nb * n);
  t.v = (double*)take(8ull * nb * p);
  t.part = (double*)take(8ull * S * nb * std::max(n, p));
  t.vals = (double*)take(8ull * nb * p);
  t.kf = (int64_t*)take(8ull * nb);
  t.fstar = (double*)take(8ull * nb);
  t.out = (double*)take(8ull * nb);
  if (w) *w = t;
  return off + 256;
}

static int bb_sms() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

template <typename TX>
static cudaError_t bb_pass(const EngineArgs& a, bool trans, const double* V, int64_t ldv, int nb, int S,
                           double* part, double* out, cudaStream_t s) {
  const int64_t M = trans ? a.p : a.n, K = trans ? a.n : a.p;
  int64_t kchunk = (K + S - 1) / S;
  kchunk = ((kchunk + kMrBK - 1) / kMrBK) * kMrBK;
  const int Sx = (int)((K + kchunk - 1) / kchunk);
  dim3 grid((unsigned)((M + kMrBM - 1) / kMrBM), (unsigned)((nb + kMrBN - 1) / kMrBN), (unsigned)Sx);
  double* dst = Sx == 1 ? out : part;
  if (trans)
    k_mrhs<TX, true><<<grid, kMrThreads, 0, s>>>(static_cast<const TX*>(a.X), a.ld, M, K, V, ldv, nb, kchunk, dst);
  else
    k_mrhs<TX, false><<<grid, kMrThreads, 0, s>>>(static_cast<const TX*>(a.X), a.ld, M, K, V, ldv, nb, kchunk, dst);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || Sx == 1) return e;
  k_split_sum<<<(unsigned)std::min<int64_t>(4096, (M * nb + 255) / 256), 256, 0, s>>>(part, M, nb, Sx, out);
  return cudaGetLastError();
}

}  // namespace l0

extern "C" {

int32_t l0_safe_lower_bound_batched_workspace(l0_problem* P, int64_t nb, uint64_t* bytes) {
  if (!P || !bytes || nb < 1 || nb > INT32_MAX) return set_error(ST_INVALID, "bad arguments");
  const int sms = bb_sms();
  const int S = std::max(bb_splits(P->a.n, P->a.p, (int)nb, sms), bb_splits(P->a.p, P->a.n, (int)nb, sms));
  *bytes = bb_carve(P->a.n, P->a.p, (int)nb, S, nullptr, nullptr);
  return ST_OK;
}

// perspective.py:162-190 for nb nodes at once
int32_t l0_safe_lower_bound_batched(l0_problem* P, const double* d_betas, int64_t nb, const int64_t* h_k_free,
                                    double M, double lambda2, const uint8_t* d_node_class, double* h_out,
                                    void* d_ws, uint64_t ws_bytes, void* stream) {
  int rc = problem_ready(P);
  if (rc) return rc;
  if (nb < 1 || nb > INT32_MAX || !d_betas || !h_k_free || !h_out || !d_ws)
    return set_error(ST_INVALID, "bad arguments");
  const EngineArgs& a = P->a;
  const int sms = bb_sms();
  const int nbi = (int)nb;
  const int S1 = bb_splits(a.n, a.p, nbi, sms), S2 = bb_splits(a.p, a.n, nbi, sms);
  const int S = std::max(S1, S2);
  if (ws_bytes < bb_carve(a.n, a.p, nbi, S, nullptr, nullptr)) return set_error(ST_INVALID, "workspace too small");
  BbWs w;
  bb_carve(a.n, a.p, nbi, S, (char*)d_ws, &w);
  cudaStream_t s = (cudaStream_t)stream;
  OPS_CUDA(cudaMemcpyAsync(w.kf, h_k_free, 8 * (size_t)nb, cudaMemcpyHostToDevice, s));
  const bool f64 = a.dtype == F64;
  // U = X B^T
  OPS_CUDA(f64 ? bb_pass<double>(a, false, d_betas, a.p, nbi, S1, w.part, w.uz, s)
               : bb_pass<float>(a, false, d_betas, a.p, nbi, S1, w.part, w.uz, s));
  k_loss_conj_b<<<nbi, 1024, 0, s>>>(a.loss, w.uz, a.y, a.n, w.fstar);
  OPS_CUDA(cudaGetLastError());
  // V = X^T Z
  OPS_CUDA(f64 ? bb_pass<double>(a, true, w.uz, a.n, nbi, S2, w.part, w.v, s)
               : bb_pass<float>(a, true, w.uz, a.n, nbi, S2, w.part, w.v, s));
  const double two_l2 = 2.0 * lambda2;
  k_huber_free_b<<<grid_for(a.p * nb), 256, 0, s>>>(w.v, a.p, nbi, two_l2, M, d_node_class, w.vals);
  k_bound_final_b<<<nbi, 1024, 0, s>>>(w.v, w.vals, a.p, w.kf, two_l2, M, d_node_class, w.fstar, w.out);
  OPS_CUDA(cudaGetLastError());
  OPS_CUDA(cudaMemcpyAsync(h_out, w.out, 8 * (size_t)nb, cudaMemcpyDeviceToHost, s));
  OPS_CUDA(cudaStreamSynchronize(s));
  return ST_OK;
}

}  // extern "C"
