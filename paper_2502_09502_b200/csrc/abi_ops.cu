// C ABI of the standalone operators (prox.py, perspective.py, model.py entry
// points) and of the problem-level matvec / power iteration / safe bound.

#include <cmath>
#include <cstring>

#include <cub/device/device_radix_sort.cuh>

#include "engine.cuh"
#include "prox.cuh"

namespace l0 {

struct OpsWs {
  double *key, *xs, *tail, *absb, *sorted, *small;
  int *perm, *iota, *flags;
  void* sort_tmp;
  size_t sort_bytes;
};

static size_t ops_sort_bytes(int64_t len) {
  size_t a = 0, b = 0;
  const int m = (int)std::max<int64_t>(len, 1);
  cub::DeviceRadixSort::SortPairsDescending<double, int>(nullptr, a, (const double*)nullptr,
                                                         (double*)nullptr, (const int*)nullptr,
                                                         (int*)nullptr, m);
  cub::DeviceRadixSort::SortKeysDescending<double>(nullptr, b, (const double*)nullptr,
                                                   (double*)nullptr, m);
  return std::max(a, b);
}

static uint64_t ops_carve(int64_t len, char* base, OpsWs* w) {
  uint64_t off = 0;
  auto take = [&](uint64_t bytes) -> char* {
    off = (off + 255) & ~uint64_t(255);
    char* r = base ? base + off : nullptr;
    off += bytes;
    return r;
  };
  const uint64_t L = (uint64_t)std::max<int64_t>(len, 1);
  OpsWs t{};
  t.key = (double*)take(8 * L);
  t.xs = (double*)take(8 * L);
  t.tail = (double*)take(8 * L);
  t.absb = (double*)take(8 * L);
  t.sorted = (double*)take(8 * L);
  t.small = (double*)take(8 * 64);
  t.perm = (int*)take(4 * L);
  t.iota = (int*)take(4 * L);
  t.flags = (int*)take(64);
  t.sort_bytes = ops_sort_bytes(len);
  t.sort_tmp = take(t.sort_bytes);
  if (w) *w = t;
  return off + 256;
}

static int grid_for(int64_t len) { return (int)std::max<int64_t>(1, std::min<int64_t>((len + 255) / 256, 1024)); }

int set_error(int code, const std::string& msg);

}  // namespace l0

using namespace l0;

#define OPS_CUDA(expr)                                                                \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess)                                                            \
      return set_error(ST_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));  \
  } while (0)

static int ops_ws(int64_t len, void* d_ws, uint64_t bytes, OpsWs* w) {
  if (!d_ws) return set_error(ST_INVALID, "workspace is null");
  if (bytes < ops_carve(len, nullptr, nullptr)) return set_error(ST_INVALID, "workspace too small");
  ops_carve(len, (char*)d_ws, w);
  return ST_OK;
}

extern "C" {

int32_t l0_ops_workspace_bytes(int64_t len, uint64_t* bytes) {
  if (!bytes) return set_error(ST_INVALID, "null argument");
  *bytes = ops_carve(len, nullptr, nullptr);
  return ST_OK;
}

int32_t l0_prox(const double* d_in, int64_t p, double rho, int64_t k, double M,
                const uint8_t* d_node_class, int32_t g_mode, double* d_out, int32_t* d_perm_out,
                int64_t* h_pool_out, void* d_ws, uint64_t ws_bytes, void* stream) {
  if (p < 0 || !d_out || (p > 0 && !d_in)) return set_error(ST_INVALID, "bad arguments");
  if (p == 0) return ST_OK;
  if (p > (int64_t)INT32_MAX - 4096) return set_error(ST_INVALID, "p too large");
  OpsWs w;
  int rc = ops_ws(p, d_ws, ws_bytes, &w);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  k_prox_keys<<<grid_for(p), 256, 0, s>>>(d_in, p, rho, g_mode, d_node_class, w.key, w.iota);
  OPS_CUDA(cudaGetLastError());
  PostArgs q{};
  q.p = p;
  q.nf = d_node_class ? -1 : p;
  q.kk = k;
  q.kg = 0;
  q.rho = rho;
  q.M = M;
  q.xs = w.xs;
  q.perm = w.perm;
  q.tail = w.tail;
  q.in = d_in;
  q.out = d_out;
  q.absb = w.absb;
  q.mask = d_node_class;
  q.fone = nullptr;
  q.n_fone = 0;
  q.gmode = g_mode;
  q.want_g = 0;
  q.g_out = nullptr;
  q.st = nullptr;
  int64_t* d_pool = reinterpret_cast<int64_t*>(w.small);
  if (p <= 16384) {
    size_t smem;
    if (p <= 1024) {
      smem = sizeof(ProxSmem) + sizeof(typename cub::BlockRadixSort<double, 256, 4, int, 6>::TempStorage);
      OPS_CUDA(cudaFuncSetAttribute(k_prox_op_block<256, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_prox_op_block<256, 4><<<1, 256, smem, s>>>(q, w.key, d_pool);
    } else if (p <= 4096) {
      smem = sizeof(ProxSmem) + sizeof(typename cub::BlockRadixSort<double, 512, 8, int, 6>::TempStorage);
      OPS_CUDA(cudaFuncSetAttribute(k_prox_op_block<512, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_prox_op_block<512, 8><<<1, 512, smem, s>>>(q, w.key, d_pool);
    } else {
      smem = sizeof(ProxSmem) + sizeof(typename cub::BlockRadixSort<double, 1024, 16, int, 6>::TempStorage);
      OPS_CUDA(cudaFuncSetAttribute(k_prox_op_block<1024, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_prox_op_block<1024, 16><<<1, 1024, smem, s>>>(q, w.key, d_pool);
    }
    OPS_CUDA(cudaGetLastError());
  } else {
    size_t bytes = w.sort_bytes;
    OPS_CUDA(cub::DeviceRadixSort::SortPairsDescending(w.sort_tmp, bytes, w.key, w.xs, w.iota,
                                                       w.perm, (int)p, 0, 64, s));
    const size_t smem = sizeof(ProxSmem);
    OPS_CUDA(cudaFuncSetAttribute(k_prox_op_post, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_prox_op_post<<<1, 1024, smem, s>>>(q, d_pool);
    OPS_CUDA(cudaGetLastError());
  }
  if (d_perm_out)
    OPS_CUDA(cudaMemcpyAsync(d_perm_out, w.perm, 4 * (size_t)p, cudaMemcpyDeviceToDevice, s));
  if (h_pool_out) {
    OPS_CUDA(cudaMemcpyAsync(h_pool_out, d_pool, 16, cudaMemcpyDeviceToHost, s));
    OPS_CUDA(cudaStreamSynchronize(s));
  }
  return ST_OK;
}

int32_t l0_g_value(const double* d_beta, int64_t p, int64_t k_free, double M,
                   const uint8_t* d_node_class, const int32_t* d_fixed_one, int64_t n_fixed_one,
                   double* h_out, void* d_ws, uint64_t ws_bytes, void* stream) {
  if (!h_out) return set_error(ST_INVALID, "bad arguments");
  if (p == 0) { *h_out = 0.0; return ST_OK; }
  OpsWs w;
  int rc = ops_ws(p, d_ws, ws_bytes, &w);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  OPS_CUDA(cudaMemsetAsync(w.flags, 0, 8, s));
  k_abs_free<<<grid_for(p), 256, 0, s>>>(d_beta, p, d_node_class, M, w.absb, w.flags);
  OPS_CUDA(cudaGetLastError());
  size_t bytes = w.sort_bytes;
  OPS_CUDA(cub::DeviceRadixSort::SortKeysDescending(w.sort_tmp, bytes, w.absb, w.sorted, (int)p, 0, 64, s));
  k_g_value_final<<<1, 1024, 0, s>>>(w.sorted, p, d_node_class ? -1 : p, k_free, M, d_beta,
                                     d_node_class ? (const int*)d_fixed_one : nullptr,
                                     n_fixed_one, w.flags, w.small);
  OPS_CUDA(cudaGetLastError());
  OPS_CUDA(cudaMemcpyAsync(h_out, w.small, 8, cudaMemcpyDeviceToHost, s));
  OPS_CUDA(cudaStreamSynchronize(s));
  return ST_OK;
}

int32_t l0_g_conjugate(const double* d_alpha, int64_t p, int64_t k_free, double M,
                       const uint8_t* d_node_class, double* h_out, void* d_ws, uint64_t ws_bytes,
                       void* stream) {
  if (!h_out) return set_error(ST_INVALID, "bad arguments");
  if (p == 0) { *h_out = 0.0; return ST_OK; }
  OpsWs w;
  int rc = ops_ws(p, d_ws, ws_bytes, &w);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  k_huber_free<<<grid_for(p), 256, 0, s>>>(d_alpha, p, 1.0, M, d_node_class, w.absb);
  k_g_conj_final<<<1, 1024, 0, s>>>(d_alpha, w.absb, p, k_free, d_node_class ? -1 : p, 1.0, M,
                                    d_node_class, w.small);
  OPS_CUDA(cudaGetLastError());
  OPS_CUDA(cudaMemcpyAsync(h_out, w.small, 8, cudaMemcpyDeviceToHost, s));
  OPS_CUDA(cudaStreamSynchronize(s));
  return ST_OK;
}

int32_t l0_huber(const double* d_x, int64_t n, double w, double M, int32_t prox, double* d_out,
                 void* stream) {
  if (n <= 0) return ST_OK;
  k_huber_elem<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(d_x, n, w, M, prox, d_out);
  OPS_CUDA(cudaGetLastError());
  return ST_OK;
}

int32_t l0_loss_value(int32_t loss, const double* d_u, const double* d_y, int64_t n,
                      double* h_value, double* d_grad, int32_t* h_nonfinite, void* d_ws,
                      uint64_t ws_bytes, void* stream) {
  if (loss < 0 || loss > 4) return set_error(ST_UNSUPPORTED, "loss not evaluated by the engine");
  OpsWs w;
  int rc = ops_ws(1, d_ws, ws_bytes, &w);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  k_loss_eval<<<1, 1024, 0, s>>>(loss, d_u, d_y, n, d_grad, w.small);
  OPS_CUDA(cudaGetLastError());
  double out[2];
  OPS_CUDA(cudaMemcpyAsync(out, w.small, 16, cudaMemcpyDeviceToHost, s));
  OPS_CUDA(cudaStreamSynchronize(s));
  if (h_value) *h_value = out[0];
  if (h_nonfinite) *h_nonfinite = out[1] > 0.0 ? 1 : 0;
  return ST_OK;
}

int32_t l0_loss_conjugate(int32_t loss, const double* d_zeta, const double* d_y, int64_t n,
                          double* h_out, void* d_ws, uint64_t ws_bytes, void* stream) {
  if (loss < 0 || loss > 4) return set_error(ST_UNSUPPORTED, "loss not evaluated by the engine");
  OpsWs w;
  int rc = ops_ws(1, d_ws, ws_bytes, &w);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  k_loss_conj<<<1, 1024, 0, s>>>(loss, d_zeta, d_y, n, 0, nullptr, w.small);
  OPS_CUDA(cudaGetLastError());
  OPS_CUDA(cudaMemcpyAsync(h_out, w.small, 8, cudaMemcpyDeviceToHost, s));
  OPS_CUDA(cudaStreamSynchronize(s));
  return ST_OK;
}

int32_t l0_all_finite(const void* d_x, int32_t dtype, int64_t rows, int64_t cols, int64_t ld,
                      int32_t* h_ok, void* d_ws, uint64_t ws_bytes, void* stream) {
  OpsWs w;
  int rc = ops_ws(1, d_ws, ws_bytes, &w);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  OPS_CUDA(cudaMemsetAsync(w.flags, 0, 4, s));
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((rows * cols + 255) / 256, 148 * 16));
  if (dtype == F64) k_all_finite<double><<<blocks, 256, 0, s>>>((const double*)d_x, rows, cols, ld, w.flags);
  else k_all_finite<float><<<blocks, 256, 0, s>>>((const float*)d_x, rows, cols, ld, w.flags);
  OPS_CUDA(cudaGetLastError());
  int bad = 0;
  OPS_CUDA(cudaMemcpyAsync(&bad, w.flags, 4, cudaMemcpyDeviceToHost, s));
  OPS_CUDA(cudaStreamSynchronize(s));
  *h_ok = bad ? 0 : 1;
  return ST_OK;
}

// ---- problem-level ops -----------------------------------------------------------
static int problem_ready(l0_problem* P, bool local_ok = false) {
  if (!P) return set_error(ST_INVALID, "null problem");
  if (!P->ws) return set_error(ST_INVALID, "problem has no workspace");
  // matvecs act on this rank's rows; global reductions are the caller's
  if (P->a.multi && !local_ok)
    return set_error(ST_UNSUPPORTED, "operator needs a global reduction in row-sharded mode");
  return ST_OK;
}

static int plain_k1(l0_problem* P, const double* v, double* out, cudaStream_t s) {
  EngineArgs a = P->a;
  a.in_vec = v;
  a.out_vec = out;
  OPS_CUDA(launch_k1(a, MODE_PLAIN, s));
  return ST_OK;
}

static int plain_k2(l0_problem* P, const double* r, double* out, cudaStream_t s) {
  EngineArgs a = P->a;
  a.in_vec = r;
  a.out_vec = out;
  a.plain_rhs2 = 1;
  OPS_CUDA(launch_k2(a, MODE_PLAIN, s));
  return ST_OK;
}

int32_t l0_matvec(l0_problem* P, const double* d_v, double* d_out, void* stream) {
  int rc = problem_ready(P, true);
  if (rc) return rc;
  return plain_k1(P, d_v, d_out, (cudaStream_t)stream);
}

int32_t l0_rmatvec(l0_problem* P, const double* d_r, double* d_out, void* stream) {
  int rc = problem_ready(P, true);
  if (rc) return rc;
  return plain_k2(P, d_r, d_out, (cudaStream_t)stream);
}

// model.py:283-306 (the caller passes the normalised seed-0 start vector)
int32_t l0_power_iteration(l0_problem* P, const double* d_v0, double tol, int64_t max_iter,
                           double* h_lambda, int64_t* h_iterations, void* stream) {
  int rc = problem_ready(P);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  EngineArgs& a = P->a;
  double* v = P->d_vec_p;
  double* w = P->d_vec_n;
  double* sm = P->d_small;
  OPS_CUDA(cudaMemcpyAsync(v, d_v0, 8 * (size_t)a.p, cudaMemcpyDeviceToDevice, s));
  double prev = INFINITY;
  for (int64_t it = 0; it < max_iter; ++it) {
    if ((rc = plain_k1(P, v, w, s))) return rc;
    k_sqnorm<<<1, 1024, 0, s>>>(w, a.n, sm);
    if ((rc = plain_k2(P, w, v, s))) return rc;
    k_sqnorm<<<1, 1024, 0, s>>>(v, a.p, sm + 1);
    k_scale_div<<<grid_for(a.p), 256, 0, s>>>(v, a.p, sm + 1);
    OPS_CUDA(cudaGetLastError());
    double hv[2];
    OPS_CUDA(cudaMemcpyAsync(hv, sm, 16, cudaMemcpyDeviceToHost, s));
    OPS_CUDA(cudaStreamSynchronize(s));
    const double lam = hv[0];
    if (h_iterations) *h_iterations = it + 1;
    if (lam == 0.0 || hv[1] == 0.0) { *h_lambda = 0.0; return ST_OK; }
    if (std::fabs(lam - prev) <= tol * lam) { *h_lambda = lam; return ST_OK; }
    prev = lam;
  }
  *h_lambda = prev;
  return set_error(ST_NUMERICAL, "power iteration did not converge within " +
                                     std::to_string(max_iter) + " iterations");
}

// perspective.py:162-190
int32_t l0_safe_lower_bound(l0_problem* P, const double* d_beta, int64_t k_free, double M,
                            double lambda2, const uint8_t* d_node_class, double* h_out,
                            void* stream) {
  int rc = problem_ready(P);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  EngineArgs& a = P->a;
  double* u = P->d_vec_n;
  double* v = P->d_vec_p;
  double* sm = P->d_small;
  if ((rc = plain_k1(P, d_beta, u, s))) return rc;                       // u = X beta
  k_loss_conj<<<1, 1024, 0, s>>>(a.loss, u, a.y, a.n, 1, u, sm);          // zeta, F*(-zeta)
  OPS_CUDA(cudaGetLastError());
  if ((rc = plain_k2(P, u, v, s))) return rc;                            // v = X^T zeta
  const double two_l2 = 2.0 * lambda2;
  k_huber_free<<<grid_for(a.p), 256, 0, s>>>(v, a.p, two_l2, M, d_node_class, a.scratch);
  k_g_conj_final<<<1, 1024, 0, s>>>(v, a.scratch, a.p, k_free, d_node_class ? -1 : a.p, two_l2, M,
                                    d_node_class, sm + 1);
  OPS_CUDA(cudaGetLastError());
  double hv[2];
  OPS_CUDA(cudaMemcpyAsync(hv, sm, 16, cudaMemcpyDeviceToHost, s));
  OPS_CUDA(cudaStreamSynchronize(s));
  if (!std::isfinite(hv[0])) { *h_out = -INFINITY; return ST_OK; }
  *h_out = -hv[0] - two_l2 * hv[1];
  return ST_OK;
}

}  // extern "C"
