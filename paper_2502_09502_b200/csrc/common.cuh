// Shared device-side definitions for the B200 dual-bound engine.
//
// Numerical contract: every elementwise formula
// that the reference evaluates with numpy is evaluated here with one IEEE
// rounding per operation in the same order (the __d*_rn intrinsics are never
// contracted into FMA), so prox inputs, Huber values, losses and the momentum
// step are bit-identical to the reference on identical inputs.  Reductions
// (dot products, sums) use fixed-order trees: results are deterministic
// run-to-run and differ from numpy/OpenBLAS only by summation order.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <math_constants.h>

namespace l0 {

// solver-grade (0..2) and the bound-grade losses the engine evaluates (3, 4;
// model.py:174-177, :196-199, :259-273): they have no global gradient
// Lipschitz constant, so only the bound operations accept them
enum Loss : int { SQUARED_ERROR = 0, LOGISTIC = 1, SQUARED_HINGE = 2, POISSON = 3, GAMMA = 4 };
enum Dtype : int { F64 = 0, F32 = 1 };
enum Status : int {
  ST_OK = 0, ST_INVALID = 1, ST_NUMERICAL = 2, ST_INFEASIBLE = 3, ST_UNSUPPORTED = 4, ST_CUDA = 5,
  // internal: the windowed prox met an exact tie group larger than its window
  // (duplicated columns); the host re-runs the solve on the full key sort
  ST_TIE_OVERFLOW = 7
};
enum Termination : int {
  TERM_CONVERGED = 0, TERM_ITERATION_LIMIT = 1, TERM_TIME_LIMIT = 2,
  TERM_PRIMAL_BELOW = 3, TERM_DUAL_ABOVE = 4
};
// per-coordinate node class (fista.py:109-128)
enum NodeClass : uint8_t { FREE = 0, FIXED_ONE = 1, FIXED_ZERO = 2 };

constexpr double kFeasRtol = 1e-9;     // perspective.py:23
constexpr double kZeroAtol = 1e-9;     // perspective.py:25
constexpr double kDomainSlack = 1e-12; // model.py:39

// ---------------------------------------------------------------------------
// exact (uncontracted) double arithmetic
// ---------------------------------------------------------------------------
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// np.sign: -1, 0, +1 (0 for +-0; NaN never reaches here)
__device__ __forceinline__ double dsign(double x) { return x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0); }

// prox.py:35-43 — argmin_v (v-x)^2/2 + w H_M(v), x >= 0
__device__ __forceinline__ double hprox(double x, double w, double M) {
  double opw = dadd(1.0, w);
  return (x <= dmul(M, opw)) ? ddiv(x, opw) : dsub(x, dmul(w, M));
}

// prox.py:27-32 — Huber H_M(x)
__device__ __forceinline__ double huber(double x, double M) {
  double a = fabs(x);
  return (a <= M) ? dmul(dmul(0.5, x), x) : dsub(dmul(M, a), dmul(dmul(0.5, M), M));
}

// numpy's logaddexp(0, t) (npy_logaddexp with x = 0)
__device__ __forceinline__ double logaddexp0(double t) {
  if (t == 0.0) return 0.6931471805599453;  // x == y: x + log(2)
  double tmp = -t;                          // x - y
  if (tmp > 0.0) return log1p(exp(-tmp));
  return dadd(t, log1p(exp(tmp)));
}

// scipy.special.expit: 1 / (1 + exp(-x))
__device__ __forceinline__ double expit(double x) { return ddiv(1.0, dadd(1.0, exp(-x))); }

// model.py:164-172 — per-sample loss term (summed by the caller)
__device__ __forceinline__ double loss_term(int loss, double u, double y) {
  if (loss == SQUARED_ERROR) { double d = dsub(u, y); return dmul(d, d); }
  if (loss == LOGISTIC) return logaddexp0(dmul(-y, u));
  if (loss == POISSON) return dsub(exp(u), dmul(y, u));           // model.py:174-175
  if (loss == GAMMA) return dadd(dmul(y, exp(-u)), u);            // model.py:176-177
  double m = fmax(0.0, dsub(1.0, dmul(y, u)));
  return dmul(m, m);
}

// model.py:190-195 — dF/du
__device__ __forceinline__ double loss_grad(int loss, double u, double y) {
  if (loss == SQUARED_ERROR) return dmul(2.0, dsub(u, y));
  if (loss == LOGISTIC) return dmul(-y, expit(dmul(-y, u)));
  if (loss == POISSON) return dsub(exp(u), y);                    // model.py:196-197
  if (loss == GAMMA) return dsub(1.0, dmul(y, exp(-u)));          // model.py:198-199
  double m = fmax(0.0, dsub(1.0, dmul(y, u)));
  return dmul(dmul(-2.0, y), m);
}

// fp32-mode loss evaluations (single-pass kernel with fp32_forward): the
// logistic exp / log1p chains in single precision (relative error ~1e-7, the
// fp32 mode's budget is 1e-5); every other loss keeps its fp64 formula.  The
// bound stays safe: F*(-zeta) is evaluated in fp64 for the zeta produced.
__device__ __forceinline__ double loss_grad_f32m(int loss, double u, double y) {
  if (loss != LOGISTIC) return loss_grad(loss, u, y);
  const float t = (float)(y * u);                  // expit(-y u) = 1 / (1 + exp(y u))
  return -y * (double)(1.0f / (1.0f + __expf(t)));
}
__device__ __forceinline__ double loss_term_f32m(int loss, double u, double y) {
  if (loss != LOGISTIC) return loss_term(loss, u, y);
  const float t = (float)(-y * u);                 // logaddexp(0, t)
  return (double)(fmaxf(t, 0.0f) + log1pf(__expf(-fabsf(t))));
}

// xlogy(r, r) with 0 log 0 = 0
__device__ __forceinline__ double xlogx(double r) { return r == 0.0 ? 0.0 : dmul(r, log(r)); }

// F*(-zeta) accumulators (model.py:239-253).  acc[0], acc[1] are sums, acc[2]
// counts out-of-domain samples.  The conjugate is
//   SE:     0.25 * acc0 - acc1   (acc0 = zeta.zeta, acc1 = y.zeta)
//   others: acc0                  (+inf when acc2 > 0)
__device__ __forceinline__ void conj_accumulate(int loss, double zeta, double y, double acc[3]) {
  if (loss == SQUARED_ERROR) {
    acc[0] = dadd(acc[0], dmul(zeta, zeta));
    acc[1] = dadd(acc[1], dmul(y, zeta));
  } else if (loss == LOGISTIC) {
    double r = ddiv(zeta, y);
    if (r < -kDomainSlack || r > dadd(1.0, kDomainSlack)) { acc[2] += 1.0; return; }
    r = fmin(fmax(r, 0.0), 1.0);
    acc[0] = dadd(acc[0], dadd(xlogx(r), xlogx(dsub(1.0, r))));
  } else if (loss == POISSON) {                                   // model.py:259-264
    double z = dsub(y, zeta);
    if (z < -kDomainSlack) { acc[2] += 1.0; return; }
    z = fmax(z, 0.0);
    acc[0] = dadd(acc[0], dsub(xlogx(z), z));
  } else if (loss == GAMMA) {                                     // model.py:266-273
    double z = ddiv(dadd(1.0, zeta), y);
    if (z < -kDomainSlack) { acc[2] += 1.0; return; }
    z = fmax(z, 0.0);
    acc[0] = dadd(acc[0], dmul(y, dsub(xlogx(z), z)));
  } else {
    double z = dmul(-y, zeta);
    if (z > kDomainSlack) { acc[2] += 1.0; return; }
    z = fmin(z, 0.0);
    acc[0] = dadd(acc[0], dadd(z, dmul(dmul(0.25, z), z)));
  }
}

__device__ __forceinline__ double conj_finish(int loss, const double acc[3]) {
  if (acc[2] > 0.0) return CUDART_INF;
  if (loss == SQUARED_ERROR) return dsub(dmul(0.25, acc[0]), acc[1]);
  return acc[0];
}

// ---------------------------------------------------------------------------
// deterministic reductions
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum, fixed order (warp trees, then warp 0 over warp results).
// `scratch` needs blockDim.x/32 doubles; result valid in every thread.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[w] = v;
  __syncthreads();
  if (w == 0) {
    double x = lane < nw ? scratch[lane] : 0.0;
    x = warp_sum(x);
    if (lane == 0) scratch[0] = x;
  }
  __syncthreads();
  double r = scratch[0];
  __syncthreads();
  return r;
}

__device__ __forceinline__ double block_max(double v, double* scratch) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) scratch[w] = v;
  __syncthreads();
  if (w == 0) {
    double x = lane < nw ? scratch[lane] : -CUDART_INF;
    x = warp_max(x);
    if (lane == 0) scratch[0] = x;
  }
  __syncthreads();
  double r = scratch[0];
  __syncthreads();
  return r;
}

// block_sum of four values in one pass (same trees and arithmetic as four
// block_sum calls); `scratch` needs 4 x 32 doubles.
__device__ __forceinline__ void block_sum4(double (&v)[4], double* scratch) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = warp_sum(v[i]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < 4; ++i) scratch[32 * i + w] = v[i];
  __syncthreads();
  if (w == 0) {
    double x[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = warp_sum(lane < nw ? scratch[32 * i + lane] : 0.0);
    __syncwarp();
    if (lane == 0)
#pragma unroll
      for (int i = 0; i < 4; ++i) scratch[32 * i] = x[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = scratch[32 * i];
  __syncthreads();
}

// block_sum(s), block_max(m1), block_max(m2) in one pass: the same trees and
// the same arithmetic as the three calls, three barriers instead of twelve.
// `scratch` needs 3 x 32 doubles.
__device__ __forceinline__ void block_sum_max_max(double& s, double& m1, double& m2, double* scratch) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  s = warp_sum(s);
  m1 = warp_max(m1);
  m2 = warp_max(m2);
  __syncthreads();
  if (lane == 0) {
    scratch[w] = s;
    scratch[32 + w] = m1;
    scratch[64 + w] = m2;
  }
  __syncthreads();
  if (w == 0) {
    double x = lane < nw ? scratch[lane] : 0.0;
    double y = lane < nw ? scratch[32 + lane] : -CUDART_INF;
    double z = lane < nw ? scratch[64 + lane] : -CUDART_INF;
    x = warp_sum(x);
    y = warp_max(y);
    z = warp_max(z);
    __syncwarp();
    if (lane == 0) {
      scratch[0] = x;
      scratch[32] = y;
      scratch[64] = z;
    }
  }
  __syncthreads();
  s = scratch[0];
  m1 = scratch[32];
  m2 = scratch[64];
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Engine-wide structures (device memory)
// ---------------------------------------------------------------------------

// Per-solve scalars, read by the kernels from device memory so one captured
// CUDA graph serves every solve on the same problem.
struct Params {
  double L, rho, two_l2, M;
  double gap_tol, gap_tol_rel;
  double early_primal, early_dual;  // NaN = unset
  double parent_bound;
  int64_t max_iter;
  int64_t k;          // instance k
  int64_t k_rem;      // prox budget over free coordinates: min(k - |F1|, |free|)
  int64_t k_g;        // envelope budget over free coordinates: k - |F1| (unclipped)
  int64_t n_free;     // number of free coordinates
  int64_t n_fone;     // number of fixed-one coordinates
  int bci;
  int restart;
  int stop_on_gap;
  int node_mode;      // 0: trivial node
  int loss;
  int pad_;
};

// Trace record pushed at every bound check (fista.py:185-194)
struct TraceRec {
  double iteration, primal, dual, gap, restarted;
};

constexpr int kTraceCap = 256;

// Iteration state machine (device memory; mirrored to pinned host memory at
// the end of every captured chunk).
struct State {
  int64_t t;              // iterations completed
  int64_t restarts;
  int64_t err_iter;
  int64_t trace_count;    // records ever written (ring index = count % kTraceCap)
  int64_t phi;
  int done;
  int termination;
  int err;                // Status
  int dual_pending;       // a bound evaluation at beta_t is due (K2 adds the zeta column)
  int check_pending;      // ... and it is a bound CHECK (max, gap, trace, tests)
  int dual_only;          // no further iterations: K2 computes zeta only, K3 the bound only
  int stop_term;          // termination applied after the pending check (-1: none)
  int last_restarted;
  int topk_fallbacks;     // diagnostics: g top-k window verification misses
  int win_ext;            // diagnostics: K3 iterations whose pool reached past the candidate window
  int kf_token;           // SPEC: 1 until one of the two single-pass kernels has run this iteration
                          // (the second one would otherwise see the advanced t); KR re-arms it
  double obj;             // composite objective at beta_t
  double g_next;          // g(beta_next) from the prox kernel
  double best_dual;
  double gap;
  double last_dual;
  double loss_cur;
  double theta;           // window-candidate threshold K2 applies (set by K3)
  int64_t slow_prox;      // diagnostics: K3 iterations that needed a full key pass
  long long probe[16];     // clock64 phase stamps of the last K3 (L0_PROBE builds)
  TraceRec trace[kTraceCap];
};

#ifdef L0_PROBE
#define L0_STAMP(st, i) do { if (threadIdx.x == 0) (st)->probe[i] = clock64(); } while (0)
#else
#define L0_STAMP(st, i) do { } while (0)
#endif

}  // namespace l0
