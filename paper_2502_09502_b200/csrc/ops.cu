// Standalone operator kernels behind the reference's operator API
// (prox.py:134-201, perspective.py:114-190, model.py:159-306).  The FISTA
// engine fuses the same device functions into its iteration kernels.

#include "control.cuh"
#include "engine.cuh"
#include "prox.cuh"

namespace l0 {

// keys |mu| (mu = rho*in for prox_g) ; fixed coordinates -> -1
__global__ void k_prox_keys(const double* in, int64_t p, double rho, int gmode,
                            const uint8_t* mask, double* key, int* iota) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < p;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double mu = gmode ? dmul(rho, in[j]) : in[j];
    const bool fixed = mask != nullptr && mask[j] != FREE;
    key[j] = fixed ? -1.0 : fabs(mu);
    iota[j] = (int)j;
  }
}

template <int T, int IPT>
__global__ void __launch_bounds__(T, 1) k_prox_op_block(PostArgs q, const double* key,
                                                       int64_t* pool_out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using Sort = cub::BlockRadixSort<double, T, IPT, int, 6>;
  ProxSmem& sm = *reinterpret_cast<ProxSmem*>(smem_raw);
  typename Sort::TempStorage& tmp =
      *reinterpret_cast<typename Sort::TempStorage*>(smem_raw + sizeof(ProxSmem));
  double keys[IPT];
  int ids[IPT];
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int j = threadIdx.x * IPT + i;
    keys[i] = j < q.p ? key[j] : -CUDART_INF;
    ids[i] = j;
  }
  Sort(tmp).SortDescending(keys, ids);
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int pos = threadIdx.x * IPT + i;
    if (pos < q.p) {
      const_cast<double*>(q.xs)[pos] = keys[i];
      const_cast<int*>(q.perm)[pos] = ids[i];
    }
  }
  __syncthreads();
  prox_post_sort<T>(q, sm);
  if (threadIdx.x == 0 && pool_out != nullptr) {
    pool_out[0] = sm.found > 0 ? sm.astar : -1;
    pool_out[1] = sm.found > 0 ? sm.cstar : -1;
  }
}

__global__ void __launch_bounds__(1024, 1) k_prox_op_post(PostArgs q, int64_t* pool_out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ProxSmem& sm = *reinterpret_cast<ProxSmem*>(smem_raw);
  prox_post_sort<1024>(q, sm);
  if (threadIdx.x == 0 && pool_out != nullptr) {
    pool_out[0] = sm.found > 0 ? sm.astar : -1;
    pool_out[1] = sm.found > 0 ? sm.cstar : -1;
  }
}

// |beta| over free coordinates (-1 elsewhere) + node feasibility flags
// (perspective.py:119-129): flags[0] fixed-zero violation, flags[1] fixed-one box
__global__ void k_abs_free(const double* beta, int64_t p, const uint8_t* mask, double M,
                           double* vals, int* flags) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < p;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int cls = mask ? mask[j] : FREE;
    const double ab = fabs(beta[j]);
    vals[j] = cls == FREE ? ab : -1.0;
    if (cls == FIXED_ZERO && ab > kZeroAtol) atomicOr(flags, 1);
    if (cls == FIXED_ONE && ab > dmul(M, dadd(1.0, kFeasRtol))) atomicOr(flags + 1, 1);
  }
}

// g from free magnitudes sorted descending (negatives at the end); nf < 0:
// count the free entries first
__global__ void __launch_bounds__(1024) k_g_value_final(const double* sorted, int64_t p,
                                                        int64_t nf, int64_t kg, double M,
                                                        const double* beta, const int* fone,
                                                        int64_t n_fone, const int* flags,
                                                        double* out) {
  __shared__ double red[32];
  __shared__ double s_gfree;
  if (nf < 0) {
    double c = 0.0;
    for (int64_t i = threadIdx.x; i < p; i += blockDim.x) c += sorted[i] >= 0.0 ? 1.0 : 0.0;
    nf = (int64_t)block_sum(c, red);
  }
  double total = 0.0;
  for (int64_t i = threadIdx.x; i < nf; i += blockDim.x) total += sorted[i];
  total = block_sum(total, red);
  const double amax = nf > 0 ? sorted[0] : 0.0;
  int path = 0;
  double gfree = 0.0;
  if (nf == 0) path = 2;
  else if (amax > dmul(M, dadd(1.0, kFeasRtol))) { gfree = CUDART_INF; path = 2; }
  else if (total > dmul(dmul((double)kg, M), dadd(1.0, kFeasRtol))) { gfree = CUDART_INF; path = 2; }
  else if (kg == 0) path = 2;
  if (path == 0) {
    const int64_t kkg = kg < nf ? kg : nf;
    if (threadIdx.x < 32) {
      const double g = envelope_from_top(sorted, kkg, total);
      if (threadIdx.x == 0) s_gfree = g;
    }
    __syncthreads();
    gfree = s_gfree;
  }
  if (threadIdx.x == 0) {
    double g;
    if (flags[0] || flags[1]) {
      g = CUDART_INF;
    } else if (fone == nullptr) {
      g = gfree;
    } else {
      double s2 = 0.0;
      for (int64_t i = 0; i < n_fone; ++i) s2 = fma(beta[fone[i]], beta[fone[i]], s2);
      g = dadd(dadd(0.0, dmul(0.5, s2)), gfree);
    }
    *out = g;
  }
}

// Huber values of alpha = in / div over free coordinates (-1 elsewhere)
__global__ void k_huber_free(const double* in, int64_t p, double div, double M,
                             const uint8_t* mask, double* vals) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < p;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double al = div == 1.0 ? in[j] : ddiv(in[j], div);
    const int cls = mask ? mask[j] : FREE;
    vals[j] = cls == FREE ? huber(al, M) : -1.0;
  }
}

// g*(alpha) = sum_{fixed-one} H + TopSum_{kg}(H over free)  (perspective.py:143-159)
__global__ void __launch_bounds__(1024) k_g_conj_final(const double* in, const double* vals,
                                                       int64_t p, int64_t kg, int64_t nf,
                                                       double div, double M,
                                                       const uint8_t* mask, double* out) {
  __shared__ SelectSmem sel;
  __shared__ double red[32];
  double fsum = 0.0;
  if (mask) {
    for (int64_t j = threadIdx.x; j < p; j += blockDim.x)
      if (mask[j] == FIXED_ONE) fsum += huber(div == 1.0 ? in[j] : ddiv(in[j], div), M);
  }
  fsum = block_sum(fsum, red);
  if (nf < 0) {
    double c = 0.0;
    for (int64_t j = threadIdx.x; j < p; j += blockDim.x) c += vals[j] >= 0.0 ? 1.0 : 0.0;
    nf = (int64_t)block_sum(c, red);
  }
  const double top = block_topk_sum(vals, p, kg, nf, sel, red);
  if (threadIdx.x == 0) *out = mask ? dadd(fsum, top) : top;
}

// F(u) and optionally grad F(u), non-finite detection (model.py:152-218)
__global__ void __launch_bounds__(1024) k_loss_eval(int loss, const double* u, const double* y,
                                                    int64_t n, double* grad, double* out2) {
  __shared__ double red[32];
  double s = 0.0, bad = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double ui = u[i];
    if (!isfinite(ui)) bad = 1.0;
    s += loss_term(loss, ui, y[i]);
    if (grad) grad[i] = loss_grad(loss, ui, y[i]);
  }
  s = block_sum(s, red);
  bad = block_max(bad, red);
  if (threadIdx.x == 0) { out2[0] = s; out2[1] = bad; }
}

// F*(-zeta) (model.py:226-253); zeta_from_u: zeta = -grad F(u) first
__global__ void __launch_bounds__(1024) k_loss_conj(int loss, const double* z_or_u,
                                                    const double* y, int64_t n, int zeta_from_u,
                                                    double* zeta_out, double* out) {
  __shared__ double red[32];
  double acc[3] = {0.0, 0.0, 0.0};
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    double z = z_or_u[i];
    if (zeta_from_u) {
      z = -loss_grad(loss, z, y[i]);
      zeta_out[i] = z;
    }
    conj_accumulate(loss, z, y[i], acc);
  }
  acc[0] = block_sum(acc[0], red);
  acc[1] = block_sum(acc[1], red);
  acc[2] = block_sum(acc[2], red);
  if (threadIdx.x == 0) *out = conj_finish(loss, acc);
}

// ||x||^2 (one CTA, fixed order) and x /= ||x||
__global__ void __launch_bounds__(1024) k_sqnorm(const double* x, int64_t n, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = fma(x[i], x[i], s);
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

__global__ void k_scale_div(double* x, int64_t n, const double* sq) {
  const double nrm = sqrt(*sq);
  if (nrm == 0.0) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] = ddiv(x[i], nrm);
}

// finiteness check of fp64 / fp32 arrays (input validation, model.py:100-101)
template <typename T>
__global__ void k_all_finite(const T* x, int64_t rows, int64_t cols, int64_t ld, int* bad) {
  int b = 0;
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    if (!isfinite((double)x[r * ld + c])) b = 1;
  }
  if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}

// FISTA state initialisation (fista.py:140-148)
__global__ void k_state_init(State* st, double parent_bound) {
  st->t = 0;
  st->restarts = 0;
  st->err_iter = 0;
  st->trace_count = 0;
  st->phi = 1;
  st->done = 0;
  st->termination = TERM_ITERATION_LIMIT;
  st->err = ST_OK;
  st->dual_pending = 0;
  st->check_pending = 0;
  st->dual_only = 0;
  st->stop_term = -1;
  st->last_restarted = 0;
  st->topk_fallbacks = 0;
  st->obj = 0.0;
  st->g_next = 0.0;
  st->best_dual = parent_bound;
  st->gap = CUDART_NAN;
  st->last_dual = CUDART_NAN;
  st->loss_cur = 0.0;
  st->theta = 0.0;
  st->slow_prox = 0;
  st->win_ext = 0;
}

// host-requested stop (time limit, trace-hook abort): fista.py:204-206
__global__ void k_request_stop(State* st, const Params* P, int term) {
  if (st->done) return;
  if (st->check_pending) {
    if (st->stop_term < 0) st->stop_term = term;
    st->dual_only = 1;
  } else {
    request_stop(st, P, term);
  }
}

// elementwise Huber (prox.py:27-32) or its prox (prox.py:35-43)
__global__ void k_huber_elem(const double* x, int64_t n, double w, double M, int prox,
                             double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = prox ? hprox(x[i], w, M) : huber(x[i], M);
}

__global__ void k_iota(int* x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] = (int)i;
}

}  // namespace l0
