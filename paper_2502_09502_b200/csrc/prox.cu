// K3: exact prox of the perspective term, envelope value g, Fenchel bound.
//
//   sort      stable descending |mu| (prox.py:111)         CUB BlockRadixSort in one CTA
//                                                           (p <= 16384) or CUB onesweep
//   PAVA      single merged pool [a*, c*] straddling k-1|k: tail prefix
//             sums + one warp per candidate a, 32-ary search for c(a)   (prox.py:46-98)
//   scatter   beta+ = gamma - sign*nu/rho, node classes      (fista.py:104-128)
//   g(beta+)  feasibility, top-k via the prox permutation (verified; radix-select fallback),
//             suffix averages                                  (perspective.py:76-132)
//   bound     -F*(-zeta) - 2 l2 TopSum_k(H_M(X^T zeta / 2 l2))  (fista.py:150-157,
//             perspective.py:135-159), radix select for the k-th largest Huber value
//
// Everything after the sort runs in one CTA: p-length work is latency-bound,
// and a single CTA keeps every reduction in a fixed order without grid syncs.

#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>

#include "control.cuh"
#include "engine.cuh"
#include "prox.cuh"

namespace l0 {

// ---------------------------------------------------------------------------
// block-wide k-th largest among non-negative doubles (negative entries are
// excluded).  Radix select on the IEEE bit pattern, 8 bits per pass,
// warp-aggregated shared-memory histograms.
// ---------------------------------------------------------------------------
__device__ void block_kth_largest(const double* vals, int64_t m, int64_t kk, SelectSmem& sm,
                                  double* tau_out, int64_t* cnt_gt_out) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    sm.prefix = 0ull;
    sm.pmask = 0ull;
    sm.remaining = kk;
  }
  __syncthreads();
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += blockDim.x) sm.hist[i] = 0u;
    __syncthreads();
    const unsigned long long prefix = sm.prefix, pmask = sm.pmask;
    const int64_t rounds = (m + blockDim.x - 1) / blockDim.x;
    for (int64_t r = 0; r < rounds; ++r) {
      int64_t i = r * blockDim.x + tid;
      int digit = -1;
      if (i < m) {
        double v = vals[i];
        unsigned long long b = (unsigned long long)__double_as_longlong(v);
        if (v >= 0.0 && (b & pmask) == prefix) digit = (int)((b >> shift) & 255ull);
      }
      unsigned peers = __match_any_sync(0xffffffffu, digit);
      int leader = __ffs(peers) - 1;
      if (digit >= 0 && lane == leader) atomicAdd(&sm.hist[digit], (unsigned)__popc(peers));
    }
    __syncthreads();
    if (warp == 0) {
      // lane l owns bins 255-8l .. 248-8l (descending)
      unsigned cnt[8];
      unsigned s = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) { cnt[q] = sm.hist[255 - (lane * 8 + q)]; s += cnt[q]; }
      unsigned incl = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned excl = incl - s;
      const int64_t rem = sm.remaining;
      const bool mine = (int64_t)excl < rem && rem <= (int64_t)incl;
      if (mine) {
        unsigned cum = excl;
        for (int q = 0; q < 8; ++q) {
          if ((int64_t)(cum + cnt[q]) >= rem) {
            const int d = 255 - (lane * 8 + q);
            sm.remaining = rem - cum;
            sm.prefix = prefix | ((unsigned long long)d << shift);
            sm.pmask = pmask | (255ull << shift);
            break;
          }
          cum += cnt[q];
        }
      }
    }
    __syncthreads();
  }
  *tau_out = __longlong_as_double((long long)sm.prefix);
  *cnt_gt_out = kk - sm.remaining;
  __syncthreads();
}

// Sum of the kk largest non-negative entries (perspective.py:135-140); all of
// them when kk >= count.  Fixed-order reduction.
__device__ double block_topk_sum(const double* vals, int64_t m, int64_t kk, int64_t count,
                                 SelectSmem& sm, double* red) {
  if (kk <= 0 || count == 0) return 0.0;
  double local = 0.0;
  if (kk >= count) {
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
      double v = vals[i];
      if (v >= 0.0) local += v;
    }
    return block_sum(local, red);
  }
  double tau;
  int64_t cnt_gt;
  block_kth_largest(vals, m, kk, sm, &tau, &cnt_gt);
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    double v = vals[i];
    if (v > tau) local += v;
  }
  double s = block_sum(local, red);
  return s + (double)(kk - cnt_gt) * tau;
}

// ---------------------------------------------------------------------------
// Fenchel bound at beta_t from gv = [g | v = X^T zeta | F* acc]  (fista.py:150-157)
// Returns 1 (all threads) when the solve is finished.
// ---------------------------------------------------------------------------
__device__ int dual_step(const EngineArgs& a, ProxSmem& sm) {
  const Params* P = a.prm;
  State* st = a.st;
  const int tid = threadIdx.x;
  const int64_t p = a.p;
  const double* v = a.gv + a.pv;
  const double acc[3] = {a.gv[2 * a.pv], a.gv[2 * a.pv + 1], a.gv[2 * a.pv + 2]};
  const double fstar = conj_finish(P->loss, acc);
  double d = -CUDART_INF;
  if (isfinite(fstar)) {
    // H_M(v / 2 l2) (perspective.py:151); fixed-zero ignored, fixed-one summed
    double fone_local = 0.0;
    for (int64_t j = tid; j < p; j += blockDim.x) {
      const double h = huber(ddiv(v[j], P->two_l2), P->M);
      const int cls = P->node_mode ? a.mask[j] : FREE;
      a.scratch[j] = (cls == FREE) ? h : -1.0;
      if (cls == FIXED_ONE) fone_local += h;
    }
    __syncthreads();
    const double fone_sum = block_sum(fone_local, sm.red);
    const int64_t kg = P->node_mode ? P->k_g : P->k;
    const int64_t nfree = P->node_mode ? P->n_free : p;
    const double top = block_topk_sum(a.scratch, p, kg, nfree, sm.sel, sm.red);
    const double gstar = P->node_mode ? dadd(fone_sum, top) : top;
    d = dsub(-fstar, dmul(P->two_l2, gstar));
  }
  if (tid == 0) {
    bound_update(st, P, d);
    sm.done = st->done;
  }
  __syncthreads();
  return sm.done;
}

// ---------------------------------------------------------------------------
// PAVA closed form on sorted magnitudes xs[0..nf) with budget kk (1 <= kk < nf)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double pool_value(double S, double N, double P, double M) {
  return hprox(ddiv(S, N), ddiv(P, N), M);  // prox.py:86-91
}

__device__ void pava_search(const double* xs, const double* tail, int64_t nf, int64_t kk,
                            double rho, double M, ProxSmem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  if (tid == 0) sm.found = -1;
  __syncthreads();
  for (int64_t base = kk - 1; base >= 0; base -= nw) {
    const int64_t aa = base - warp;
    int valid = 0;
    int64_t cA = 0;
    double VA = 0.0;
    if (aa >= 0) {
      double hs = 0.0;
      for (int64_t j = aa + lane; j < kk; j += 32) hs += xs[j];
      hs = warp_sum(hs);
      const double Pw = dmul(rho, (double)(kk - aa));
      int64_t lo = kk, hi = nf - 1;  // pred(nf-1) is true by definition
      while (lo < hi) {
        const int64_t span = hi - lo;
        const int64_t c = lo + (span * lane) / 32;
        bool pr;
        if (c >= nf - 1) {
          pr = true;
        } else {
          const double V = pool_value(dadd(hs, tail[c]), (double)(c - aa + 1), Pw, M);
          pr = xs[c + 1] <= V;
        }
        const unsigned b = __ballot_sync(0xffffffffu, pr);
        if (b == 0u) {
          lo = lo + (span * 31) / 32 + 1;
        } else {
          const int f = __ffs(b) - 1;
          if (f == 0) {
            hi = lo;
          } else {
            const int64_t cprev = lo + (span * (f - 1)) / 32;
            hi = lo + (span * f) / 32;
            lo = cprev + 1;
          }
        }
      }
      cA = lo;
      VA = pool_value(dadd(hs, tail[cA]), (double)(cA - aa + 1), Pw, M);
      valid = (aa == 0) || (hprox(xs[aa - 1], rho, M) >= VA);
    }
    if (lane == 0) {
      sm.wvalid[warp] = valid;
      sm.wc[warp] = cA;
      sm.wv[warp] = VA;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 0; w < nw; ++w) {
        if (base - w < 0) break;
        if (sm.wvalid[w]) {
          sm.found = 1;
          sm.astar = base - w;
          sm.cstar = sm.wc[w];
          sm.vstar = sm.wv[w];
          break;
        }
      }
    }
    __syncthreads();
    if (sm.found > 0) break;
  }
}

// ---------------------------------------------------------------------------
// g over the free coordinates from sorted-descending top values top[0..kkg)
// (perspective.py:102-111); one warp.
// ---------------------------------------------------------------------------
__device__ double envelope_from_top(const double* top, int64_t kkg, double total) {
  const int lane = threadIdx.x & 31;
  double carry = 0.0;
  int64_t jstar = -1;
  double avg_star = 0.0;
  for (int64_t b = 0; b < kkg && jstar < 0; b += 32) {
    const int64_t j = b + lane;
    const double x = j < kkg ? top[j] : 0.0;
    double incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      double y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    double excl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) excl = 0.0;
    const double before = carry + excl;  // prefix_j = sum_{i<j} top_i
    bool hit = false;
    double avg = 0.0;
    if (j < kkg) {
      avg = ddiv(dsub(total, before), (double)(kkg - j));
      hit = avg >= x;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, hit);
    if (bal) {
      const int f = __ffs(bal) - 1;
      jstar = b + f;
      avg_star = __shfl_sync(0xffffffffu, avg, f);
    }
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (jstar < 0) {  // round-off fallback: last slot (perspective.py:106-108)
    jstar = kkg - 1;
    double pre = 0.0;
    for (int64_t i = lane; i < jstar; i += 32) pre += top[i];
    pre = warp_sum(pre);
    avg_star = ddiv(dsub(total, pre), (double)(kkg - jstar));
  }
  double h2 = 0.0;
  for (int64_t i = lane; i < jstar; i += 32) h2 = fma(top[i], top[i], h2);
  h2 = warp_sum(h2);
  return dmul(0.5, dadd(h2, dmul(dmul((double)(kkg - jstar), avg_star), avg_star)));
}

// rank sort (descending) of m <= kCandCap values held in smem `src` into `dst`
__device__ void block_rank_sort_desc(const double* src, double* dst, int m) {
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double x = src[i];
    int r = 0;
    for (int j = 0; j < m; ++j) {
      const double y = src[j];
      r += (y > x) || (y == x && j < i);
    }
    dst[r] = x;
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// After the sort: PAVA, scatter, g.  Shared by the one-CTA and onesweep paths
// and by the standalone operator.  xs/perm hold the sorted keys/ids.
//   in    : gamma (g-mode) or mu (gstar-mode), indexed by coordinate
//   out   : beta+ (g-mode) or prox_gstar (gstar-mode)
// ---------------------------------------------------------------------------
template <int T>
__device__ void prox_post_sort(const PostArgs& q_in, ProxSmem& sm) {
  const int tid = threadIdx.x;
  PostArgs q = q_in;
  if (q.nf < 0) {  // standalone operator: count the free (non-negative) keys
    double c = 0.0;
    for (int64_t pos = tid; pos < q.p; pos += T) c += q.xs[pos] >= 0.0 ? 1.0 : 0.0;
    q.nf = (int64_t)block_sum(c, sm.red);
    if (q.kk > q.nf) q.kk = q.nf;
    if (q.kg > q.nf && q.kg < 0) q.kg = q.nf;
  }
  const int64_t p = q.p, nf = q.nf, kk = q.kk;
  const double rho = q.rho, M = q.M;
  // _prox_gstar_core cases (prox.py:104-112)
  const int how = (kk <= 0 || nf == 0) ? 0 : (kk >= nf ? 1 : 2);  // pass / elementwise / PAVA
  if (tid == 0) { sm.found = -1; sm.astar = -1; sm.cstar = -1; }
  __syncthreads();
  if (how == 2) {
    // tail prefix sums T[c] = x_kk + ... + x_c (c in [kk, nf)), blocked ranges
    const int64_t per = (nf + T - 1) / T;
    const int64_t b0 = min(nf, (int64_t)tid * per), b1 = min(nf, b0 + per);
    double local = 0.0;
    for (int64_t i = max(b0, kk); i < b1; ++i) local += q.xs[i];
    double excl;
    {
      using Scan = cub::BlockScan<double, T>;
      static_assert(sizeof(typename Scan::TempStorage) <= sizeof(sm.u), "scan storage");
      Scan(reinterpret_cast<typename Scan::TempStorage&>(sm.u)).ExclusiveSum(local, excl);
    }
    double run = excl;
    for (int64_t i = max(b0, kk); i < b1; ++i) {
      run += q.xs[i];
      q.tail[i] = run;
    }
    __syncthreads();
    const double xk = q.xs[kk];
    if (xk > hprox(q.xs[kk - 1], rho, M)) {  // prox.py:80 first merge at k-1|k
      pava_search(q.xs, q.tail, nf, kk, rho, M, sm);
    }
    __syncthreads();
  }
  const int64_t astar = sm.found > 0 ? sm.astar : INT64_MAX;
  const int64_t cstar = sm.found > 0 ? sm.cstar : -1;
  const double vstar = sm.vstar;
  if (q.rec != nullptr)
    record_prox(q.rec, q.rec_cap, q.rec_w, q.perm, q.rec_iter, how, sm.found > 0 ? 1 : 0, astar,
                cstar, how == 2 ? nf : 0, 2, nf);

  // scatter
  double total = 0.0, amax = 0.0, rest = 0.0;
  const int64_t kkg = q.kg < nf ? q.kg : nf;
  const int64_t W = min(nf, kkg + 64);
  for (int64_t pos = tid; pos < p; pos += T) {
    const int j = q.perm[pos];
    const double gin = q.in[j];
    const double mu = q.gmode ? dmul(rho, gin) : gin;
    const int cls = q.mask ? q.mask[j] : FREE;
    double out;
    if (cls == FIXED_ZERO) {
      out = mu;  // passes through prox_gstar_node (prox.py:181)
    } else if (cls == FIXED_ONE) {
      out = dmul(dsign(mu), hprox(fabs(mu), rho, M));  // prox.py:182-184
    } else if (how == 0) {
      out = mu;  // prox.py:104-105 (copy)
    } else if (how == 1) {
      out = dmul(dsign(mu), hprox(fabs(mu), rho, M));  // prox.py:108-110
    } else {
      const double x = q.xs[pos];
      double nu;
      if (pos < astar) nu = (pos < kk) ? hprox(x, rho, M) : x;
      else if (pos <= cstar) nu = vstar;
      else nu = (pos < kk) ? hprox(x, rho, M) : x;
      out = dmul(nu, dsign(mu));  // out[order] = nu; out *= signs (prox.py:113-115)
    }
    double res;
    if (q.gmode) {
      res = (cls == FIXED_ZERO && q.mask) ? 0.0 : dsub(gin, ddiv(out, rho));  // fista.py:107/126-127
    } else {
      res = out;
    }
    q.out[j] = res;
    if (q.want_g && cls == FREE) {
      const double ab = fabs(res);
      total += ab;
      amax = fmax(amax, ab);
      if (pos < W) sm.cand[pos] = ab;
      else rest = fmax(rest, ab);
      q.absb[pos] = ab;
    } else if (q.want_g) {
      q.absb[pos] = -1.0;
    }
  }
  if (!q.want_g) return;
  total = block_sum(total, sm.red);
  amax = block_max(amax, sm.red);
  rest = block_max(rest, sm.red);

  // fixed-one part: 0.5 * sum beta_j^2 with a box check (perspective.py:124-129)
  double fone_val = 0.0;
  bool fone_bad = false;
  if (tid == 0 && q.fone != nullptr) {
    double s2 = 0.0;
    for (int64_t i = 0; i < q.n_fone; ++i) {
      const double b = q.out[q.fone[i]];
      if (fabs(b) > dmul(M, dadd(1.0, kFeasRtol))) fone_bad = true;
      s2 = fma(b, b, s2);
    }
    fone_val = dmul(0.5, s2);
  }
  // free part (perspective.py:76-111)
  double gfree;
  int path = 0;  // 0 window, 1 radix select, 2 trivial
  if (nf == 0) { gfree = 0.0; path = 2; }
  else if (amax > dmul(M, dadd(1.0, kFeasRtol))) { gfree = CUDART_INF; path = 2; }
  else if (total > dmul(dmul((double)q.kg, M), dadd(1.0, kFeasRtol))) { gfree = CUDART_INF; path = 2; }
  else if (q.kg == 0) { gfree = 0.0; path = 2; }
  else gfree = 0.0;
  if (path == 0) {
    if (W > kCandCap) path = 1;
    else {
      block_rank_sort_desc(sm.cand, sm.cand2, (int)W);
      if (W < nf && rest > sm.cand2[kkg - 1]) path = 1;  // window missed a larger value
    }
    if (path == 1 && kkg > kCandCap) {
      if (tid == 0) { atomicExch(&q.st->err, (int)ST_UNSUPPORTED); q.st->done = 1; }
      return;
    }
    if (path == 1) {
      // exact top-kk multiset: kk-th largest tau, all values > tau, then copies of tau
      __syncthreads();
      double tau;
      int64_t cgt;
      block_kth_largest(q.absb, p, kkg, sm.sel, &tau, &cgt);
      if (tid == 0) sm.ncand = 0;
      __syncthreads();
      for (int64_t pos = tid; pos < p; pos += T) {
        const double x = q.absb[pos];
        if (x > tau) sm.cand[atomicAdd(&sm.ncand, 1)] = x;
      }
      __syncthreads();
      for (int64_t i = cgt + tid; i < kkg; i += T) sm.cand[i] = tau;
      __syncthreads();
      block_rank_sort_desc(sm.cand, sm.cand2, (int)kkg);
      if (tid == 0 && q.st) q.st->topk_fallbacks += 1;
    }
    if (threadIdx.x < 32) {
      const double gv = envelope_from_top(sm.cand2, kkg, total);
      if (threadIdx.x == 0) sm.gfree = gv;
    }
    __syncthreads();
    gfree = sm.gfree;
  }
  if (tid == 0) {
    double g = gfree;
    if (q.fone != nullptr) g = fone_bad ? CUDART_INF : dadd(dadd(0.0, fone_val), gfree);
    *q.g_out = g;
  }
}

// ---------------------------------------------------------------------------
// FISTA prox kernels
// ---------------------------------------------------------------------------
__device__ __forceinline__ PostArgs iter_post_args(const EngineArgs& a) {
  const Params* P = a.prm;
  State* st = a.st;
  PostArgs q;
  q.p = a.p;
  q.nf = P->node_mode ? P->n_free : a.p;
  q.kk = P->node_mode ? P->k_rem : P->k;
  q.kg = P->node_mode ? P->k_g : P->k;
  q.rho = P->rho;
  q.M = P->M;
  q.xs = a.xs;
  q.perm = a.perm;
  q.tail = a.tail;
  q.in = a.gam;
  q.out = a.beta + ring(st->t + 1) * a.pv;
  q.absb = a.scratch;
  q.mask = P->node_mode ? a.mask : nullptr;
  q.fone = P->node_mode ? a.fone : nullptr;
  q.n_fone = P->n_fone;
  q.gmode = 1;
  q.want_g = 1;
  q.g_out = &st->g_next;
  q.st = st;
  q.rec = a.prox_rec;
  q.rec_cap = a.prox_rec_cap;
  q.rec_w = a.prox_rec_w;
  q.rec_iter = st->t + 1;
  return q;
}

template <int T, int IPT>
__global__ void __launch_bounds__(T, 1) k3_prox_block(EngineArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using Sort = cub::BlockRadixSort<double, T, IPT, int, 6>;
  ProxSmem& sm = *reinterpret_cast<ProxSmem*>(smem_raw);
  typename Sort::TempStorage& tmp =
      *reinterpret_cast<typename Sort::TempStorage*>(smem_raw + sizeof(ProxSmem));
  const State* st = a.st;
  if (st->done) return;
  if (st->dual_pending) {
    if (dual_step(a, sm)) return;
  }
  if (a.st->dual_only) return;
  double keys[IPT];
  int ids[IPT];
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int j = threadIdx.x * IPT + i;
    keys[i] = j < a.p ? a.key[j] : -CUDART_INF;
    ids[i] = j;
  }
  Sort(tmp).SortDescending(keys, ids);  // stable: ties keep ascending ids (prox.py:111)
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int pos = threadIdx.x * IPT + i;
    if (pos < a.p) {
      a.xs[pos] = keys[i];
      a.perm[pos] = ids[i];
    }
  }
  __syncthreads();
  prox_post_sort<T>(iter_post_args(a), sm);
}

__global__ void __launch_bounds__(1024, 1) k3_prox_post(EngineArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ProxSmem& sm = *reinterpret_cast<ProxSmem*>(smem_raw);
  const State* st = a.st;
  if (st->done) return;
  if (st->dual_pending) {
    if (dual_step(a, sm)) return;
  }
  if (a.st->dual_only) return;
  prox_post_sort<1024>(iter_post_args(a), sm);
}

// block-path configurations: capacity T * IPT
template <int T, int IPT>
static size_t block_smem() {
  return sizeof(ProxSmem) + sizeof(typename cub::BlockRadixSort<double, T, IPT, int, 6>::TempStorage);
}

template <int T, int IPT>
static cudaError_t launch_block(const EngineArgs& a, cudaStream_t s) {
  const size_t smem = block_smem<T, IPT>();
  cudaError_t e = cudaFuncSetAttribute(k3_prox_block<T, IPT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k3_prox_block<T, IPT><<<1, T, smem, s>>>(a);
  return cudaGetLastError();
}

bool prox_block_path(int64_t p) { return p <= 16384; }

size_t prox_sort_tmp_bytes(int64_t p) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairsDescending<double, int>(nullptr, bytes, (const double*)nullptr,
                                                         (double*)nullptr, (const int*)nullptr,
                                                         (int*)nullptr, (int)p);
  return bytes;
}

cudaError_t launch_prox_window(const EngineArgs& a, cudaStream_t s);

cudaError_t launch_prox_iter(const EngineArgs& a, void* sort_tmp, size_t sort_tmp_bytes,
                             cudaStream_t s) {
  if (a.prox_full_sort == 0) return launch_prox_window(a, s);
  if (a.p <= 1024) return launch_block<256, 4>(a, s);
  if (a.p <= 4096) return launch_block<512, 8>(a, s);
  if (a.p <= 16384) return launch_block<1024, 16>(a, s);
  size_t bytes = sort_tmp_bytes;
  cudaError_t e = cub::DeviceRadixSort::SortPairsDescending(sort_tmp, bytes, a.key, a.xs, a.iota,
                                                            a.perm, (int)a.p, 0, 64, s);
  if (e != cudaSuccess) return e;
  const size_t smem = sizeof(ProxSmem);
  e = cudaFuncSetAttribute(k3_prox_post, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k3_prox_post<<<1, 1024, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace l0
