// The two HBM passes of a FISTA iteration and their fused epilogues.
//
//   K1  u = X.beta          fista.py:165 (and :141, :209)      + loss, objective, restart
//   K2  g = X^T grad F(u_g)  fista.py:162 (X@gamma by linearity) + X^T zeta (fista.py:156)
//                                                               + gradient step fista.py:161-163
//
// X is row-major n x ld (fp64, or fp32 widened to fp64 in registers), read
// with 128-bit streaming loads (ld.global.cs: X is touched once per pass and
// must not evict the L2-resident vectors/partials).  All accumulation is in
// fp64 with fixed summation order, so results are deterministic.
//
// Cross-CTA combination uses the "last CTA finishes the job" pattern: every
// CTA publishes its partial, fences, bumps a counter; the CTA that observes
// the final count performs the reduction in a fixed order and resets the
// counter for the next launch (so the kernels are CUDA-graph replayable).

#include "control.cuh"
#include "engine.cuh"
#include "slab_epilogue.cuh"

namespace l0 {

template <typename TX> struct Vec16;
template <> struct Vec16<double> {
  using T = double2;
  static constexpr int N = 2;
  __device__ __forceinline__ static void widen(const T& v, double* o) { o[0] = v.x; o[1] = v.y; }
};
template <> struct Vec16<float> {
  using T = float4;
  static constexpr int N = 4;
  __device__ __forceinline__ static void widen(const T& v, double* o) {
    o[0] = (double)v.x; o[1] = (double)v.y; o[2] = (double)v.z; o[3] = (double)v.w;
  }
};

__device__ __forceinline__ double2 ld_stream(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ float4 ld_stream(const float4* p) { return __ldcs(p); }

// ===========================================================================
// K1: forward pass u = X beta.  Persistent CTAs pull (chunk, slab) items from
// a work counter; an item is `k1_rows` rows x kK1Slab columns.
// ===========================================================================
template <typename TX>
__device__ __forceinline__ void k1_rows_dot(const EngineArgs& a, const double* sbeta, int slab,
                                            int64_t r0, int64_t r1, int warp, int lane) {
  using V = Vec16<TX>;
  constexpr int VE = V::N;
  constexpr int U = 8;
  const int64_t c0 = (int64_t)slab * kK1Slab;
  const int64_t width = min((int64_t)kK1Slab, a.ld - c0);  // multiple of VE
  const int nvec = (int)(width / VE);
  for (int64_t r = r0 + warp; r < r1; r += kK1Threads / 32) {
    const typename V::T* xv = reinterpret_cast<const typename V::T*>(
        static_cast<const TX*>(a.X) + r * a.ld + c0);
    double acc = 0.0;
    for (int v0 = lane; v0 < nvec; v0 += 32 * U) {
      typename V::T buf[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int v = v0 + q * 32;
        if (v < nvec) buf[q] = ld_stream(xv + v);
      }
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int v = v0 + q * 32;
        if (v < nvec) {
          double x[VE];
          V::widen(buf[q], x);
#pragma unroll
          for (int e = 0; e < VE; ++e) acc = fma(x[e], sbeta[v * VE + e], acc);
        }
      }
    }
    acc = warp_sum(acc);
    if (lane == 0) a.u_part[(int64_t)slab * a.n + r] = acc;
  }
}

template <typename TX>
__global__ void __launch_bounds__(kK1Threads) k1_forward(EngineArgs a, int mode) {
  __shared__ __align__(16) double sbeta[kK1Slab];
  __shared__ double red[32];
  __shared__ unsigned s_item;
  __shared__ int s_last;
  __shared__ int s_bad;

  State* st = a.st;
  int64_t t = 0;
  const double* bvec;
  if (mode == MODE_ITER) {
    if (st->done || st->dual_only) return;
    t = st->t + 1;
    bvec = a.beta + ring(t) * a.pv;
  } else if (mode == MODE_INIT) {
    bvec = a.beta;  // slot 0 holds beta_0
  } else {
    bvec = a.in_vec;
  }
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t n = a.n;
  const unsigned items = (unsigned)a.k1_slabs * (unsigned)a.k1_chunks;
  int cur_slab = -1;
  for (;;) {
    __syncthreads();
    if (tid == 0) s_item = atomicAdd(cnt_k1_work(a), 1u);
    __syncthreads();
    const unsigned item = s_item;
    if (item >= items) break;
    const int chunk = (int)(item / a.k1_slabs), slab = (int)(item % a.k1_slabs);
    if (slab != cur_slab) {
      const int64_t c0 = (int64_t)slab * kK1Slab;
      for (int j = tid; j < kK1Slab; j += kK1Threads) {
        const int64_t col = c0 + j;
        sbeta[j] = col < a.p ? bvec[col] : 0.0;
      }
      cur_slab = slab;
      __syncthreads();
    }
    const int64_t r0 = (int64_t)chunk * a.k1_rows;
    const int64_t r1 = min(n, r0 + a.k1_rows);
    k1_rows_dot<TX>(a, sbeta, slab, r0, r1, warp, lane);

    // ---- last slab of this chunk: u = sum over slabs, loss terms ------------
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(cnt_k1_chunk(a) + chunk, 1u) == (unsigned)(a.k1_slabs - 1));
    __syncthreads();
    if (!s_last) continue;
    __threadfence();
    double lsum = 0.0;
    int bad = 0;
    for (int64_t r = r0 + tid; r < r1; r += kK1Threads) {
      double u = 0.0;
      for (int s = 0; s < a.k1_slabs; ++s) u += __ldcg(a.u_part + (int64_t)s * n + r);
      if (mode == MODE_PLAIN) {
        a.out_vec[r] = u;
        continue;
      }
      if (mode == MODE_ITER) {
        a.u[ring(t) * n + r] = u;
      } else {
        a.u[r] = u;
        a.u[2 * n + r] = u;
      }
      if (!isfinite(u)) bad = 1;
      lsum += loss_term(a.loss, u, a.y[r]);
    }
    if (tid == 0) {
      cnt_k1_chunk(a)[chunk] = 0u;
      s_bad = 0;
    }
    if (mode == MODE_PLAIN) continue;
    __syncthreads();
    if (bad) s_bad = 1;
    const double csum = block_sum(lsum, red);  // barrier inside: s_bad settled
    if (tid == 0) {
      a.loss_part[2 * chunk] = csum;
      a.loss_part[2 * chunk + 1] = (double)s_bad;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(cnt_k1_all(a), 1u) == (unsigned)(a.k1_chunks - 1));
    __syncthreads();
    if (!s_last) continue;
    __threadfence();
    // ---- very last chunk: F(u) over chunks (fixed order), objective -------
    double tot = 0.0, nb = 0.0;
    for (int ch = tid; ch < a.k1_chunks; ch += kK1Threads) {
      tot += __ldcg(a.loss_part + 2 * ch);
      nb += __ldcg(a.loss_part + 2 * ch + 1);
    }
    tot = block_sum(tot, red);
    nb = block_sum(nb, red);
    if (tid == 0) {
      cnt_k1_all(a)[0] = 0u;
      if (a.multi) {  // row-sharded: the objective runs after the all-reduce of this pair
        a.gv[2 * a.pv + 4] = tot;
        a.gv[2 * a.pv + 5] = nb;
      } else if (nb > 0.0) {  // loss_value on non-finite predictions (model.py:152-161)
        st->err = ST_INVALID;
        st->err_iter = (mode == MODE_ITER) ? t : 0;
        if (mode == MODE_ITER) st->t = t;
        st->done = 1;
      } else if (mode == MODE_ITER) {
        objective_update(st, a.prm, tot);
      } else {
        st->loss_cur = tot;
        st->obj = dadd(tot, dmul(a.prm->two_l2, st->g_next));  // fista.py:143
      }
    }
  }
  // ---- exit: the last CTA out re-arms the work counter ----------------------
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(cnt_k1_exit(a), 1u) == gridDim.x - 1) {
      *cnt_k1_work(a) = 0u;
      *cnt_k1_exit(a) = 0u;
      __threadfence();
    }
  }
}

// Objective from the all-reduced loss pair gv[2pv+4 .. 2pv+6) (row-sharded mode).
__global__ void k_objective(EngineArgs a, int mode) {
  State* st = a.st;
  if (mode == MODE_ITER && (st->done || st->dual_only)) return;
  double tot = a.gv[2 * a.pv + 4], nb = a.gv[2 * a.pv + 5];
  if (nb > 0.0) {
    st->err = ST_INVALID;
    st->err_iter = (mode == MODE_ITER) ? st->t + 1 : 0;
    if (mode == MODE_ITER) st->t += 1;
    st->done = 1;
  } else if (mode == MODE_ITER) {
    objective_update(st, a.prm, tot);
  } else {
    st->loss_cur = tot;
    st->obj = dadd(tot, dmul(a.prm->two_l2, st->g_next));
  }
}

// ===========================================================================
// K2: transpose pass g = X^T r (and v = X^T zeta on bound checks).
// Persistent CTAs pull (chunk, slab group) items; an item is `k2_rows` rows x
// kK2Cw<TX> slabs of 256 columns (2 for fp32, so every row segment a CTA
// streams is 2 KB as for fp64).  Each lane owns 8 columns per slab; the 8
// warps split the rows and are combined in a fixed order through shared memory.
// ===========================================================================
template <typename TX, bool WG, bool WZ>
__device__ __forceinline__ void k2_accumulate(const EngineArgs& a, const double (*sr)[kK2StageRows],
                                              int64_t s0, int rows, int64_t col0, int lane,
                                              int warp, double* accg, double* accz) {
  using V = Vec16<TX>;
  constexpr int VE = V::N;
  constexpr int CW = kK2Cw<TX>;
  constexpr int NV = 8 * CW / VE;  // vectors per lane per row (8 columns per lane per slab)
  const TX* xbase = static_cast<const TX*>(a.X) + s0 * a.ld + col0 + lane * VE;
  // vectors of this lane that lie inside the row (ld is a multiple of VE)
  const int64_t width = min((int64_t)(kK2Slab * CW), a.ld - col0);
  bool vok[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) vok[v] = (v * 32 * VE + lane * VE) < width;
  // warp w takes rows w, w+8, ...; RS rows per step for memory parallelism
  constexpr int RS = 2;
  for (int rr = warp; rr < rows; rr += 8 * RS) {
    typename V::T b[RS][NV];
#pragma unroll
    for (int i = 0; i < RS; ++i) {
      const int ri = rr + 8 * i;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        if (vok[v] && ri < rows)
          b[i][v] = ld_stream(reinterpret_cast<const typename V::T*>(xbase + (int64_t)ri * a.ld + v * 32 * VE));
        else
          b[i][v] = typename V::T{};
      }
    }
#pragma unroll
    for (int i = 0; i < RS; ++i) {
      const int ri = rr + 8 * i;
      if (ri >= rows) break;
      const double rg = WG ? sr[0][ri] : 0.0;
      const double rz = WZ ? sr[1][ri] : 0.0;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        double x[VE];
        V::widen(b[i][v], x);
#pragma unroll
        for (int e = 0; e < VE; ++e) {
          if (WG) accg[v * VE + e] = fma(x[e], rg, accg[v * VE + e]);
          if (WZ) accz[v * VE + e] = fma(x[e], rz, accz[v * VE + e]);
        }
      }
    }
  }
}

struct K2Smem {
  double sr[2][kK2StageRows];
  union {
    double sacc[8][2][kK2Slab];  // per-warp column sums (fixed-order combine)
    EpiSmem epi;                 // slab epilogue (after the partials are published)
  };
  double red[32];
  unsigned item;
  int last;
};

template <typename TX, bool WG, bool WZ>
__device__ __forceinline__ void k2_body(const EngineArgs& a, int mode, int64_t t, double c,
                                        K2Smem& sm) {
  using V = Vec16<TX>;
  constexpr int VE = V::N;
  constexpr int CW = kK2Cw<TX>;
  constexpr int NV = 8 * CW / VE;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t n = a.n;
  const int groups = (a.k2_slabs + CW - 1) / CW;
  const unsigned items = (unsigned)groups * (unsigned)a.k2_chunks;
  int bad = 0;
  for (;;) {
    __syncthreads();
    if (tid == 0) sm.item = atomicAdd(cnt_k2_work(a), 1u);
    __syncthreads();
    const unsigned item = sm.item;
    if (item >= items) break;
    const int chunk = (int)(item / groups), grp = (int)(item % groups);
    const int64_t col0 = (int64_t)grp * CW * kK2Slab;
    const int64_t r0 = (int64_t)chunk * a.k2_rows;
    const int64_t r1 = min(n, r0 + a.k2_rows);
    const bool fst = WZ && mode == MODE_ITER && grp == 0;  // this item owns the F* partial

    double accg[8 * CW], accz[8 * CW];
#pragma unroll
    for (int i = 0; i < 8 * CW; ++i) { accg[i] = 0.0; accz[i] = 0.0; }
    double facc[3] = {0.0, 0.0, 0.0};

    for (int64_t s0 = r0; s0 < r1; s0 += kK2StageRows) {
      const int rows = (int)min((int64_t)kK2StageRows, r1 - s0);
      __syncthreads();
      if (tid < rows) {
        const int64_t i = s0 + tid;
        if (mode == MODE_ITER) {
          const double ucur = a.u[ring(t - 1) * n + i];
          const double yi = a.y[i];
          if (WG) {
            // X gamma = u_{t-1} + c (u_{t-1} - u_{t-2})   (linearity; fista.py:161-162)
            const double up = a.u[ring(t - 2) * n + i];
            const double ug = dadd(ucur, dmul(c, dsub(ucur, up)));
            if (!isfinite(ug)) bad = 1;
            sm.sr[0][tid] = loss_grad(a.loss, ug, yi);
          }
          if (WZ) {
            const double z = -loss_grad(a.loss, ucur, yi);  // zeta = -grad F(u) (fista.py:152)
            sm.sr[1][tid] = z;
            if (fst) conj_accumulate(a.loss, z, yi, facc);
          }
        } else {
          if (WG) sm.sr[0][tid] = a.in_vec[i];
          if (WZ) sm.sr[1][tid] = a.in_vec2[i];
        }
      }
      __syncthreads();
      if (col0 < a.ld)
        k2_accumulate<TX, WG, WZ>(a, sm.sr, s0, rows, col0, lane, warp, accg, accz);
    }

    // ---- combine the 8 warps (fixed order) and publish the item partial -----
    // (one 256-column slab of the group at a time: lane vectors 2h.. belong to slab h)
#pragma unroll
    for (int h = 0; h < CW; ++h) {
      __syncthreads();
#pragma unroll
      for (int v = h * (NV / CW); v < (h + 1) * (NV / CW); ++v) {
#pragma unroll
        for (int e = 0; e < VE; ++e) {
          const int col = (v - h * (NV / CW)) * 32 * VE + lane * VE + e;
          if (WG) sm.sacc[warp][0][col] = accg[v * VE + e];
          if (WZ) sm.sacc[warp][1][col] = accz[v * VE + e];
        }
      }
      __syncthreads();
      const int col = tid;  // 256 threads <-> 256 columns
      if (WG) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) s += sm.sacc[w][0][col];
        a.k2_part[(int64_t)chunk * a.pv + col0 + h * kK2Slab + col] = s;
      }
      if (WZ) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) s += sm.sacc[w][1][col];
        a.k2_part[((int64_t)a.k2_chunks + chunk) * a.pv + col0 + h * kK2Slab + col] = s;
      }
    }
    if (fst) {
      const double f0 = block_sum(facc[0], sm.red);
      const double f1 = block_sum(facc[1], sm.red);
      const double f2 = block_sum(facc[2], sm.red);
      if (tid == 0) {
        a.k2_fpart[4 * chunk + 0] = f0;
        a.k2_fpart[4 * chunk + 1] = f1;
        a.k2_fpart[4 * chunk + 2] = f2;
      }
    }

    // ---- last chunk of this slab group: reduce over chunks, gradient step -----
    __threadfence();
    __syncthreads();
    if (tid == 0) sm.last = (atomicAdd(cnt_k2_slab(a) + grp, 1u) == (unsigned)(a.k2_chunks - 1));
    __syncthreads();
    if (!sm.last) continue;
    __threadfence();
#pragma unroll
    for (int h = 0; h < CW; ++h) {
      const int slab = grp * CW + h;
      if (slab >= a.k2_slabs) break;
      const int64_t col = (int64_t)slab * kK2Slab + tid;
      double g = 0.0, v = 0.0;
      if (col < a.p) {
        if (WG) {
          for (int ch = 0; ch < a.k2_chunks; ++ch) g += __ldcg(a.k2_part + (int64_t)ch * a.pv + col);
          if (mode == MODE_PLAIN) a.out_vec[col] = g;
          else a.gv[col] = g;
        }
        if (WZ) {
          for (int ch = 0; ch < a.k2_chunks; ++ch)
            v += __ldcg(a.k2_part + ((int64_t)a.k2_chunks + ch) * a.pv + col);
          if (mode == MODE_PLAIN) a.out_vec2[col] = v;
          else a.gv[a.pv + col] = v;
        }
      }
      // single GPU: the prox's elementwise work for these 256 columns
      if (mode == MODE_ITER && !a.multi) {
        __syncthreads();
        slab_epilogue(a, slab, t, c, WG, WZ, g, v, sm.epi);
      }
    }
    if (tid == 0) cnt_k2_slab(a)[grp] = 0u;
    if (!(WZ && mode == MODE_ITER)) continue;
    // ---- very last slab: F*(-zeta) accumulators over chunks (fixed order) ---
    __threadfence();
    __syncthreads();
    if (tid == 0) sm.last = (atomicAdd(cnt_k2_all(a), 1u) == (unsigned)(groups - 1));
    __syncthreads();
    if (!sm.last) continue;
    __threadfence();
    if (tid == 0) {
      double f0 = 0.0, f1 = 0.0, f2 = 0.0;
      for (int ch = 0; ch < a.k2_chunks; ++ch) {
        f0 += __ldcg(a.k2_fpart + 4 * ch + 0);
        f1 += __ldcg(a.k2_fpart + 4 * ch + 1);
        f2 += __ldcg(a.k2_fpart + 4 * ch + 2);
      }
      a.gv[2 * a.pv + 0] = f0;
      a.gv[2 * a.pv + 1] = f1;
      a.gv[2 * a.pv + 2] = f2;
      cnt_k2_all(a)[0] = 0u;
    }
  }
  if (WG && mode == MODE_ITER && bad) {
    // loss_gradient on non-finite predictions: model.py:215 -> InvalidInputError
    atomicExch(&a.st->err, (int)ST_INVALID);
    a.st->err_iter = t;
    a.st->done = 1;
  }
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(cnt_k2_exit(a), 1u) == gridDim.x - 1) {
      *cnt_k2_work(a) = 0u;
      *cnt_k2_exit(a) = 0u;
      __threadfence();
    }
  }
}

template <typename TX>
__global__ void __launch_bounds__(kK2Threads, 2) k2_transpose(EngineArgs a, int mode) {
  __shared__ K2Smem sm;
  bool wg = true, wz = false;
  int64_t t = 0;
  double c = 0.0;
  if (mode == MODE_ITER) {
    const State* st = a.st;
    if (st->done) return;
    // behind the SPEC single-pass kernel (fused.cu): only the iterations KR left
    // (restart: the restart candidate; bound pass: X^T zeta -- the gradient of a
    // bound-check iteration that did not restart stays KR's)
    if (a.k2_cond == 1 && !(st->last_restarted || st->dual_pending || st->dual_only)) return;
    if (a.k2_cond == 2 && !(st->last_restarted || st->dual_only)) return;
    wz = st->dual_pending != 0 && (a.k2_cond != 2 || st->dual_only);
    wg = st->dual_only == 0 && (!a.k2_cond || st->last_restarted);
    t = st->t + 1;
    c = momentum(st->phi);
  } else {
    wz = a.plain_rhs2 > 1;
  }
  if (wg && wz) k2_body<TX, true, true>(a, mode, t, c, sm);
  else if (wg) k2_body<TX, true, false>(a, mode, t, c, sm);
  else if (wz) k2_body<TX, false, true>(a, mode, t, c, sm);
}

// gradient step + slab epilogue as its own pass (row-sharded mode: after the
// all-reduce of [g | v]); one CTA per slab of 256 columns
__global__ void __launch_bounds__(kK2Slab) k_grad_step(EngineArgs a) {
  __shared__ EpiSmem sm;
  const State* st = a.st;
  if (st->done) return;
  const bool wg = st->dual_only == 0;       // final bound pass: Huber values only
  const bool wz = st->dual_pending != 0;
  if (!wg && !wz) return;
  const int64_t t = st->t + 1;
  const double c = momentum(st->phi);
  const int64_t j = (int64_t)blockIdx.x * kK2Slab + threadIdx.x;
  const double g = (wg && j < a.p) ? a.gv[j] : 0.0;
  const double v = (wz && j < a.p) ? a.gv[a.pv + j] : 0.0;
  slab_epilogue(a, blockIdx.x, t, c, wg, wz, g, v, sm);
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
cudaError_t launch_k1(const EngineArgs& a, int mode, cudaStream_t s) {
  if (a.dtype == F64) k1_forward<double><<<a.k1_grid, kK1Threads, 0, s>>>(a, mode);
  else k1_forward<float><<<a.k1_grid, kK1Threads, 0, s>>>(a, mode);
  return cudaGetLastError();
}

cudaError_t launch_k2(const EngineArgs& a, int mode, cudaStream_t s) {
  if (a.dtype == F64) k2_transpose<double><<<a.k2_grid, kK2Threads, 0, s>>>(a, mode);
  else k2_transpose<float><<<a.k2_grid, kK2Threads, 0, s>>>(a, mode);
  return cudaGetLastError();
}

// resident CTAs per SM of the persistent kernels (grid sizing)
int k1_blocks_per_sm(int dtype) {
  int nb = 0;
  if (dtype == F64) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k1_forward<double>, kK1Threads, 0);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k1_forward<float>, kK1Threads, 0);
  return nb > 0 ? nb : 1;
}
int k2_blocks_per_sm(int dtype) {
  int nb = 0;
  if (dtype == F64) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k2_transpose<double>, kK2Threads, 0);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k2_transpose<float>, kK2Threads, 0);
  return nb > 0 ? nb : 1;
}

cudaError_t launch_grad_step(const EngineArgs& a, cudaStream_t s) {
  k_grad_step<<<a.k2_slabs, kK2Slab, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_objective(const EngineArgs& a, int mode, cudaStream_t s) {
  k_objective<<<1, 1, 0, s>>>(a, mode);
  return cudaGetLastError();
}

}  // namespace l0
