// KF: one physical pass over X per FISTA iteration.
//
// Iteration t needs u_t = X beta_t (objective, restart test) and the next
// gradient X^T grad F(u_t + c_{t+1} (u_t - u_{t-1})), whose momentum c_{t+1}
// depends on the restart decision, i.e. on ALL rows of u_t.  KF computes both
// candidates -- c = 1/4 (restart, phi -> 1) and c = (phi+1)/(phi+4) (no
// restart) -- plus X^T zeta_t for the bound check, from the same X tile:
//
//   * a thread-block cluster of fz_cs CTAs spans a full row block; CTA c owns
//     columns [c W, (c+1) W) with its beta slice in shared memory;
//   * row tiles (fz_rows rows x W columns) stream HBM -> shared memory with
//     cp.async.bulk (TMA bulk copies, one mbarrier per double buffer);
//   * forward: per-row partial dots, block-reduced, exchanged through
//     distributed shared memory after one cluster barrier -> u_t for the tile,
//     identical in every CTA (fixed order over the cluster);
//   * transpose: the same shared-memory tile accumulates X^T [r_R | r_N | zeta]
//     in registers (8..12 columns per thread);
//   * the last CTA of the grid reduces the per-cluster loss (fixed order) and
//     runs the objective / restart logic (control.cuh).
//
// KR then reduces the per-cluster partials over clusters (fixed order), picks
// the candidate matching the restart decision and runs the slab epilogue
// (gradient step, keys, window candidates, Huber values).
//
// Arithmetic per row and column is the 2-pass engine's (gemv.cu), so results
// agree with it to summation-order rounding.

#include <cstdio>
#include <cstdlib>

#include "control.cuh"
#include "engine.cuh"
#include "slab_epilogue.cuh"

namespace l0 {

constexpr int kFzThreads = 256;
constexpr int kFzMaxRows = 8;
// vectors (16 B) per thread per row: 8 fp64 or 12 fp32 columns per thread,
// i.e. 24 / 36 fp64 accumulators for the three right-hand sides
template <typename TX> constexpr int fz_maxv() { return sizeof(TX) == 8 ? 4 : 3; }

// ---------------------------------------------------------------------------
// PTX helpers: mbarrier, bulk copy, cluster barrier, DSMEM
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t saddr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(saddr(bar)), "r"(phase)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar))
      : "memory");
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ double ld_dsmem(const double* local, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(saddr(local)), "r"(rank));
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra) : "memory");
  return v;
}

template <typename TX> struct FzVec;
template <> struct FzVec<double> {
  using T = double2;
  static constexpr int N = 2;
  __device__ __forceinline__ static void widen(const T& v, double* o) { o[0] = v.x; o[1] = v.y; }
};
template <> struct FzVec<float> {
  using T = float4;
  static constexpr int N = 4;
  __device__ __forceinline__ static void widen(const T& v, double* o) {
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
  }
};

struct FzShared {
  uint64_t bar[3];
  double xpart[2][kFzMaxRows];   // this CTA's row partials (tile parity)
  double wpart[2][kFzThreads / 32][kFzMaxRows];
  double rr[2][3][kFzMaxRows];   // r_R, r_N, zeta of the tile rows (tile parity)
  double red[32];
  int bad;
};

// shared memory: FzShared | beta slice (W doubles) | 3 tiles (rows x W x sizeof(TX))
template <typename TX>
__global__ void __launch_bounds__(kFzThreads, 2) kf_fused(EngineArgs a, int mode) {
  extern __shared__ __align__(128) unsigned char smem[];
  using V = FzVec<TX>;
  constexpr int VE = V::N;
  constexpr int kFzMaxV = fz_maxv<TX>();
  FzShared& sh = *reinterpret_cast<FzShared*>(smem);
  double* sbeta = reinterpret_cast<double*>(smem + ((sizeof(FzShared) + 127) & ~size_t(127)));
  const int64_t W = a.fz_w;
  TX* tiles = reinterpret_cast<TX*>(sbeta + W);
  const int R = a.fz_rows;

  State* st = a.st;
  int64_t t = 0;
  double cN = 0.25;
  bool want_z;
  if (mode == MODE_ITER) {
    if (st->done || st->dual_only) return;
    t = st->t + 1;
    cN = momentum(st->phi + 1);
    // zeta_t is needed by a bound check at t, or by a final bound pass
    want_z = is_check(t, a.prm->bci) || !isfinite(st->best_dual);
  } else {
    want_z = false;
  }
  const double cR = 0.25;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cs = a.fz_cs;
  const uint32_t crank = cs > 1 ? cluster_rank() : 0;
  const int cid = cs > 1 ? (int)cluster_id() : (int)blockIdx.x;
  const int ncl = a.fz_ncl;
  const int64_t n = a.n, ld = a.ld;
  const int64_t c0 = (int64_t)crank * W;                      // first column of this CTA
  const int64_t wvalid = max((int64_t)0, min(W, ld - c0));    // columns inside the row
  const uint32_t row_bytes = (uint32_t)(wvalid * (int64_t)sizeof(TX));
  const double* bsrc = (mode == MODE_ITER) ? a.beta + ring(t) * a.pv : a.beta;

  // beta slice (zero beyond p) and barriers
  for (int64_t j = tid; j < W; j += kFzThreads) {
    const int64_t col = c0 + j;
    sbeta[j] = col < a.p ? bsrc[col] : 0.0;
  }
  if (tid == 0) {
    mbar_init(&sh.bar[0], 1);
    mbar_init(&sh.bar[1], 1);
    mbar_init(&sh.bar[2], 1);
    sh.bad = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (cs > 1) cluster_barrier();

  // static tile schedule of this cluster: cid, cid + ncl, ... ; tile k of this
  // cluster lives in buffer k % 3
  const int64_t ntiles = a.fz_tiles;
  const int64_t mytiles = cid < ntiles ? (ntiles - cid + ncl - 1) / ncl : 0;
  auto tile_of = [&](int64_t k) -> int64_t { return cid + k * ncl; };
  auto tile_rows = [&](int64_t tile) -> int { return (int)min((int64_t)R, n - tile * R); };
  auto issue = [&](int64_t k) {
    const int64_t tile = tile_of(k);
    const int buf = (int)(k % 3);
    const int rows = tile_rows(tile);
    TX* dst = tiles + (int64_t)buf * R * W;
    if (row_bytes == 0) {
      mbar_arrive_expect(&sh.bar[buf], 0);
      return;
    }
    mbar_arrive_expect(&sh.bar[buf], row_bytes * rows);
    for (int r = 0; r < rows; ++r)
      bulk_g2s(dst + (int64_t)r * W, static_cast<const TX*>(a.X) + (tile * R + r) * ld + c0,
               row_bytes, &sh.bar[buf]);
  };
  if (tid == 0)
    for (int64_t k = 0; k < 3 && k < mytiles; ++k) issue(k);

  // per-thread vectors: v-th vector covers columns v*256*VE + tid*VE .. +VE
  const int nv = a.fz_nv;
  double accR[kFzMaxV * VE], accN[kFzMaxV * VE], accZ[kFzMaxV * VE];
#pragma unroll
  for (int i = 0; i < kFzMaxV * VE; ++i) { accR[i] = 0.0; accN[i] = 0.0; accZ[i] = 0.0; }
  double loss_acc = 0.0, f_acc[3] = {0.0, 0.0, 0.0};
  int bad = 0, gbad_R = 0, gbad_N = 0;
  uint32_t phase[3] = {0u, 0u, 0u};

  // forward partial dots of tile k into xpart[k & 1] (block-reduced, fixed order)
  auto forward = [&](int64_t k) {
    const int buf = (int)(k % 3);
    const int rows = tile_rows(tile_of(k));
    mbar_wait(&sh.bar[buf], phase[buf]);
    phase[buf] ^= 1u;
    const TX* tl = tiles + (int64_t)buf * R * W;
    double dot[kFzMaxRows];
#pragma unroll
    for (int r = 0; r < kFzMaxRows; ++r) dot[r] = 0.0;
#pragma unroll
    for (int v = 0; v < kFzMaxV; ++v) {
      if (v < nv) {
        const int64_t col = (int64_t)v * kFzThreads * VE + tid * VE;
        if (col < wvalid) {
          double b[VE];
#pragma unroll
          for (int e = 0; e < VE; ++e) b[e] = sbeta[col + e];
#pragma unroll
          for (int r = 0; r < kFzMaxRows; ++r) {
            if (r < rows) {
              double x[VE];
              V::widen(*reinterpret_cast<const typename V::T*>(tl + (int64_t)r * W + col), x);
#pragma unroll
              for (int e = 0; e < VE; ++e) dot[r] = fma(x[e], b[e], dot[r]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kFzMaxRows; ++r) {
      if (r < rows) {
        const double w = warp_sum(dot[r]);
        if (lane == 0) sh.wpart[k & 1][warp][r] = w;
      }
    }
    __syncthreads();
    if (tid < rows) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kFzThreads / 32; ++w) s += sh.wpart[k & 1][w][tid];
      sh.xpart[k & 1][tid] = s;
    }
  };
  // u for the rows of tile k from the cluster's partials; r_R, r_N, zeta
  auto gather = [&](int64_t k) {
    const int64_t tile = tile_of(k);
    const int rows = tile_rows(tile);
    const int par = (int)(k & 1);
    if (tid < rows) {
      double u = 0.0;
      for (int c = 0; c < cs; ++c)
        u += (cs > 1) ? ld_dsmem(&sh.xpart[par][tid], (uint32_t)c) : sh.xpart[par][tid];
      const int64_t row = tile * R + tid;
      const double yi = a.y[row];
      const double up = (mode == MODE_ITER) ? a.u[ring(t - 1) * n + row] : u;
      const double dlt = dsub(u, up);
      const double ugR = dadd(u, dmul(cR, dlt));   // X gamma for the two momenta (fista.py:161-162)
      const double ugN = dadd(u, dmul(cN, dlt));
      if (!isfinite(ugR)) gbad_R = 1;
      if (!isfinite(ugN)) gbad_N = 1;
      sh.rr[par][0][tid] = loss_grad(a.loss, ugR, yi);
      sh.rr[par][1][tid] = loss_grad(a.loss, ugN, yi);
      const double z = -loss_grad(a.loss, u, yi);     // zeta_t = -grad F(u_t) (fista.py:152)
      sh.rr[par][2][tid] = z;
      if (crank == 0) {
        if (mode == MODE_ITER) {
          a.u[ring(t) * n + row] = u;
        } else {
          a.u[row] = u;
          a.u[2 * n + row] = u;
        }
        if (!isfinite(u)) bad = 1;
        loss_acc += loss_term(a.loss, u, yi);
        if (want_z) conj_accumulate(a.loss, z, yi, f_acc);
      }
    }
    __syncthreads();
  };
  // transpose accumulation of tile k (rows' r from rr[k & 1])
  auto transpose = [&](int64_t k) {
    const int buf = (int)(k % 3);
    const int rows = tile_rows(tile_of(k));
    const int par = (int)(k & 1);
    const TX* tl = tiles + (int64_t)buf * R * W;
#pragma unroll
    for (int r = 0; r < kFzMaxRows; ++r) {
      if (r < rows) {
        const double rR = sh.rr[par][0][r], rN = sh.rr[par][1][r], rZ = sh.rr[par][2][r];
#pragma unroll
        for (int v = 0; v < kFzMaxV; ++v) {
          if (v < nv) {
            const int64_t col = (int64_t)v * kFzThreads * VE + tid * VE;
            if (col < wvalid) {
              double x[VE];
              V::widen(*reinterpret_cast<const typename V::T*>(tl + (int64_t)r * W + col), x);
#pragma unroll
              for (int e = 0; e < VE; ++e) {
                accR[v * VE + e] = fma(x[e], rR, accR[v * VE + e]);
                accN[v * VE + e] = fma(x[e], rN, accN[v * VE + e]);
                if (want_z) accZ[v * VE + e] = fma(x[e], rZ, accZ[v * VE + e]);
              }
            }
          }
        }
      }
    }
  };

  // software pipeline: the cluster exchange of tile k+1 overlaps the
  // transpose of tile k (split arrive / wait of the cluster barrier)
  if (mytiles > 0) {
    forward(0);
    if (cs > 1) cluster_barrier();
    else __syncthreads();
    gather(0);
  }
  for (int64_t k = 0; k < mytiles; ++k) {
    const bool more = k + 1 < mytiles;
    if (more) {
      forward(k + 1);
      if (cs > 1) cluster_arrive();
    }
    transpose(k);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();                              // tile k's buffer is free
    if (tid == 0 && k + 3 < mytiles) issue(k + 3);
    if (more) {
      if (cs > 1) cluster_wait();
      else __syncthreads();
      gather(k + 1);
    }
  }

  // ---- publish per-cluster partials -------------------------------------------
  const int64_t pv = a.pv;
#pragma unroll
  for (int v = 0; v < kFzMaxV; ++v) {
    if (v < nv) {
#pragma unroll
      for (int e = 0; e < VE; ++e) {
        const int64_t col = c0 + (int64_t)v * kFzThreads * VE + tid * VE + e;
        if (col < pv) {
          a.fz_part[(0 * (int64_t)ncl + cid) * pv + col] = accR[v * VE + e];
          a.fz_part[(1 * (int64_t)ncl + cid) * pv + col] = accN[v * VE + e];
          if (want_z) a.fz_part[(2 * (int64_t)ncl + cid) * pv + col] = accZ[v * VE + e];
        }
      }
    }
  }
  if (bad) sh.bad = 1;
  if (gbad_R) atomicOr(&sh.bad, 2);
  if (gbad_N) atomicOr(&sh.bad, 4);
  const double lsum = block_sum(loss_acc, sh.red);
  const double f0 = block_sum(f_acc[0], sh.red);
  const double f1 = block_sum(f_acc[1], sh.red);
  const double f2 = block_sum(f_acc[2], sh.red);
  if (crank == 0 && tid == 0) {
    double* cp = a.fz_cpart + 8 * (int64_t)cid;
    cp[0] = lsum;
    cp[1] = (double)sh.bad;
    cp[2] = f0;
    cp[3] = f1;
    cp[4] = f2;
  }
  if (cs > 1) cluster_barrier();  // DSMEM reads of this CTA's xpart are over
  __threadfence();
  __syncthreads();
  __shared__ int s_last;
  if (tid == 0) s_last = (atomicAdd(cnt_fused(a), 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // ---- last CTA: loss over clusters (fixed order), objective / restart ---------
  if (tid == 0) {
    *cnt_fused(a) = 0u;
    double tot = 0.0, fs0 = 0.0, fs1 = 0.0, fs2 = 0.0;
    int flags = 0;
    for (int c = 0; c < ncl; ++c) {
      const double* cp = a.fz_cpart + 8 * (int64_t)c;
      tot += __ldcg(cp);
      flags |= (int)__ldcg(cp + 1);
      fs0 += __ldcg(cp + 2);
      fs1 += __ldcg(cp + 3);
      fs2 += __ldcg(cp + 4);
    }
    a.gv[2 * pv + 0] = fs0;
    a.gv[2 * pv + 1] = fs1;
    a.gv[2 * pv + 2] = fs2;
    a.gv[2 * pv + 6] = (double)flags;   // gradient-candidate validity for KR
    a.gv[2 * pv + 7] = want_z ? 1.0 : 0.0;
    if (a.multi) {
      a.gv[2 * pv + 4] = tot;
      a.gv[2 * pv + 5] = (double)(flags & 1);
    } else if (flags & 1) {
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

// KR: reduce the per-cluster partials (fixed order), pick the candidate of
// the restart decision, slab epilogue.  One CTA per 256-column slab.
__global__ void __launch_bounds__(kK2Slab) kr_reduce(EngineArgs a, int mode, int epilogue) {
  __shared__ EpiSmem sm;
  const State* st = a.st;
  if (st->done) return;
  const int64_t pv = a.pv, p = a.p;
  const bool wg = st->dual_only == 0;
  // row-sharded: the objective (which sets dual_pending) runs after this
  // kernel, so reduce zeta whenever KF produced it
  const bool wz = epilogue ? st->dual_pending != 0 : a.gv[2 * pv + 7] != 0.0;
  const int ncl = a.fz_ncl;
  const int64_t j = (int64_t)blockIdx.x * kK2Slab + threadIdx.x;
  // restart -> phi = 1 -> c = 1/4 (candidate R); else candidate N
  const bool use_R = (mode != MODE_ITER) || st->last_restarted;
  double g = 0.0, gn = 0.0, v = 0.0;
  if (j < p) {
    if (wg || !epilogue) {
      for (int c = 0; c < ncl; ++c) g += __ldcg(a.fz_part + (0 * (int64_t)ncl + c) * pv + j);
      for (int c = 0; c < ncl; ++c) gn += __ldcg(a.fz_part + (1 * (int64_t)ncl + c) * pv + j);
    }
    if (wz)
      for (int c = 0; c < ncl; ++c) v += __ldcg(a.fz_part + (2 * (int64_t)ncl + c) * pv + j);
  }
  if (!epilogue) {  // row-sharded: both candidates go through the all-reduce
    if (j < p) {
      a.gv[j] = g;
      a.gv[2 * pv + 8 + j] = gn;
      a.gv[pv + j] = v;
    }
    return;
  }
  const double gsel = use_R ? g : gn;
  if (j < p) {
    a.gv[j] = gsel;
    a.gv[pv + j] = v;
  }
  if (wg && blockIdx.x == 0 && threadIdx.x == 0) {
    // non-finite X gamma of the chosen momentum: loss_gradient raises (model.py:215)
    const int flags = (int)a.gv[2 * pv + 6];
    if (flags & (use_R ? 2 : 4)) {
      State* sw = a.st;
      atomicExch(&sw->err, (int)ST_INVALID);
      sw->err_iter = sw->t + 1;
      sw->done = 1;
    }
  }
  const int64_t t = st->t + 1;
  const double c = momentum(st->phi);
  slab_epilogue(a, blockIdx.x, t, c, wg, wz, gsel, v, sm);
}

// row-sharded fused mode: pick the all-reduced candidate, then the epilogue
__global__ void __launch_bounds__(kK2Slab) kr_pick(EngineArgs a) {
  __shared__ EpiSmem sm;
  const State* st = a.st;
  if (st->done) return;
  const bool wg = st->dual_only == 0;
  const bool wz = st->dual_pending != 0;
  if (!wg && !wz) return;
  const int64_t pv = a.pv;
  const int64_t j = (int64_t)blockIdx.x * kK2Slab + threadIdx.x;
  const bool use_R = st->last_restarted != 0;
  const double g = j < a.p ? (use_R ? a.gv[j] : a.gv[2 * pv + 8 + j]) : 0.0;
  const double v = (wz && j < a.p) ? a.gv[pv + j] : 0.0;
  const int64_t t = st->t + 1;
  slab_epilogue(a, blockIdx.x, t, momentum(st->phi), wg, wz, g, v, sm);
}

// ---------------------------------------------------------------------------
// planning and launch
// ---------------------------------------------------------------------------
static size_t fused_smem(const EngineArgs& a) {
  const size_t es = a.dtype == F64 ? 8 : 4;
  return ((sizeof(FzShared) + 127) & ~size_t(127)) + 8 * (size_t)a.fz_w +
         3 * (size_t)a.fz_rows * (size_t)a.fz_w * es;
}

template <typename TX>
static cudaError_t fused_config(const EngineArgs& a, cudaLaunchConfig_t& cfg, cudaLaunchAttribute* at) {
  const size_t smem = fused_smem(a);
  cudaError_t e = cudaFuncSetAttribute(kf_fused<TX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (a.fz_cs > 8) {
    e = cudaFuncSetAttribute(kf_fused<TX>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cfg = cudaLaunchConfig_t{};
  cfg.gridDim = dim3((unsigned)(a.fz_cs * a.fz_ncl));
  cfg.blockDim = dim3(kFzThreads);
  cfg.dynamicSmemBytes = smem;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)a.fz_cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaSuccess;
}

int fused_plan(EngineArgs& a, int sms) {
  (void)sms;
  const int VE = a.dtype == F64 ? 2 : 4;
  const int64_t unit = (int64_t)kFzThreads * VE;   // columns per vector sweep
  const size_t es = a.dtype == F64 ? 8 : 4;
  for (int cs : {1, 2, 4, 8}) {
    const int64_t need = (a.p + cs - 1) / cs;
    const int64_t W = ((need + unit - 1) / unit) * unit;
    const int nv = (int)(W / unit);
    if (nv > (a.dtype == F64 ? fz_maxv<double>() : fz_maxv<float>())) continue;
    // rows per tile: three tiles + beta slice within 113 KB (2 CTAs per SM)
    int R = (int)((113 * 1024 - 8 * W - 1536) / (3 * W * (int64_t)es));
    R = std::min(R, kFzMaxRows);
    if (R < 1) continue;
    a.fz_cs = cs;
    a.fz_w = W;
    a.fz_nv = nv;
    a.fz_rows = R;
    a.fz_tiles = (a.n + R - 1) / R;
    a.fz_ncl = 1;   // grid of one cluster for the occupancy query
    int ncl = 0;
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute at[1];
    cudaError_t e = (a.dtype == F64) ? fused_config<double>(a, cfg, at) : fused_config<float>(a, cfg, at);
    if (e != cudaSuccess) {
      if (getenv("L0_DEBUG")) fprintf(stderr, "fused_plan: config %s\n", cudaGetErrorString(e));
      cudaGetLastError();
      return 0;
    }
    e = (a.dtype == F64) ? cudaOccupancyMaxActiveClusters(&ncl, kf_fused<double>, &cfg)
                         : cudaOccupancyMaxActiveClusters(&ncl, kf_fused<float>, &cfg);
    if (getenv("L0_DEBUG"))
      fprintf(stderr, "fused_plan: cs=%d W=%lld nv=%d R=%d smem=%zu ncl=%d (%s)\n", cs,
              (long long)W, nv, R, fused_smem(a), ncl, cudaGetErrorString(e));
    if (e != cudaSuccess || ncl < 1) {
      cudaGetLastError();
      return 0;
    }
    a.fz_ncl = (int)std::min<int64_t>(ncl, a.fz_tiles);
    return 1;
  }
  return 0;
}

cudaError_t launch_fused(const EngineArgs& a, int mode, cudaStream_t s) {
  cudaLaunchConfig_t cfg;
  cudaLaunchAttribute at[1];
  cudaError_t e = (a.dtype == F64) ? fused_config<double>(a, cfg, at) : fused_config<float>(a, cfg, at);
  if (e != cudaSuccess) return e;
  cfg.stream = s;
  if (a.dtype == F64) e = cudaLaunchKernelEx(&cfg, kf_fused<double>, a, mode);
  else e = cudaLaunchKernelEx(&cfg, kf_fused<float>, a, mode);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_fused_reduce(const EngineArgs& a, int mode, cudaStream_t s) {
  if (a.multi) {
    kr_reduce<<<a.k2_slabs, kK2Slab, 0, s>>>(a, mode, 0);
  } else {
    kr_reduce<<<a.k2_slabs, kK2Slab, 0, s>>>(a, mode, 1);
  }
  return cudaGetLastError();
}

cudaError_t launch_fused_pick(const EngineArgs& a, cudaStream_t s) {
  kr_pick<<<a.k2_slabs, kK2Slab, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace l0
