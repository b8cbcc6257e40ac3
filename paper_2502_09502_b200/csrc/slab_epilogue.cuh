// Per-slab epilogue of the transpose pass: everything of the prox step that is
// elementwise in the coordinates runs here, in parallel over the k2_slabs
// slabs of 256 columns (one thread per column), so the single-CTA K3 only
// touches the window of coordinates the PAVA pool can reach.
//
//   gradient step, gamma, sort key |rho gamma|         fista.py:161-163, prox.py:106-111
//   outputs of every coordinate that cannot be in the pool: fixed-zero -> 0,
//     fixed-one -> Huber prox, free keys below the window threshold -> tail
//     singletons (out = mu), elementwise / pass-through cases   fista.py:104-128, prox.py:104-110
//   window candidates (keys >= theta), compacted in index order
//   partial sums / maxima of |beta+| for g(beta+)       perspective.py:85-92
//   bound check: Huber values of X^T zeta / 2 l2, per-slab top-32 and
//     fixed-one sums for g*                            perspective.py:143-159
//
// theta is chosen by the previous K3 from the sorted window (State::theta);
// if the pool reaches below it K3 detects it and recomputes (slow path).
#pragma once

#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>

#include "engine.cuh"
#include "sortnet.cuh"

namespace l0 {

struct EpiSmem {
  union {
    typename cub::BlockScan<int, kK2Slab>::TempStorage scan;
    typename cub::BlockRadixSort<double, kK2Slab, 1>::TempStorage sort;
  } u;
  double red[96];
};

// how the free coordinates are treated (prox.py:104-112): 0 pass-through,
// 1 elementwise Huber prox, 2 sort + PAVA
__device__ __forceinline__ int prox_case(const Params* P, int64_t p) {
  const int64_t nf = P->node_mode ? P->n_free : p;
  const int64_t kk = P->node_mode ? P->k_rem : P->k;
  return (kk <= 0 || nf == 0) ? 0 : (kk >= nf ? 1 : 2);
}

// blockDim.x == kK2Slab; columns slab*kK2Slab + threadIdx.x
__device__ void slab_epilogue(const EngineArgs& a, int slab, int64_t t, double c, bool has_g,
                              bool has_z, double g_in, double v_in, EpiSmem& sm) {
  const Params* P = a.prm;
  const int tid = threadIdx.x;
  const int64_t j = (int64_t)slab * kK2Slab + tid;
  const bool valid = j < a.p;
  const bool node = P->node_mode != 0;
  const int cls = (valid && node) ? a.mask[j] : FREE;
  if (has_g) {
    const int how = prox_case(P, a.p);
    const double theta = a.st->theta;
    const double rho = P->rho, M = P->M;
    double key = -1.0, res = 0.0, gam = 0.0, mu = 0.0;
    bool cand = false;
    if (valid) {
      // fista.py:161-163 (gamma, gradient step), fista.py:102/:107/:119 (mu)
      const double b1 = a.beta[ring(t - 1) * a.pv + j];
      const double b2 = a.beta[ring(t - 2) * a.pv + j];
      gam = dadd(b1, dmul(c, dsub(b1, b2)));
      gam = dsub(gam, ddiv(g_in, P->L));
      a.gam[j] = gam;
      mu = dmul(rho, gam);
      key = (cls == FREE) ? fabs(mu) : -1.0;
      a.key[j] = key;
      cand = how == 2 && cls == FREE && key > 0.0 && key >= theta;
      if (cls == FIXED_ZERO) res = 0.0;
      else if (cls == FIXED_ONE || how == 1) res = dsub(gam, ddiv(dmul(dsign(mu), hprox(fabs(mu), rho, M)), rho));
      else res = dsub(gam, ddiv(mu, rho));  // pass-through / tail singleton: out = mu
      if (!cand) {
        a.beta[ring(t) * a.pv + j] = res;
        a.scratch[j] = (cls == FREE) ? fabs(res) : -1.0;
      }
    }
    const bool free_out = valid && cls == FREE && !cand;
    const double ab = free_out ? fabs(res) : 0.0;
    const double below = (valid && how == 2 && cls == FREE && key > 0.0 && !cand) ? key : 0.0;
    // candidate compaction in index order
    int pos = 0, count = 0;
    cub::BlockScan<int, kK2Slab>(sm.u.scan).ExclusiveSum(cand ? 1 : 0, pos, count);
    if (cand) {
      a.cand_key[(int64_t)slab * kK2Slab + pos] = key;
      a.cand_idx[(int64_t)slab * kK2Slab + pos] = (int)j;
    }
    double s = ab, m = ab, bl = below;
    block_sum_max_max(s, m, bl, sm.red);
    if (tid == 0) {
      a.slab_cnt[slab] = count;
      a.slab_sum[slab] = s;
      a.slab_max[slab] = m;
      a.slab_below[slab] = bl;
    }
  }
  if (has_z) {
    // H_M(v / 2 l2) of the bound check (perspective.py:151)
    double h = -1.0, hf = 0.0;
    if (valid) {
      const double hv = huber(ddiv(v_in, P->two_l2), P->M);
      if (cls == FREE) h = hv;
      else if (cls == FIXED_ONE) hf = hv;
      a.hval[j] = h;
    }
    const double fs = block_sum(hf, sm.red);
    double kv[1] = {h};
    __syncthreads();
    cub::BlockRadixSort<double, kK2Slab, 1>(sm.u.sort).SortDescending(kv);
    // blocked output: thread t holds rank t
    if (tid < kHTop) a.slab_htop[(int64_t)slab * kHTop + tid] = kv[0];
    if (tid == 0) a.slab_hfone[slab] = fs;
  }
}

}  // namespace l0
