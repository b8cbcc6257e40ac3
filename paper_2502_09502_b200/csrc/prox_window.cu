// K3 (FISTA loop variant): prox via a windowed top-of-order sort.
//
// The exact prox needs the stable descending order of |mu| only as far as the
// merged PAVA pool can reach: every free coordinate behind the pool end c* is
// a tail singleton whose output is mu itself (prox.py:104-116 with nu = x), and
// the pool never reaches a zero key.  So instead of sorting all p keys
// (SURVEY.md §7.1-4), K3 repeatedly
//   1. selects the next window W = {lb <= bits(|mu|) < ub} of at most kWinCap
//      keys by an MSD radix histogram (12+13+13+13+13 bits, usually one pass),
//   2. compacts W in ascending index order and block-sorts it (CUB, stable),
//      appending it to the sorted prefix (keys in later windows are strictly
//      smaller, so the concatenation IS the stable descending order),
//   3. runs the closed-form single-pool PAVA search on the prefix, with the
//      largest unsorted key as the right boundary,
// until the pool closes inside the prefix.  On C2 one window of <= 4096 keys
// suffices from the second iteration on (pool end 6165 -> 755).
//
// The scatter then writes beta+ for every coordinate, and g(beta+) is taken
// from the prefix (verified against the largest |beta+| outside the window,
// radix-select fallback).  Same arithmetic as prox_post_sort (prox.cu).

#include <climits>

#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>

#include "control.cuh"
#include "engine.cuh"
#include "prox.cuh"
#include "sortnet.cuh"

namespace l0 {

constexpr int kWinThreads = 512;
constexpr int kWinIpt = 8;
constexpr int kWinCap = kWinThreads * kWinIpt;  // 4096 keys per window
constexpr int kHistBins = 8192;                 // 13-bit digits

struct WinSmem {
  union {
    unsigned hist[kHistBins];
    typename cub::BlockScan<double, kWinThreads>::TempStorage dscan;
    typename cub::BlockScan<int, kWinThreads>::TempStorage iscan;
  } u;
  double wkey[kWinCap];
  int widx[kWinCap];
  double wtail[kWinCap];
  double mkey[kWinCap];   // merge ping-pong buffer
  int midx[kWinCap];
  // window selection results
  unsigned long long sel_lb;
  int sel_count;
  int sel_state;  // 0 searching, 1 done, 2 overflow
  unsigned long long sel_prefix;
  int sel_above;
  // PAVA search results
  int res;        // 0 undecided, 1 pool found, 2 no pool, 3 extend
  int64_t astar, cstar;
  double vstar;
  int wflag[32];
  int64_t wc[32];
  double wv[32];
  double red[32];
  double xnext;
  int has_next;
};

__device__ __forceinline__ unsigned long long key_bits(double k) {
  return (unsigned long long)__double_as_longlong(k);
}

// MSD radix selection of the next window among positive keys with bits < ub.
// Returns in sm.sel_lb / sm.sel_count (count <= cap) or sel_state = 2 on an
// exact tie group larger than cap.
__device__ void select_window(const double* key, int64_t p, unsigned long long ub, int cap,
                              WinSmem& sm) {
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) {
    sm.sel_state = 0;
    sm.sel_prefix = 0ull;
    sm.sel_above = 0;
  }
  __syncthreads();
  int shift = 64;
  for (int level = 0; level < 5; ++level) {
    const int w = level == 0 ? 12 : 13;   // 12 + 4 x 13 = 64 bits
    const int hi_shift = shift;  // bits >= hi_shift must equal the prefix
    shift -= w;
    const unsigned long long prefix = sm.sel_prefix;
    const unsigned mask = (1u << w) - 1u;
    for (int i = tid; i < kHistBins; i += kWinThreads) sm.u.hist[i] = 0u;
    __syncthreads();
    // U keys per thread in flight per step (the single CTA is latency-bound on L2)
    constexpr int U = 8;
    for (int64_t j0 = 0; j0 < p; j0 += (int64_t)U * kWinThreads) {
      double kv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t j = j0 + (int64_t)u * kWinThreads + tid;
        kv[u] = j < p ? __ldcg(key + j) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int digit = -1;
        const double k = kv[u];
        if (k > 0.0) {
          const unsigned long long b = key_bits(k);
          const bool in_prefix = hi_shift >= 64 || (b >> hi_shift) == (prefix >> hi_shift);
          if (b < ub && in_prefix) digit = (int)((b >> shift) & mask);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, digit);
        if (digit >= 0 && lane == __ffs(peers) - 1) atomicAdd(&sm.u.hist[digit], (unsigned)__popc(peers));
      }
    }
    __syncthreads();
    // bins in descending order: thread t owns bins kHistBins-1-B*t .. kHistBins-B-B*t
    constexpr int B = kHistBins / kWinThreads;
    unsigned c8[B];
    int s = 0;
#pragma unroll
    for (int q = 0; q < B; ++q) {
      const int d = kHistBins - 1 - (tid * B + q);
      c8[q] = (d >= 0 && d <= (int)mask) ? sm.u.hist[d] : 0u;
      s += (int)c8[q];
    }
    __syncthreads();
    int excl = 0, total = 0;
    cub::BlockScan<int, kWinThreads>(sm.u.iscan).ExclusiveSum(s, excl, total);
    const int above = sm.sel_above;
    if (tid == 0 && above + total <= cap) {
      // everything that remains fits
      sm.sel_lb = prefix;
      sm.sel_count = above + total;
      sm.sel_state = 1;
    }
    if (above + total > cap && above + excl <= cap && above + excl + s > cap) {
      int cum = above + excl;
      for (int q = 0; q < B; ++q) {
        const int d = kHistBins - 1 - (tid * B + q);
        if (cum + (int)c8[q] > cap) {
          // bin d crosses the capacity: stop above it, or refine into it
          const bool enough = cum >= cap / 2 || cum > 0 && level == 4;
          if (enough || level == 4) {
            if (cum > 0) {
              sm.sel_lb = prefix | ((unsigned long long)(d + 1) << shift);
              sm.sel_count = cum;
              sm.sel_state = 1;
            } else {
              sm.sel_state = 2;  // exact tie group larger than the window
            }
          } else {
            sm.sel_prefix = prefix | ((unsigned long long)d << shift);
            sm.sel_above = cum;
          }
          break;
        }
        cum += (int)c8[q];
      }
    }
    __syncthreads();
    if (sm.sel_state != 0) return;
  }
}

// Compact the window {lb <= bits < ub, key > 0} in ascending index order into
// sm.wkey/widx; also the largest positive key below the window (sm.xnext).
__device__ void compact_window(const double* key, int64_t p, unsigned long long lb,
                               unsigned long long ub, WinSmem& sm) {
  const int tid = threadIdx.x;
  const int64_t per = (p + kWinThreads - 1) / kWinThreads;
  const int64_t j0 = min(p, (int64_t)tid * per), j1 = min(p, j0 + per);
  int cnt = 0;
  double below = 0.0;
#pragma unroll 8
  for (int64_t j = j0; j < j1; ++j) {
    const double k = __ldcg(key + j);
    if (k > 0.0) {
      const unsigned long long b = key_bits(k);
      if (b >= lb && b < ub) ++cnt;
      else if (b < lb) below = fmax(below, k);
    }
  }
  int off = 0;
  cub::BlockScan<int, kWinThreads>(sm.u.iscan).ExclusiveSum(cnt, off);
#pragma unroll 8
  for (int64_t j = j0; j < j1; ++j) {
    const double k = __ldcg(key + j);
    if (k > 0.0) {
      const unsigned long long b = key_bits(k);
      if (b >= lb && b < ub) {
        sm.wkey[off] = k;
        sm.widx[off] = (int)j;
        ++off;
      }
    }
  }
  below = block_max(below, sm.red);
  if (tid == 0) sm.xnext = below;
  __syncthreads();
}

// Closed-form pool search on the sorted prefix xs[0..len) (len > kk) with the
// boundary element x_len = xnext (has_next) or none (len == all positives and
// no zero keys follow).  Sets sm.res: 1 pool, 2 no pool, 3 prefix too short.
__device__ void window_search(const double* xs, const double* tail, int64_t len, int64_t kk,
                              double rho, double M, bool has_next, double xnext, WinSmem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  if (tid == 0) sm.res = 0;
  __syncthreads();
  // first merge at k-1 | k (prox.py:80)
  const double xk = (kk < len) ? xs[kk] : xnext;
  if (!(xk > hprox(xs[kk - 1], rho, M))) {
    if (tid == 0) sm.res = 2;
    __syncthreads();
    return;
  }
  if (kk >= len) {  // the pool starts at an unsorted key
    if (tid == 0) sm.res = 3;
    __syncthreads();
    return;
  }
  for (int64_t base = kk - 1; base >= 0; base -= nw) {
    const int64_t aa = base - warp;
    int flag = 0;  // 1 valid, 2 beyond the prefix
    int64_t cA = 0;
    double VA = 0.0;
    if (aa >= 0) {
      double hs = 0.0;
      for (int64_t j = aa + lane; j < kk; j += 32) hs += xs[j];
      hs = warp_sum(hs);
      const double Pw = dmul(rho, (double)(kk - aa));
      auto pred = [&](int64_t c) -> int {  // 1 true, 0 false; c in [kk, len-1]
        const double V = hprox(ddiv(dadd(hs, tail[c]), (double)(c - aa + 1)),
                               ddiv(Pw, (double)(c - aa + 1)), M);
        const double xn = (c + 1 < len) ? xs[c + 1] : (has_next ? xnext : -1.0);
        return xn <= V ? 1 : 0;
      };
      int64_t lo = kk, hi = len - 1;
      // pred(len-1) decides whether the pool closes inside the prefix
      const int plast = __shfl_sync(0xffffffffu, lane == 0 ? pred(hi) : 0, 0);
      if (!plast) {
        flag = 2;
      } else {
        while (lo < hi) {
          const int64_t span = hi - lo;
          const int64_t c = lo + (span * lane) / 32;
          const bool pr = pred(c);
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
        VA = hprox(ddiv(dadd(hs, tail[cA]), (double)(cA - aa + 1)),
                   ddiv(Pw, (double)(cA - aa + 1)), M);
        flag = (aa == 0 || hprox(xs[aa - 1], rho, M) >= VA) ? 1 : 0;
      }
    }
    if (lane == 0) {
      sm.wflag[warp] = flag;
      sm.wc[warp] = cA;
      sm.wv[warp] = VA;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 0; w < nw && base - w >= 0; ++w) {
        if (sm.wflag[w] == 2) { sm.res = 3; break; }
        if (sm.wflag[w] == 1) {
          sm.res = 1;
          sm.astar = base - w;
          sm.cstar = sm.wc[w];
          sm.vstar = sm.wv[w];
          break;
        }
      }
    }
    __syncthreads();
    if (sm.res != 0) return;
  }
}

// Sort the window held in sm.wkey/widx[0..cnt) and append it to the sorted
// prefix at position len (global xs/perm/tail; the window also stays sorted
// in shared memory with its tail sums in sm.wtail); the tail prefix sums over
// positions >= kk continue from *carry.
template <int E>
__device__ void sort_window_regs(WinSmem& sm, int cnt) {
  double k[E];
  int id[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int s = e * kWinThreads + threadIdx.x;
    k[e] = s < cnt ? sm.wkey[s] : -CUDART_INF;
    id[e] = s < cnt ? sm.widx[s] : INT_MAX;
  }
  __syncthreads();
  bitonic_regs<kWinThreads, E>(k, id, sm.mkey, sm.midx);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    sm.wkey[e * kWinThreads + threadIdx.x] = k[e];
    sm.widx[e * kWinThreads + threadIdx.x] = id[e];
  }
  __syncthreads();
}

// Large windows: each warp sorts a run of 32 * E pairs in registers (shuffles
// only), then the kWinThreads / 32 sorted runs are merged pairwise by merge
// path (sortnet.cuh merge_runs_path) -- far fewer block barriers than a block
// bitonic.
template <int E>
__device__ void sort_window_runs(WinSmem& sm, int cnt) {
  constexpr int RUN = 32 * E;
  constexpr int NW = kWinThreads / 32;
  static_assert(RUN * NW == kWinCap, "runs cover the window");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double k[E];
  int id[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int s = warp * RUN + e * 32 + lane;
    k[e] = s < cnt ? sm.wkey[s] : -CUDART_INF;
    id[e] = s < cnt ? sm.widx[s] : INT_MAX - s;   // distinct: the co-rank merge needs a strict order
  }
  __syncthreads();
  bitonic_warp<E>(k, id, lane);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int s = warp * RUN + e * 32 + lane;
    sm.wkey[s] = k[e];
    sm.widx[s] = id[e];
  }
  __syncthreads();
  // merge path (one co-rank search per thread and level; the per-element
  // co-ranking of merge_runs took ~75 us on 4096 keys: C2's first iterations)
  const int res = merge_runs_path<kWinCap / kWinThreads>(sm.wkey, sm.widx, sm.mkey, sm.midx, RUN, NW);
  if (res) {
    for (int s = threadIdx.x; s < cnt; s += kWinThreads) {
      sm.wkey[s] = sm.mkey[s];
      sm.widx[s] = sm.midx[s];
    }
  }
  __syncthreads();
}

__device__ void sort_append(const EngineArgs& a, int cnt, int64_t len, int64_t kk, double* carry,
                            WinSmem& sm, bool presorted = false) {
  const int tid = threadIdx.x;
  if (!presorted) {
    if (cnt <= kWinThreads) sort_window_regs<1>(sm, cnt);
    else if (cnt <= 2 * kWinThreads) sort_window_regs<2>(sm, cnt);
    else if (cnt <= 4 * kWinThreads) sort_window_regs<4>(sm, cnt);
    else sort_window_runs<8>(sm, cnt);
  }
  // tail prefix sums: blocked ranges of kWinIpt positions per thread
  double loc = 0.0;
#pragma unroll
  for (int i = 0; i < kWinIpt; ++i) {
    const int s = tid * kWinIpt + i;
    if (s < cnt && len + s >= kk) loc += sm.wkey[s];
  }
  double excl = 0.0;
  cub::BlockScan<double, kWinThreads>(sm.u.dscan).ExclusiveSum(loc, excl);
  double run = *carry + excl;
#pragma unroll
  for (int i = 0; i < kWinIpt; ++i) {
    const int s = tid * kWinIpt + i;
    if (s < cnt) {
      const int64_t pos = len + s;
      const double x = sm.wkey[s];
      a.xs[pos] = x;
      a.perm[pos] = sm.widx[s];
      if (pos >= kk) {
        run += x;
        a.tail[pos] = run;
      }
      sm.wtail[s] = run;
      if (s == cnt - 1) sm.red[0] = run;  // running tail sum at the window's end
    }
  }
  __syncthreads();
  *carry = sm.red[0];
  __syncthreads();
}

// Fenchel bound from the slab epilogue's products (fista.py:150-157).  With
// k <= 32 the top-k Huber values are among the per-slab top-32 lists; their
// top-k sum is a radix selection over those lists (the bitonic sort of all of
// them is kept behind a constant for comparison).
constexpr bool kSortHtopLists = false;
__device__ int dual_step_slabs(const EngineArgs& a, ProxSmem& ps, WinSmem& ws) {
  const Params* P = a.prm;
  State* st = a.st;
  const int64_t p = a.p;
  const double acc[3] = {a.gv[2 * a.pv], a.gv[2 * a.pv + 1], a.gv[2 * a.pv + 2]};
  const double fstar = conj_finish(P->loss, acc);
  double d = -CUDART_INF;
  if (isfinite(fstar)) {
    const bool node = P->node_mode != 0;
    const int S = a.k2_slabs;
    double fs = 0.0;
    if (node)
      for (int s = threadIdx.x; s < S; s += blockDim.x) fs += a.slab_hfone[s];
    fs = block_sum(fs, ps.red);
    const int64_t kg = node ? P->k_g : P->k;
    const int64_t nfree = node ? P->n_free : p;
    double top;
    const int64_t m = (int64_t)S * kHTop;
    if (kg <= kHTop && m <= kWinCap && kSortHtopLists) {
      // the global top-kg is among the per-slab top-32 lists: sort them
      const int n = pow2_at_least(m > 2 ? (int)m : 2);
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        ws.wkey[i] = i < m ? a.slab_htop[i] : -CUDART_INF;
        ws.widx[i] = i;
      }
      __syncthreads();
      bitonic_desc(ws.wkey, ws.widx, n);
      double sacc = 0.0;
      if (threadIdx.x == 0) {
        for (int64_t i = 0; i < kg && i < n; ++i) {
          const double h = ws.wkey[i];
          if (h < 0.0) break;
          sacc += h;
        }
        ps.gfree = sacc;
      }
      __syncthreads();
      top = ps.gfree;
    } else if (kg <= kHTop) {
      double c = 0.0;
      for (int64_t i = threadIdx.x; i < m; i += blockDim.x) c += a.slab_htop[i] >= 0.0 ? 1.0 : 0.0;
      const int64_t cnt = (int64_t)block_sum(c, ps.red);
      top = block_topk_sum(a.slab_htop, m, kg, cnt, ps.sel, ps.red);
    } else {
      top = block_topk_sum(a.hval, p, kg, nfree, ps.sel, ps.red);
    }
    const double gstar = node ? dadd(fs, top) : top;
    d = dsub(-fstar, dmul(P->two_l2, gstar));
  }
  if (threadIdx.x == 0) {
    bound_update(st, P, d);
    ps.done = st->done;
  }
  __syncthreads();
  return ps.done;
}

// K3 body for one solve (the single engine's CTA, or one node's CTA of the
// batched engine).  Returns 1 when beta+ was produced (0: finished / bound only).
__device__ int prox_window_body(const EngineArgs& a, ProxSmem& ps, WinSmem& sm) {
  const State* st0 = a.st;
  if (st0->done) return 0;
  L0_STAMP(a.st, 0);
  if (st0->dual_pending) {
    if (dual_step_slabs(a, ps, sm)) return 0;
  }
  if (a.st->dual_only) return 0;
  const Params* P = a.prm;
  State* st = a.st;
  const int tid = threadIdx.x;
  const int64_t p = a.p;
  const bool node = P->node_mode != 0;
  const int64_t nf = node ? P->n_free : p;
  const int64_t kk = node ? P->k_rem : P->k;
  const int64_t kg = node ? P->k_g : P->k;
  const double rho = P->rho, M = P->M;
  const int how = prox_case(P, p);
  double* out = a.beta + ring(st->t + 1) * a.pv;
  const int S = a.k2_slabs;

  int64_t len = 0;                      // sorted prefix length
  unsigned long long ub = ~0ull;        // keys of the next window are below ub
  double carry = 0.0;                   // running tail prefix sum
  bool dirty = false;                   // slab partials no longer describe the outputs
  if (tid == 0) sm.res = 2;
  __syncthreads();
  L0_STAMP(st, 1);
  if (how == 2) {
    // ---- fast path: the candidates K2 compacted per slab (keys >= theta) -----
    const double theta = st->theta;
    bool fast = theta > 0.0 && S <= kWinThreads;
    int total = 0;
    if (fast) {
      // offsets of the per-slab lists (slab order = index order)
      const int c = tid < S ? a.slab_cnt[tid] : 0;
      int ex = 0;
      cub::BlockScan<int, kWinThreads>(sm.u.iscan).ExclusiveSum(c, ex, total);
      __syncthreads();
      if (tid < S) sm.u.hist[tid] = (unsigned)ex;
      if (tid == 0) sm.u.hist[S] = (unsigned)total;
      __syncthreads();
      fast = total > kk && total <= kWinCap;
    }
    if (fast) {
      const int warp = tid >> 5, lane = tid & 31;
      for (int sidx = warp; sidx < S; sidx += kWinThreads / 32) {
        const int c = a.slab_cnt[sidx];
        const int o = (int)sm.u.hist[sidx];
        for (int i = lane; i < c; i += 32) {
          sm.wkey[o + i] = a.cand_key[(int64_t)sidx * kK2Slab + i];
          sm.widx[o + i] = a.cand_idx[(int64_t)sidx * kK2Slab + i];
        }
      }
      __syncthreads();
      L0_STAMP(st, 2);
      double below = 0.0;
      for (int sidx = tid; sidx < S; sidx += kWinThreads) below = fmax(below, a.slab_below[sidx]);
      below = block_max(below, sm.red);
      L0_STAMP(st, 3);
      sort_append(a, total, 0, kk, &carry, sm);
      L0_STAMP(st, 4);
      len = total;
      ub = key_bits(theta);
      window_search(sm.wkey, sm.wtail, len, kk, rho, M, nf > len, below, sm);
      L0_STAMP(st, 5);
      if (sm.res == 3) {                 // pool reaches below theta: extend windows
        dirty = true;
        if (tid == 0) st->win_ext += 1;
      }
    } else {
      dirty = true;
      if (tid == 0) st->slow_prox += 1;
      if (tid == 0) sm.res = 3;
      __syncthreads();
    }
    // ---- slow path / extension: windows selected over all remaining keys ---
    bool more = true;
    while (sm.res == 3 && more) {
      select_window(a.key, p, ub, kWinCap, sm);
      if (sm.sel_state == 2) {   // tie group > kWinCap: the host falls back to the full sort
        if (tid == 0) { atomicExch(&st->err, (int)ST_TIE_OVERFLOW); st->done = 1; }
        return 0;
      }
      const unsigned long long lb = sm.sel_lb;
      const int cnt = sm.sel_count;
      compact_window(a.key, p, lb, ub, sm);
      const double xn = sm.xnext;
      sort_append(a, cnt, len, kk, &carry, sm);
      len += cnt;
      ub = lb;
      more = xn > 0.0;
      const bool has_next = more || (len < nf);
      if (len > kk || !more) {
        window_search(a.xs, a.tail, len, kk, rho, M, has_next, more ? xn : 0.0, sm);
        if (!more && sm.res == 3) {
          if (tid == 0) sm.res = 2;
          __syncthreads();
        }
      } else {
        if (tid == 0) sm.res = 3;
        __syncthreads();
      }
    }
  }
  const int64_t astar = (how == 2 && sm.res == 1) ? sm.astar : INT64_MAX;
  const int64_t cstar = (how == 2 && sm.res == 1) ? sm.cstar : -1;
  const double vstar = sm.vstar;
  record_prox(a.prox_rec, a.prox_rec_cap, a.prox_rec_w, a.perm, st->t + 1, how,
              (how == 2 && sm.res == 1) ? 1 : 0, astar, cstar, len, dirty ? 1 : 0, nf);

  L0_STAMP(st, 6);
  // ---- scatter ----------------------------------------------------------------
  const unsigned long long lb_last = ub;
  const int64_t kkg = kg < nf ? kg : nf;
  const int64_t W = min(len, kkg + 64);
  double total = 0.0, amax = 0.0, rest = 0.0;
  if (dirty) {
    // recompute every non-prefix coordinate (K2's speculative outputs cover a
    // smaller prefix than the one sorted here)
#pragma unroll 4
    for (int64_t j = tid; j < p; j += kWinThreads) {
      const int cls = node ? a.mask[j] : FREE;
      const double gin = a.gam[j];
      const double mu = dmul(rho, gin);
      const double k = a.key[j];
      const bool in_prefix = cls == FREE && k > 0.0 && key_bits(k) >= lb_last;
      if (in_prefix) continue;
      double res;
      if (cls == FIXED_ZERO) res = 0.0;
      else if (cls == FIXED_ONE) res = dsub(gin, ddiv(dmul(dsign(mu), hprox(fabs(mu), rho, M)), rho));
      else res = dsub(gin, ddiv(mu, rho));
      out[j] = res;
      if (cls == FREE) {
        const double ab = fabs(res);
        total += ab;
        amax = fmax(amax, ab);
        rest = fmax(rest, ab);
        a.scratch[j] = ab;
      } else {
        a.scratch[j] = -1.0;
      }
    }
  } else {
    // non-candidates were written by K2's slab epilogue; fixed-order partials
    for (int sidx = tid; sidx < S; sidx += kWinThreads) {
      total += a.slab_sum[sidx];
      amax = fmax(amax, a.slab_max[sidx]);
    }
    rest = amax;
  }
  const bool smem_prefix = !dirty;   // fast path: the whole prefix is the smem window
  if (how == 2) {
#pragma unroll 4
    for (int64_t pos = tid; pos < len; pos += kWinThreads) {
      const int j = smem_prefix ? sm.widx[pos] : a.perm[pos];
      const double x = smem_prefix ? sm.wkey[pos] : a.xs[pos];
      const double gin = a.gam[j];
      const double mu = dmul(rho, gin);
      double nu;
      if (pos < astar) nu = (pos < kk) ? hprox(x, rho, M) : x;
      else if (pos <= cstar) nu = vstar;
      else nu = (pos < kk) ? hprox(x, rho, M) : x;
      const double res = dsub(gin, ddiv(dmul(nu, dsign(mu)), rho));
      out[j] = res;
      const double ab = fabs(res);
      total += ab;
      amax = fmax(amax, ab);
      if (pos < W) ps.cand[pos] = ab;
      else rest = fmax(rest, ab);
      a.scratch[j] = ab;
    }
  }
  __syncthreads();
  total = block_sum(total, ps.red);
  amax = block_max(amax, ps.red);
  rest = block_max(rest, ps.red);

  L0_STAMP(st, 7);
  // ---- g(beta+) (perspective.py:76-132) ----------------------------------------
  double fone_val = 0.0;
  bool fone_bad = false;
  if (tid == 0 && node) {
    double s2 = 0.0;
    for (int64_t i = 0; i < P->n_fone; ++i) {
      const double b = out[a.fone[i]];
      if (fabs(b) > dmul(M, dadd(1.0, kFeasRtol))) fone_bad = true;
      s2 = fma(b, b, s2);
    }
    fone_val = dmul(0.5, s2);
  }
  double gfree = 0.0;
  int path = 0;
  if (nf == 0) path = 2;
  else if (amax > dmul(M, dadd(1.0, kFeasRtol))) { gfree = CUDART_INF; path = 2; }
  else if (total > dmul(dmul((double)kg, M), dadd(1.0, kFeasRtol))) { gfree = CUDART_INF; path = 2; }
  else if (kg == 0) path = 2;
  if (path == 0) {
    if (how == 2 && W >= kkg && W <= kCandCap) {
      block_rank_sort_desc(ps.cand, ps.cand2, (int)W);
      if (rest > ps.cand2[kkg - 1]) path = 1;
    } else {
      path = 1;
    }
    if (path == 1 && kkg > kCandCap) {
      if (tid == 0) { atomicExch(&st->err, (int)ST_UNSUPPORTED); st->done = 1; }
      return 0;
    }
    if (path == 1) {
      __syncthreads();
      double tau;
      int64_t cgt;
      block_kth_largest(a.scratch, p, kkg, ps.sel, &tau, &cgt);
      if (tid == 0) ps.ncand = 0;
      __syncthreads();
      for (int64_t j = tid; j < p; j += kWinThreads) {
        const double x = a.scratch[j];
        if (x > tau) ps.cand[atomicAdd(&ps.ncand, 1)] = x;
      }
      __syncthreads();
      for (int64_t i = cgt + tid; i < kkg; i += kWinThreads) ps.cand[i] = tau;
      __syncthreads();
      block_rank_sort_desc(ps.cand, ps.cand2, (int)kkg);
      if (tid == 0) st->topk_fallbacks += 1;
    }
    if (tid < 32) {
      const double g = envelope_from_top(ps.cand2, kkg, total);
      if (tid == 0) ps.gfree = g;
    }
    __syncthreads();
    gfree = ps.gfree;
  }
  if (tid == 0) {
    double g = gfree;
    if (node) g = fone_bad ? CUDART_INF : dadd(dadd(0.0, fone_val), gfree);
    st->g_next = g;
    // window threshold for the next iteration's K2: keep ~2x the pool (>= 1536
    // keys, <= 3/4 of the window capacity) above it
    if (how == 2 && len > 0) {
      // window for the next iteration: the pool plus a 25% (>= 64 keys) margin
      int64_t want = kk + 64;
      if (cstar >= 0) {
        const int64_t c1 = cstar + 1;
        want = max(want, c1 + max((int64_t)64, c1 / 4));
      }
      want = min(want, (int64_t)(3 * kWinCap / 4));
      const int64_t pos = min(len - 1, want);
      st->theta = a.xs[pos];
    }
  }
  L0_STAMP(st, 8);
  return 1;
}

__global__ void __launch_bounds__(kWinThreads, 1) k3_prox_window(EngineArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ProxSmem& ps = *reinterpret_cast<ProxSmem*>(smem_raw);
  WinSmem& sm = *reinterpret_cast<WinSmem*>(smem_raw + ((sizeof(ProxSmem) + 255) & ~size_t(255)));
  pdl_wait();     // KR (or the SPEC kernel's K2) of the previous iteration
  pdl_launch();   // KF may become resident and load its first X tiles while the prox runs
  prox_window_body(a, ps, sm);
}

size_t prox_window_smem() {
  return ((sizeof(ProxSmem) + 255) & ~size_t(255)) + sizeof(WinSmem);
}

cudaError_t launch_prox_window(const EngineArgs& a, cudaStream_t s) {
  const size_t smem = prox_window_smem();
  cudaError_t e = cudaFuncSetAttribute(k3_prox_window, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(kWinThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  pdl_attr(cfg, at, a.pdl != 0);
  e = cudaLaunchKernelEx(&cfg, k3_prox_window, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace l0
