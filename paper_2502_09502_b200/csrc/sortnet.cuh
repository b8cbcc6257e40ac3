// Small in-block sorting networks for (key, index) pairs in shared memory.
//
// Order: descending key, ties by ascending index -- a total order, so every
// result equals numpy's stable argsort of -|mu| (prox.py:111) on the same
// keys, independent of input order.
#pragma once

#include <climits>

#include "common.cuh"

namespace l0 {

// a precedes b in the sorted order
__device__ __forceinline__ bool precedes(double ka, int ia, double kb, int ib) {
  return ka > kb || (ka == kb && ia < ib);
}

__device__ __forceinline__ int pow2_at_least(int c) {
  int n = 1;
  while (n < c) n <<= 1;
  return n;
}

// Bitonic sort of n (power of two) pairs; every thread of the block takes part.
__device__ void bitonic_desc(double* key, int* idx, int n) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < (n >> 1); t += blockDim.x) {
        const int i = 2 * t - (t & (j - 1));
        const int l = i + j;
        const double ki = key[i], kl = key[l];
        const int ii = idx[i], il = idx[l];
        const bool ordered = precedes(ki, ii, kl, il);
        const bool want = (i & k) == 0;  // this block sorts toward the final order
        if (want != ordered) {
          key[i] = kl; key[l] = ki;
          idx[i] = il; idx[l] = ii;
        }
      }
      __syncthreads();
    }
  }
}

// In-thread compare-exchange stage of a register bitonic sort: element e of
// this thread is position e * stride + lane0, partners differ by JE in e.  JE
// is a template argument so that k / id stay in registers (a runtime JE
// puts them on the stack: 96 bytes of local memory per thread, ~50 us of the
// 4096-key window sort).
template <int E, int JE>
__device__ __forceinline__ void inreg_stage(double (&k)[E], int (&id)[E], int stride, int lane0, int kk) {
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if ((e & JE) == 0) {
      const int e2 = e | JE;
      const int i = e * stride + lane0;
      const bool dir = (i & kk) == 0;
      const bool ord = precedes(k[e], id[e], k[e2], id[e2]);
      if (dir != ord) {
        const double tk = k[e]; k[e] = k[e2]; k[e2] = tk;
        const int ti = id[e]; id[e] = id[e2]; id[e2] = ti;
      }
    }
  }
}
template <int E>
__device__ __forceinline__ void inreg_dispatch(double (&k)[E], int (&id)[E], int je, int stride, int lane0,
                                               int kk) {
  if (E > 1 && je == 1) inreg_stage<E, (E > 1 ? 1 : 0)>(k, id, stride, lane0, kk);
  else if (E > 2 && je == 2) inreg_stage<E, (E > 2 ? 2 : 0)>(k, id, stride, lane0, kk);
  else if (E > 4 && je == 4) inreg_stage<E, (E > 4 ? 4 : 0)>(k, id, stride, lane0, kk);
  else if (E > 8 && je == 8) inreg_stage<E, (E > 8 ? 8 : 0)>(k, id, stride, lane0, kk);
}

// Register bitonic sort of N = T * E pairs held E per thread (element e of
// thread t is position e * T + t).  Strides < 32 exchange through warp
// shuffles, strides 32..T/2 through shared memory (sk/si, N entries), strides
// >= T inside the thread; only the shared-memory stages need barriers.
// Requires blockDim.x == T.
template <int T, int E>
__device__ void bitonic_regs(double (&k)[E], int (&id)[E], double* sk, int* si) {
  constexpr int N = T * E;
  const int tid = threadIdx.x;
#pragma unroll 1
  for (int kk = 2; kk <= N; kk <<= 1) {
#pragma unroll 1
    for (int j = kk >> 1; j > 0; j >>= 1) {
      if (j >= T) {
        inreg_dispatch<E>(k, id, j / T, T, tid, kk);
      } else if (j >= 32) {
#pragma unroll
        for (int e = 0; e < E; ++e) { sk[e * T + tid] = k[e]; si[e * T + tid] = id[e]; }
        __syncthreads();
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int i = e * T + tid;
          const double pk = sk[i ^ j];
          const int pi = si[i ^ j];
          const bool first = precedes(k[e], id[e], pk, pi);   // mine precedes the partner
          const bool lo = (i & j) == 0, dir = (i & kk) == 0;
          if ((lo == dir) != first) { k[e] = pk; id[e] = pi; }
        }
        __syncthreads();
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int i = e * T + tid;
          const double pk = __shfl_xor_sync(0xffffffffu, k[e], j);
          const int pi = __shfl_xor_sync(0xffffffffu, id[e], j);
          const bool first = precedes(k[e], id[e], pk, pi);
          const bool lo = (i & j) == 0, dir = (i & kk) == 0;
          if ((lo == dir) != first) { k[e] = pk; id[e] = pi; }
        }
      }
    }
  }
}

// Warp-level bitonic sort of 32 * E pairs held E per lane (element e of lane
// l is run position e * 32 + l): strides < 32 through shuffles, strides >= 32
// inside the lane; no shared memory, no block barriers.
template <int E>
__device__ __forceinline__ void bitonic_warp(double (&k)[E], int (&id)[E], int lane) {
  constexpr int N = 32 * E;
#pragma unroll 1
  for (int kk = 2; kk <= N; kk <<= 1) {
#pragma unroll 1
    for (int j = kk >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        inreg_dispatch<E>(k, id, j >> 5, 32, lane, kk);
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int i = e * 32 + lane;
          const double pk = __shfl_xor_sync(0xffffffffu, k[e], j);
          const int pi = __shfl_xor_sync(0xffffffffu, id[e], j);
          const bool first = precedes(k[e], id[e], pk, pi);
          const bool lo = (i & j) == 0, dir = (i & kk) == 0;
          if ((lo == dir) != first) { k[e] = pk; id[e] = pi; }
        }
      }
    }
  }
}

// Number of elements of the sorted run [lo, hi) that precede (k, i).
__device__ __forceinline__ int count_preceding(const double* key, const int* idx, int lo, int hi,
                                               double k, int i) {
  int a = lo, b = hi;
  while (a < b) {
    const int m = (a + b) >> 1;
    if (precedes(key[m], idx[m], k, i)) a = m + 1;
    else b = m;
  }
  return a - lo;
}

// Merge S sorted runs (run r = [off[r], off[r+1]), off[S] = total) by
// pairwise co-ranking: every element's destination is its rank in its own run
// plus its rank in the partner run (binary search).  log2(S) levels,
// ping-ponging between (k0, i0) and (k1, i1); `off` (S + 1 entries, shared)
// is rewritten.  Returns 0 if the result is in (k0, i0), 1 otherwise.
__device__ int merge_runs(double* k0, int* i0, double* k1, int* i1, unsigned* off, int S,
                          int total) {
  int cur = 0;
  while (S > 1) {
    double* ks = cur ? k1 : k0;
    int* is = cur ? i1 : i0;
    double* kd = cur ? k0 : k1;
    int* id = cur ? i0 : i1;
    for (int q = threadIdx.x; q < total; q += blockDim.x) {
      // run of q: last r with off[r] <= q
      int a = 0, b = S - 1;
      while (a < b) {
        const int m = (a + b + 1) >> 1;
        if ((int)off[m] <= q) a = m;
        else b = m - 1;
      }
      const int r = a;
      const int left = r & ~1;
      const double k = ks[q];
      const int i = is[q];
      int dest;
      if (left + 1 >= S) {
        dest = q;  // odd run out: copied
      } else {
        const int sa = (int)off[left], sb = (int)off[left + 1], eb = (int)off[left + 2];
        if (r == left) dest = sa + (q - sa) + count_preceding(ks, is, sb, eb, k, i);
        else dest = sa + (q - sb) + count_preceding(ks, is, sa, sb, k, i);
      }
      kd[dest] = k;
      id[dest] = i;
    }
    __syncthreads();
    const int S2 = (S + 1) >> 1;
    unsigned o = 0;
    if ((int)threadIdx.x <= S2) o = ((int)threadIdx.x < S2) ? off[2 * threadIdx.x] : (unsigned)total;
    __syncthreads();
    if ((int)threadIdx.x <= S2) off[threadIdx.x] = o;
    __syncthreads();
    S = S2;
    cur ^= 1;
  }
  return cur;
}

// Merge S sorted runs of equal length `run` (S * run = total, S a power of
// two) pairwise, log2(S) levels, by merge path: thread t writes the ITEMS
// consecutive outputs [ITEMS t, ITEMS t + ITEMS) of its pair after ONE
// co-rank binary search on the merge-path diagonal, then a sequential merge
// of ITEMS steps -- instead of a binary search per element (scattered shared
// loads, bank conflicts).  total == ITEMS * blockDim.x.  Same strict order as
// merge_runs (key descending, index ascending); returns 0 if the result is in
// (k0, i0), 1 otherwise.
template <int ITEMS>
__device__ int merge_runs_path(double* k0, int* i0, double* k1, int* i1, int run, int S) {
  int cur = 0;
  for (; S > 1; S >>= 1, run <<= 1) {
    const double* ks = cur ? k1 : k0;
    const int* is = cur ? i1 : i0;
    double* kd = cur ? k0 : k1;
    int* id = cur ? i0 : i1;
    const int q0 = ITEMS * threadIdx.x;
    const int sa = (q0 / (2 * run)) * (2 * run);     // pair start
    const int sb = sa + run;                          // second run
    const int d = q0 - sa;                            // diagonal in the pair
    // co-rank: i elements of A = [sa, sb) and d - i of B = [sb, sb + run)
    int lo = max(0, d - run), hi = min(d, run);
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      const int j = d - mid - 1;
      if (precedes(ks[sa + mid], is[sa + mid], ks[sb + j], is[sb + j])) lo = mid + 1;
      else hi = mid;
    }
    int ia = sa + lo, ib = sb + (d - lo);
    const int ea = sb, eb = sb + run;
    double ka = ia < ea ? ks[ia] : 0.0, kb = ib < eb ? ks[ib] : 0.0;
    int xa = ia < ea ? is[ia] : 0, xb = ib < eb ? is[ib] : 0;
#pragma unroll
    for (int e = 0; e < ITEMS; ++e) {
      const bool take_a = ib >= eb || (ia < ea && precedes(ka, xa, kb, xb));
      if (take_a) {
        kd[q0 + e] = ka;
        id[q0 + e] = xa;
        ++ia;
        if (ia < ea) { ka = ks[ia]; xa = is[ia]; }
      } else {
        kd[q0 + e] = kb;
        id[q0 + e] = xb;
        ++ib;
        if (ib < eb) { kb = ks[ib]; xb = is[ib]; }
      }
    }
    __syncthreads();
    cur ^= 1;
  }
  return cur;
}

}  // namespace l0
