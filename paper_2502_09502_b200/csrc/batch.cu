// Batched node engine kernels: B branch-and-bound node relaxations on one
// shared X (north star item 4).  The per-node arithmetic
// is the single-solve engine's (fista.py:159-212 per node, with that node's
// fixed-one / fixed-zero sets); the two X passes of every iteration become
// tensor-core contractions (tc_gemm.cu) over all nodes at once:
//
//   kb_rhs   : R = grad F(U + c (U - U_prev)) per node (and Z = -grad F(U) on
//              bound checks), split hi/lo for 3xTF32; F* partials
//   kb_plan  : which node rows the transpose contraction needs
//   GEMM_T   : Ct = X^T [R | Z]             (p x 2B, split-K partials)
//   kb_step  : per (slab, node): gradient step and the slab epilogue
//   kb_window: per node (one CTA): bound check, windowed sort + PAVA, g(beta+),
//              beta+ step split hi/lo for the forward contraction
//   GEMM_F   : Cf = X beta+                 (n x B, split-K partials)
//   kb_obj   : per node: u = sum of partials, F(u), objective / restart
//
// Node-major layouts everywhere ([node][coordinate], [node][row]) so that one
// node's vectors are contiguous and the contractions' B operands are K-major.
#include "batch_ops.cuh"
#include "control.cuh"
#include "engine.cuh"
#include "prox.cuh"
#include "slab_epilogue.cuh"

namespace l0 {

struct BatchArgs {
  int64_t n, p, B;
  int64_t pv;       // stride of per-node fp64 p-vectors
  int64_t pp;       // pitch of the fp32 split p-vectors (K of GEMM_F)
  int64_t nn;       // pitch of per-node row vectors (K of GEMM_T)
  int loss;
  const double* y;
  State* st;        // [B]
  Params* prm;      // [B]
  double* beta;     // [B][3][pv] ring per node
  double* gam;      // [B][pv]
  double* key;      // [B][pv]
  double* xs;       // [B][pv]
  double* tail;     // [B][pv]
  double* scratch;  // [B][pv]
  int* perm;        // [B][pv]
  double* gv;       // [B][3 pv + 8]
  uint8_t* mask;    // [B][pv]
  int* fone;        // [B][fone_stride]
  int64_t fone_stride;
  __half* bh;       // [B][pp]  beta+ (or step) 3xFP16 split (GEMM_F B operand), scaled per row
  __half* bl;
  __half* rh;       // [2B][nn] R | Z 3xFP16 split (GEMM_T B operand), scaled per row
  __half* rl;
  float* rinv;      // [2B] 1 / scale of each GEMM_T B row (kb_rhs)
  float* binv;      // [B]  1 / scale of each GEMM_F B row (kb_window / kb_warm_scale)
  double* gbound;   // [B][rblocks] bound on |grad F| over the block's rows for any momentum (kb_obj)
  double xsc;       // power-of-two scale of X in its fp16 splits (|X xsc| < 2^14)
  float* cf;        // [sf][B][nn]
  int sf;
  float* ct;        // [st][2B][pp]
  int sct;
  double* u;        // [3][B][nn]
  double* fpart;    // [B][rblocks][4]
  double* lpart;    // [B][rblocks][2]
  unsigned* cnt;    // [B] (zero between launches)
  int* flags;       // [0] alive, [1] any zeta, [2] GEMM_T rows, [3] GEMM_F rows, [4] done count,
                    // [5] active nodes this iteration
  int* slot;        // [B] row of node b in the contractions this iteration (-1: finished)
  int rblocks;      // row blocks of kb_rhs / kb_obj
  // per-node slab epilogue products (slab_epilogue.cuh), S slabs of kK2Slab columns
  int S;
  double* hval;       // [B][pv]
  double* cand_key;   // [B][pv]
  int* cand_idx;      // [B][pv]
  int* slab_cnt;      // [B][S]
  double* slab_sum;   // [B][S]
  double* slab_max;
  double* slab_below;
  double* slab_hfone;
  double* slab_htop;  // [B][S][kHTop]
  int sf_init;        // split-K partials of the dense MODE_INIT forward contraction
  // Support-compacted forward contraction (sparse_fwd).  The forward operand
  // (the step beta_t - beta_{t-1}, or beta_t on re-syncs) is zero outside the
  // nodes' prox supports: every coordinate past the PAVA pool end is a tail
  // singleton whose output is gamma - mu / rho = 0 (prox.py:104-116 with
  // nu = x).  On C4 a node's step has ~300 nonzeros of 5000 and the union over
  // the batch ~500, so GEMM_F contracts only the X columns of that union:
  // a slot cache of X columns (hi/lo, gathered from X^T once per new column)
  // and the operand rows compacted to the same slots.  Exact zeros contribute
  // nothing to the fp32 accumulation, so this is the dense product's value.
  int sparse_fwd;
  int* umask;         // [pp] nonzero forward operand in some node (kb_window sets, kb_union clears)
  int* slot_of;       // [pp] slot of column j (-1: not cached)
  int* col_of;        // [pp] column cached in slot s (-1: free)
  int* uctl;          // [0] slots in use, [1..2] slots to gather [s0, s1), [3] GEMM_F K (slots
                      // rounded up to 32), [4] rebuilds, [5] columns gathered (statistics)
  const __half* xth;  // X^T hi/lo (p x nn): the gather source (coalesced rows)
  const __half* xtl;
  __half* xuh;        // [n][pp] cached X columns by slot (GEMM_F A operand)
  __half* xul;
  __half* bsh;        // [B][pp] forward operand by slot (GEMM_F B operand)
  __half* bsl;
  int* fx_n;          // [B] fixed-one columns of node b outside the cache with a nonzero step
  int* fx_j;          // [B][kFoneDirect] their ids
  double* fx_v;       // [B][kFoneDirect] and steps (kb_gather -> kb_obj)
};

constexpr int kRowThreads = 256;
constexpr int kRowsPerBlock = 2048;
// u_{t} = u_{t-1} + X (beta_t - beta_{t-1}) between re-syncs u_t = X beta_t:
// the contraction's fp32-class error then scales with the step, not with u,
// so the restart test F(u_t) + ... >= previous (fista.py:168) sees accurate
// differences; every kResync iterations u is recomputed from beta_t.
constexpr int64_t kResync = 40;
// sparse_fwd: nodes with at most this many fixed-one coordinates get their
// step on those columns added by kb_obj (fp64) unless the column is cached
constexpr int kFoneDirect = 32;
__device__ __forceinline__ bool resync_at(int64_t t) { return t % kResync == 0; }

__device__ __forceinline__ int64_t gvs(const BatchArgs& g) { return 3 * g.pv + 8; }

// warm starts: beta_0 of every node into ring slots 0 and 2 (t = 0, t = -1)
// and its TF32 split into the forward contraction's rows
__global__ void kb_warm(BatchArgs g, const double* warm) {
  const int64_t b = blockIdx.y;
  const double sc = 1.0 / (double)g.binv[b];   // power of two (kb_warm_scale)
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < g.pp; j += (int64_t)gridDim.x * blockDim.x) {
    const double w = j < g.p ? warm[b * g.p + j] : 0.0;
    if (j < g.pv) {
      g.beta[(b * 3 + 0) * g.pv + j] = w;
      g.beta[(b * 3 + 2) * g.pv + j] = w;
    }
    __half h, l;
    f16_split(w * sc, h, l);
    g.bh[b * g.pp + j] = h;
    g.bl[b * g.pp + j] = l;
  }
}

// per-node fp16 scale of the warm starts (rows b of the MODE_INIT forward operand)
__global__ void kb_warm_scale(BatchArgs g, const double* warm) {
  __shared__ double red[32];
  const int64_t b = blockIdx.x;
  double m = 0.0;
  for (int64_t j = threadIdx.x; j < g.p; j += blockDim.x) m = fmax(m, fabs(warm[b * g.p + j]));
  m = block_max(m, red);
  if (threadIdx.x == 0) g.binv[b] = ldexpf(1.f, -f16_exp(m));
}

// per-node classes from a compact list (node b: entries [off[b], off[b+1]),
// its fixed-one indices first, ascending): the mask rows were memset to FREE
__global__ void kb_fill_nodes(BatchArgs g, const int64_t* off, const int* idx, const uint8_t* cls) {
  const int64_t b = blockIdx.x;
  const int64_t e0 = off[b], e1 = off[b + 1];
  for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    const int j = idx[e];
    g.mask[b * g.pv + j] = cls[e];
    if (cls[e] == FIXED_ONE) g.fone[b * g.fone_stride + (e - e0)] = j;
  }
}

// g(beta_0) of each node's warm start (perspective.py:76-132, the per-node
// envelope of the initial composite objective, fista.py:143) -- one CTA per
// node: fixed-zero / fixed-one / box / budget feasibility, then the top
// k_g free magnitudes (radix selection + rank sort) into the majorization
// greedy (envelope_from_top), as the single engine's envelope_of.
__global__ void __launch_bounds__(512) kb_g0(BatchArgs g, const double* __restrict__ warm, double* __restrict__ g0) {
  __shared__ SelectSmem sel;
  __shared__ double red[32];
  __shared__ double cand[kCandCap], cand2[kCandCap];
  __shared__ int ncand;
  __shared__ double s_gfree;
  const int64_t b = blockIdx.x, p = g.p;
  const Params* P = g.prm + b;
  const double* w = warm + b * p;
  const uint8_t* mk = g.mask + b * g.pv;
  double* mag = g.scratch + b * g.pv;   // |beta| on free coordinates, -1 elsewhere
  const double M = P->M, Mtol = dmul(M, dadd(1.0, kFeasRtol));
  double total = 0.0, amax = 0.0, s2 = 0.0;
  int bad = 0;
  for (int64_t j = threadIdx.x; j < p; j += blockDim.x) {
    const double x = w[j];
    const int c = mk[j];
    if (c == FREE) {
      const double a = fabs(x);
      mag[j] = a;
      total += a;
      amax = fmax(amax, a);
    } else {
      mag[j] = -1.0;
      if (c == FIXED_ZERO && fabs(x) > kZeroAtol) bad = 1;
      if (c == FIXED_ONE) {
        if (fabs(x) > Mtol) bad = 1;
        s2 = fma(x, x, s2);
      }
    }
  }
  total = block_sum(total, red);
  amax = block_max(amax, red);
  s2 = block_sum(s2, red);
  bad = __syncthreads_or(bad);
  const int64_t nf = P->n_free, kg = P->k_g;
  int path = 0;
  if (bad) path = 3;
  else if (nf == 0 || kg == 0) path = 2;
  else if (amax > Mtol || total > dmul(dmul((double)kg, M), dadd(1.0, kFeasRtol))) path = 3;
  double gfree = 0.0;
  if (path == 0) {
    const int64_t kk = kg < nf ? kg : nf;
    if (kk > kCandCap) {   // beyond the on-chip top-k: flag (the host checks n_free / k)
      path = 3;
    } else {
      double tau;
      int64_t cgt;
      block_kth_largest(mag, p, kk, sel, &tau, &cgt);
      if (threadIdx.x == 0) ncand = 0;
      __syncthreads();
      for (int64_t j = threadIdx.x; j < p; j += blockDim.x)
        if (mag[j] > tau) cand[atomicAdd(&ncand, 1)] = mag[j];
      __syncthreads();
      for (int64_t i = cgt + threadIdx.x; i < kk; i += blockDim.x) cand[i] = tau;
      __syncthreads();
      block_rank_sort_desc(cand, cand2, (int)kk);
      __syncthreads();
      if (threadIdx.x < 32) {
        const double gv = envelope_from_top(cand2, kk, total);
        if (threadIdx.x == 0) s_gfree = gv;
      }
      __syncthreads();
      gfree = s_gfree;
    }
  }
  if (threadIdx.x == 0) {
    double v;
    if (path == 3) v = CUDART_INF;
    else if (P->node_mode) v = dadd(dadd(0.0, dmul(0.5, s2)), gfree);
    else v = gfree;
    g0[b] = v;
  }
}

__global__ void kb_state_init(BatchArgs g, const double* g0) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.B) return;
  State* st = g.st + b;
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
  st->g_next = g0 ? g0[b] : 0.0;          // g(beta_0) for the initial objective (fista.py:143)
  st->best_dual = g.prm[b].parent_bound;
  st->gap = CUDART_NAN;
  st->last_dual = CUDART_NAN;
  st->loss_cur = 0.0;
  st->theta = 0.0;
  st->slow_prox = 0;
  st->win_ext = 0;
}

// Contraction rows for this iteration: the unfinished nodes, compacted in
// node order (finished nodes drop out of both contractions)
__global__ void __launch_bounds__(1024) kb_compact(BatchArgs g) {
  __shared__ int warp_tot[32];
  __shared__ int base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t b0 = 0; b0 < g.B; b0 += 1024) {
    const int64_t b = b0 + threadIdx.x;
    const int act = (b < g.B && !g.st[b].done) ? 1 : 0;
    const unsigned m = __ballot_sync(0xffffffffu, act);
    const int before = __popc(m & ((1u << lane) - 1u));
    if (lane == 0) warp_tot[warp] = __popc(m);
    __syncthreads();
    int off = base;
    for (int w = 0; w < warp; ++w) off += warp_tot[w];
    if (b < g.B) g.slot[b] = act ? off + before : -1;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w = 0; w < 32; ++w) tot += warp_tot[w];
      base += tot;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) g.flags[5] = base;
}

// R / Z rows of node blockIdx.y for rows [blockIdx.x * kRowsPerBlock, ...)
__global__ void __launch_bounds__(kRowThreads, 4) kb_rhs(BatchArgs g) {
  __shared__ double red[32];
  const int64_t b = blockIdx.y;
  State* st = g.st + b;
  if (st->done) return;
  const bool wz = st->dual_pending != 0;
  const bool wg = st->dual_only == 0;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    if (wg || wz) atomicOr(g.flags + 0, 1);
    if (wz) atomicOr(g.flags + 1, 1);
  }
  const int64_t t = st->t + 1;
  const double c = momentum(st->phi);
  const int64_t n = g.n, nn = g.nn, B = g.B;
  const double* ucur = g.u + (ring(t - 1) * B + b) * nn;
  const double* uprev = g.u + (ring(t - 2) * B + b) * nn;
  // compacted contraction rows: R at slot, Z at (active count) + slot
  const int64_t pos = g.slot[b], nact = g.flags[5];
  __half* rh = g.rh + pos * nn;
  __half* rl = g.rl + pos * nn;
  __half* zh = g.rh + (nact + pos) * nn;
  __half* zl = g.rl + (nact + pos) * nn;
  // fp16 scale of the node's rows: kb_obj bounded |grad F(u_t + c (u_t - u_{t-1}))|
  // for every c in [0, 1] (and c = 0 is zeta), so |R sc|, |Z sc| < 2^14
  double gb = 0.0;
  for (int r = 0; r < g.rblocks; ++r) gb = fmax(gb, g.gbound[b * g.rblocks + r]);
  const int sx = f16_exp(gb);
  const double sc = ldexp(1.0, sx);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    g.rinv[pos] = ldexpf(1.f, -sx);
    g.rinv[nact + pos] = ldexpf(1.f, -sx);
  }
  double facc[3] = {0.0, 0.0, 0.0};
  int bad = 0;
  const int r0 = blockIdx.x * kRowsPerBlock;
  const int r1 = (int)min(n, (int64_t)r0 + kRowsPerBlock);
  // two rows per thread per step (16-byte loads; nn and r0 are even)
  auto row = [&](double uc, double up, double yi, double& gr, double& zv) {
    // X gamma = u_t + c (u_t - u_{t-1})   (linearity; fista.py:161-162)
    const double ug = dadd(uc, dmul(c, dsub(uc, up)));
    if (!isfinite(ug)) bad = 1;
    gr = loss_grad(g.loss, ug, yi);
    zv = -loss_grad(g.loss, uc, yi);              // zeta = -grad F(u) (fista.py:152)
  };
#pragma unroll 2
  for (int i = r0 + 2 * (int)threadIdx.x; i < r1; i += 2 * kRowThreads) {
    const bool two = i + 1 < r1;
    double uc[2], up[2], yi[2];
    if (two) {
      const double2 a2 = *reinterpret_cast<const double2*>(ucur + i);
      const double2 b2 = *reinterpret_cast<const double2*>(uprev + i);
      const double2 y2 = *reinterpret_cast<const double2*>(g.y + i);
      uc[0] = a2.x; uc[1] = a2.y; up[0] = b2.x; up[1] = b2.y; yi[0] = y2.x; yi[1] = y2.y;
    } else {
      uc[0] = ucur[i]; up[0] = uprev[i]; yi[0] = g.y[i];
      uc[1] = 0.0; up[1] = 0.0; yi[1] = 0.0;
    }
    __half gh[2], gl[2], zh2[2], zl2[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 1 && !two) break;
      double gr = 0.0, zv = 0.0;
      row(uc[h], up[h], yi[h], gr, zv);
      f16_split(gr * sc, gh[h], gl[h]);
      if (wz) {
        f16_split(zv * sc, zh2[h], zl2[h]);
        conj_accumulate(g.loss, zv, yi[h], facc);
      }
    }
    if (two) {
      if (wg) {
        *reinterpret_cast<__half2*>(rh + i) = __halves2half2(gh[0], gh[1]);
        *reinterpret_cast<__half2*>(rl + i) = __halves2half2(gl[0], gl[1]);
      }
      if (wz) {
        *reinterpret_cast<__half2*>(zh + i) = __halves2half2(zh2[0], zh2[1]);
        *reinterpret_cast<__half2*>(zl + i) = __halves2half2(zl2[0], zl2[1]);
      }
    } else {
      if (wg) { rh[i] = gh[0]; rl[i] = gl[0]; }
      if (wz) { zh[i] = zh2[0]; zl[i] = zl2[0]; }
    }
  }
  if (!wg) bad = 0;
  if (wz) {
    const double f0 = block_sum(facc[0], red);
    const double f1 = block_sum(facc[1], red);
    const double f2 = block_sum(facc[2], red);
    if (threadIdx.x == 0) {
      double* fp = g.fpart + (b * g.rblocks + blockIdx.x) * 4;
      fp[0] = f0;
      fp[1] = f1;
      fp[2] = f2;
    }
  }
  if (wg && bad) {
    // loss_gradient on non-finite predictions: model.py:215 -> InvalidInputError
    atomicExch(&st->err, (int)ST_INVALID);
    st->err_iter = t;
    st->done = 1;
  }
}

__global__ void kb_plan(BatchArgs g) {
  const int alive = g.flags[0], anyz = g.flags[1], nact = g.flags[5];
  g.flags[2] = alive ? (anyz ? 2 * nact : nact) : 0;
  g.flags[3] = alive ? nact : 0;
  g.flags[0] = 0;
  g.flags[1] = 0;
}

__device__ __forceinline__ EngineArgs node_view(const BatchArgs& g, int64_t b) {
  EngineArgs a{};
  a.n = g.n;
  a.p = g.p;
  a.pv = g.pv;
  a.loss = g.loss;
  a.st = g.st + b;
  a.prm = g.prm + b;
  a.beta = g.beta + b * 3 * g.pv;
  a.gam = g.gam + b * g.pv;
  a.key = g.key + b * g.pv;
  a.xs = g.xs + b * g.pv;
  a.tail = g.tail + b * g.pv;
  a.scratch = g.scratch + b * g.pv;
  a.perm = g.perm + b * g.pv;
  a.gv = g.gv + b * gvs(g);
  a.mask = g.mask + b * g.pv;
  a.fone = g.fone + b * g.fone_stride;
  a.k2_slabs = g.S;
  a.hval = g.hval + b * g.pv;
  a.cand_key = g.cand_key + b * g.pv;
  a.cand_idx = g.cand_idx + b * g.pv;
  a.slab_cnt = g.slab_cnt + b * g.S;
  a.slab_sum = g.slab_sum + b * g.S;
  a.slab_max = g.slab_max + b * g.S;
  a.slab_below = g.slab_below + b * g.S;
  a.slab_hfone = g.slab_hfone + b * g.S;
  a.slab_htop = g.slab_htop + b * g.S * kHTop;
  return a;
}

// (slab, node): reduce the transpose contraction's split-K partials for 256
// columns of one node, then the single engine's slab epilogue (gradient step,
// keys, speculative outputs, window candidates, Huber values)
__global__ void __launch_bounds__(kK2Slab) kb_step(BatchArgs g) {
  __shared__ EpiSmem sm;
  const int64_t b = blockIdx.y;
  const int slab = blockIdx.x;
  const EngineArgs a = node_view(g, b);
  const State* st = a.st;
  if (st->done) return;
  const bool wz = st->dual_pending != 0;
  const bool wg = st->dual_only == 0;
  if (!wg && !wz) return;
  const int64_t t = st->t + 1;
  const double c = momentum(st->phi);
  const int64_t B = g.B, pv = g.pv;
  const int64_t pos = g.slot[b], nact = g.flags[5];   // compacted contraction rows
  const int64_t j = (int64_t)slab * kK2Slab + threadIdx.x;
  double gsum = 0.0, v = 0.0;
  if (j < g.p) {
    const float* ct = g.ct;
    const int64_t split = 2 * B * g.pp;
    if (wg) {
#pragma unroll 4
      for (int s = 0; s < g.sct; ++s) gsum += (double)__ldcg(ct + s * split + pos * g.pp + j);
    }
    if (wz) {
#pragma unroll 4
      for (int s = 0; s < g.sct; ++s) v += (double)__ldcg(ct + s * split + (nact + pos) * g.pp + j);
    }
  }
  if (wz && slab == 0 && threadIdx.x == 0) {
    // F*(-zeta) accumulators over the row blocks (fixed order)
    double f0 = 0.0, f1 = 0.0, f2 = 0.0;
    for (int r = 0; r < g.rblocks; ++r) {
      const double* fp = g.fpart + (b * g.rblocks + r) * 4;
      f0 += fp[0];
      f1 += fp[1];
      f2 += fp[2];
    }
    a.gv[2 * pv + 0] = f0;
    a.gv[2 * pv + 1] = f1;
    a.gv[2 * pv + 2] = f2;
  }
  slab_epilogue(a, slab, t, c, wg, wz, gsum, v, sm);
}

// one CTA per node: bound check, windowed sort + PAVA, g(beta+) (the single
// engine's K3), then beta+ (or its step) split hi/lo for GEMM_F
__global__ void __launch_bounds__(kWinThreads, 1) kb_window(BatchArgs g) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ProxSmem& ps = *reinterpret_cast<ProxSmem*>(smem_raw);
  WinSmem& sm = *reinterpret_cast<WinSmem*>(smem_raw + ((sizeof(ProxSmem) + 255) & ~size_t(255)));
  const int64_t b = blockIdx.x;
  const EngineArgs a = node_view(g, b);
  if (a.st->done) return;
  const int64_t t = a.st->t + 1;
  if (!prox_window_body(a, ps, sm)) return;
  __syncthreads();
  // beta+ (re-sync) or beta+ - beta_t -> hi/lo operand rows of the forward contraction
  const bool full = resync_at(t);
  const double* out = a.beta + ring(t) * g.pv;
  const double* bprev = a.beta + ring(t - 1) * g.pv;
  const int64_t pos = g.slot[b];                      // compacted contraction row
  const bool direct_fone = a.prm->node_mode && a.prm->n_fone <= kFoneDirect;
  // exact per-row fp16 scale from the largest |operand| of this node
  double am = 0.0;
  for (int64_t j = threadIdx.x; j < g.p; j += kWinThreads)
    am = fmax(am, fabs(full ? out[j] : dsub(out[j], bprev[j])));
  am = block_max(am, ps.red);
  const int sx = f16_exp(am);
  const double sc = ldexp(1.0, sx);
  if (threadIdx.x == 0) g.binv[pos] = ldexpf(1.f, -sx);
  for (int64_t j = threadIdx.x; j < g.pp; j += kWinThreads) {
    __half h = __ushort_as_half(0), l = __ushort_as_half(0);
    if (j < g.p) f16_split((full ? out[j] : dsub(out[j], bprev[j])) * sc, h, l);
    g.bh[pos * g.pp + j] = h;
    g.bl[pos * g.pp + j] = l;
    // a node's few fixed-one columns stay out of the shared column cache (they
    // would widen every node's contraction for one node's sake); kb_obj adds
    // their step in fp64 instead
    if (g.sparse_fwd && (f16_nonzero(h) || f16_nonzero(l)) && !(direct_fone && a.mask[j] == FIXED_ONE))
      g.umask[j] = 1;
  }
}

// rank of this thread's flag among the block's set flags (thread order) and
// the block total; all threads call it
__device__ __forceinline__ int block_flag_rank(int f, int* wtot, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned m = __ballot_sync(0xffffffffu, f);
  if (lane == 0) wtot[warp] = __popc(m);
  __syncthreads();
  int off = 0, tot = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
    const int c = wtot[w];
    if (w < warp) off += c;
    tot += c;
  }
  __syncthreads();
  *total = tot;
  return off + __popc(m & ((1u << lane) - 1u));
}

// Union of the forward operand's supports over the nodes -> slots of the X
// column cache.  New columns are appended (ascending index) after the slots
// in use; when the stale slots (columns no longer in the union, operand 0
// there) would exceed a quarter of the union, the cache is rebuilt compactly.
// kb_gather then fetches the X columns of the slots [s0, s1) only: in steady
// state the union is unchanged and nothing is gathered.
__global__ void __launch_bounds__(1024) kb_union(BatchArgs g) {
  __shared__ int wtot[32];
  __shared__ int red[2][32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t p = g.p;
  int cu = 0, cn = 0;
  for (int64_t j = tid; j < p; j += blockDim.x) {
    const int m = g.umask[j];
    cu += m;
    cn += (m && g.slot_of[j] < 0) ? 1 : 0;
  }
  cu = __reduce_add_sync(0xffffffffu, cu);
  cn = __reduce_add_sync(0xffffffffu, cn);
  if (lane == 0) { red[0][warp] = cu; red[1][warp] = cn; }
  __syncthreads();
  cu = 0;
  cn = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { cu += red[0][w]; cn += red[1][w]; }
  const int ext0 = g.uctl[0];
  const bool rebuild = ext0 + cn > cu + cu / 4 + 64 || ext0 + cn > (int)g.pp;
  if (rebuild) {
    for (int s = tid; s < ext0; s += blockDim.x) {
      const int j = g.col_of[s];
      if (j >= 0) g.slot_of[j] = -1;
      g.col_of[s] = -1;
    }
    __syncthreads();
  }
  int base = rebuild ? 0 : ext0;
  for (int64_t j0 = 0; j0 < p; j0 += blockDim.x) {
    const int64_t j = j0 + tid;
    const int m = j < p ? g.umask[j] : 0;
    const int f = m && (rebuild || g.slot_of[j] < 0);
    int tot;
    const int r = block_flag_rank(f, wtot, &tot);
    if (f) {
      g.slot_of[j] = base + r;
      g.col_of[base + r] = (int)j;
    }
    if (m) g.umask[j] = 0;
    base += tot;
  }
  if (tid == 0) {
    const int s0 = rebuild ? 0 : ext0;
    g.uctl[0] = base;
    g.uctl[1] = s0;
    g.uctl[2] = base;
    g.uctl[3] = min((base + 63) / 64 * 64, (int)g.pp);   // whole fp16 K blocks
    if (rebuild) g.uctl[4] += 1;
    g.uctl[5] += base - s0;
  }
}

// (1) X columns of the new slots [s0, s1) from X^T (32 slots x 64 rows per
// item through shared memory: coalesced reads along rows of X^T, 128-byte
// row segments written); (2) the forward operand rows by slot (zero in free
// slots and in the padding up to the K of GEMM_F).  Persistent grid.
constexpr int kGatherRows = 64;
__global__ void __launch_bounds__(256) kb_gather(BatchArgs g) {
  __shared__ __half th[32][kGatherRows + 2], tl[32][kGatherRows + 2];
  const int s0 = g.uctl[1], s1 = g.uctl[2], kpad = g.uctl[3];
  const int64_t n = g.n, pp = g.pp, nn = g.nn;
  const int rtiles = (int)((n + kGatherRows - 1) / kGatherRows);
  const int items = rtiles * ((s1 - s0 + 31) / 32);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    const int sb = s0 + (it / rtiles) * 32;
    const int64_t r0 = (int64_t)(it % rtiles) * kGatherRows;
    for (int i = ty; i < 32; i += 8) {
      const int sl = sb + i;
      const int j = sl < s1 ? g.col_of[sl] : -1;
      for (int c = tx; c < kGatherRows; c += 32) {
        const int64_t r = r0 + c;
        __half h = __ushort_as_half(0), l = __ushort_as_half(0);
        if (j >= 0 && r < n) {
          h = g.xth[(int64_t)j * nn + r];
          l = g.xtl[(int64_t)j * nn + r];
        }
        th[i][c] = h;
        tl[i][c] = l;
      }
    }
    __syncthreads();
    for (int c = ty; c < kGatherRows; c += 8) {
      const int64_t r = r0 + c;
      const int sl = sb + tx;
      if (r < n && sl < s1) {
        g.xuh[r * pp + sl] = th[tx][c];
        g.xul[r * pp + sl] = tl[tx][c];
      }
    }
    __syncthreads();
  }
  // per node: its fixed-one columns that stay outside the cache, with their
  // step (fp64), for kb_obj -- one warp per node
  {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = gw; b < g.B; b += nw) {
      const Params* P = g.prm + b;
      const State* st = g.st + b;
      if (!P->node_mode || P->n_fone > kFoneDirect || st->done || st->dual_only) continue;
      const int64_t t = st->t + 1;
      const bool full = resync_at(t);
      int j = -1;
      double v = 0.0;
      if (lane < P->n_fone) {
        j = g.fone[b * g.fone_stride + lane];
        const double bt = g.beta[(b * 3 + ring(t)) * g.pv + j];
        v = full ? bt : dsub(bt, g.beta[(b * 3 + ring(t - 1)) * g.pv + j]);
        if (g.slot_of[j] >= 0 || v == 0.0) j = -1;
      }
      const unsigned m = __ballot_sync(0xffffffffu, j >= 0);
      if (j >= 0) {
        const int r = __popc(m & ((1u << lane) - 1u));
        g.fx_j[b * kFoneDirect + r] = j;
        g.fx_v[b * kFoneDirect + r] = v;
      }
      if (lane == 0) g.fx_n[b] = __popc(m);
    }
  }
  const int64_t rows = g.flags[3];
  const int64_t tot = rows * kpad;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / kpad;
    const int sl = (int)(e - r * kpad);
    const int j = g.col_of[sl];
    __half h = __ushort_as_half(0), l = __ushort_as_half(0);
    if (j >= 0) {
      h = g.bh[r * pp + j];
      l = g.bl[r * pp + j];
    }
    g.bsh[r * pp + sl] = h;
    g.bsl[r * pp + sl] = l;
  }
}

// u = X beta+ (sum of split-K partials, fixed order), F(u), objective
__global__ void __launch_bounds__(kRowThreads, 3) kb_obj(BatchArgs g, int mode) {
  __shared__ double red[32];
  __shared__ int s_last;
  const int64_t b = blockIdx.y;
  State* st = g.st + b;
  if (mode == MODE_ITER && (st->done || st->dual_only)) return;
  if (mode == MODE_INIT && st->done) return;
  const int64_t t = mode == MODE_ITER ? st->t + 1 : 0;
  const int64_t n = g.n, nn = g.nn, B = g.B;
  const int64_t r0 = (int64_t)blockIdx.x * kRowsPerBlock;
  const int64_t r1 = min(n, r0 + kRowsPerBlock);
  double lsum = 0.0, gmax = 0.0;
  int bad = 0;
  const bool delta = mode == MODE_ITER && !resync_at(t);
  const double* uprev = g.u + (ring(t - 1) * B + b) * nn;
  double* uo = g.u + ((mode == MODE_ITER ? ring(t) : 0) * B + b) * nn;
  double* uo2 = g.u + (2 * B + b) * nn;           // MODE_INIT: u_{-1} = u_0
  // compacted contraction row (MODE_INIT: every node, slot = node)
  const float* cfb = g.cf + (mode == MODE_ITER ? (int64_t)g.slot[b] : b) * nn;
  const int64_t cstride = B * nn;
  // fixed-one columns outside the column cache (sparse_fwd, see kb_window):
  // u += X[:, j] * step_j in fp64, X[:, j] = hi + lo of X^T's row j (exact);
  // the (j, step) list was made by kb_gather
  __shared__ int fx_j[kFoneDirect];
  __shared__ double fx_v[kFoneDirect];
  const Params* Pb = g.prm + b;
  const bool fx = mode == MODE_ITER && g.sparse_fwd && Pb->node_mode && Pb->n_fone <= kFoneDirect;
  int fx_n = 0;
  if (fx) {
    fx_n = g.fx_n[b];
    if (threadIdx.x < fx_n) {
      fx_j[threadIdx.x] = g.fx_j[b * kFoneDirect + threadIdx.x];
      fx_v[threadIdx.x] = g.fx_v[b * kFoneDirect + threadIdx.x];
    }
    __syncthreads();
  }
  const int nfx = fx_n;
  const int sf = mode == MODE_ITER ? g.sf : g.sf_init;
  const int i0 = (int)r0, i1 = (int)r1;
  // two rows per thread per step (16-byte loads; nn and r0 are even); two
  // steps unrolled so their loads are in flight together
#pragma unroll 2
  for (int i = i0 + 2 * (int)threadIdx.x; i < i1; i += 2 * kRowThreads) {
    const bool two = i + 1 < i1;
    double u[2] = {0.0, 0.0}, yv[2], upv[2] = {0.0, 0.0};
    if (two) {
      for (int s = 0; s < sf; ++s) {
        const float2 c2 = *reinterpret_cast<const float2*>(cfb + s * cstride + i);
        u[0] += (double)c2.x;
        u[1] += (double)c2.y;
      }
      const double2 y2 = *reinterpret_cast<const double2*>(g.y + i);
      yv[0] = y2.x; yv[1] = y2.y;
      if (mode == MODE_ITER) {   // the step base, and u_{t-1} of the gradient bound
        const double2 p2 = *reinterpret_cast<const double2*>(uprev + i);
        upv[0] = p2.x; upv[1] = p2.y;
      }
    } else {
      for (int s = 0; s < sf; ++s) u[0] += (double)cfb[s * cstride + i];
      yv[0] = g.y[i];
      yv[1] = 0.0;
      if (mode == MODE_ITER) upv[0] = uprev[i];
    }
    for (int e = 0; e < nfx; ++e) {
      const int64_t o = (int64_t)fx_j[e] * nn + i;   // even: 4-byte aligned pairs
      const double v = fx_v[e] / g.xsc;
      const float2 xh = __half22float2(*reinterpret_cast<const __half2*>(g.xth + o));
      const float2 xl = __half22float2(*reinterpret_cast<const __half2*>(g.xtl + o));
      u[0] = fma((double)xh.x + (double)xl.x, v, u[0]);
      if (two) u[1] = fma((double)xh.y + (double)xl.y, v, u[1]);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 1 && !two) break;
      if (delta) u[h] = dadd(upv[h], u[h]);
      if (!isfinite(u[h])) bad = 1;
      lsum += loss_term(g.loss, u[h], yv[h]);
      // |grad F(u + c (u - u_prev))| for every c in [0, 1] (the next kb_rhs's fp16 scale)
      const double du = mode == MODE_ITER ? fabs(u[h] - upv[h]) : 0.0;
      const double ay = fabs(yv[h]);
      double gbd;
      if (g.loss == SQUARED_ERROR) gbd = 2.0 * (fabs(u[h] - yv[h]) + du);
      else if (g.loss == LOGISTIC) gbd = ay;
      else gbd = 2.0 * ay * (1.0 + ay * (fabs(u[h]) + du));
      gmax = fmax(gmax, gbd * (1.0 + 1e-12));
    }
    if (two) {
      *reinterpret_cast<double2*>(uo + i) = make_double2(u[0], u[1]);
      if (mode != MODE_ITER) *reinterpret_cast<double2*>(uo2 + i) = make_double2(u[0], u[1]);
    } else {
      uo[i] = u[0];
      if (mode != MODE_ITER) uo2[i] = u[0];
    }
  }
  const double csum = block_sum(lsum, red);
  gmax = block_max(gmax, red);
  const int anybad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    g.gbound[b * g.rblocks + blockIdx.x] = gmax;
    double* lp = g.lpart + (b * g.rblocks + blockIdx.x) * 2;
    lp[0] = csum;
    lp[1] = anybad ? 1.0 : 0.0;
    __threadfence();
    s_last = atomicAdd(g.cnt + b, 1u) == (unsigned)(gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  __threadfence();
  g.cnt[b] = 0u;
  double tot = 0.0, nb = 0.0;
  for (int r = 0; r < (int)gridDim.x; ++r) {
    const double* lp = g.lpart + (b * g.rblocks + r) * 2;
    tot += __ldcg(lp);
    nb += __ldcg(lp + 1);
  }
  const Params* P = g.prm + b;
  if (nb > 0.0) {  // loss_value on non-finite predictions (model.py:152-161)
    st->err = ST_INVALID;
    st->err_iter = t;
    if (mode == MODE_ITER) st->t = t;
    st->done = 1;
  } else if (mode == MODE_ITER) {
    objective_update(st, P, tot);
  } else {
    st->loss_cur = tot;
    st->obj = dadd(tot, dmul(P->two_l2, st->g_next));  // fista.py:143
  }
}

// nodes finished -> flags[4]
__global__ void kb_count(BatchArgs g) {
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  int local = 0;
  for (int64_t b = threadIdx.x; b < g.B; b += blockDim.x) local += g.st[b].done ? 1 : 0;
  atomicAdd(&cnt, local);
  __syncthreads();
  if (threadIdx.x == 0) g.flags[4] = cnt;
}

__global__ void kb_request_stop(BatchArgs g, int term) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.B) return;
  State* st = g.st + b;
  const Params* P = g.prm + b;
  if (st->done) return;
  if (st->check_pending) {
    if (st->stop_term < 0) st->stop_term = term;
    st->dual_only = 1;
  } else {
    request_stop(st, P, term);
  }
}

inline int64_t kb_prox_capacity() { return (int64_t)kWinThreads * kK2Slab; }

cudaError_t kb_sparse_fwd_prep(const BatchArgs& g, int grid, cudaStream_t s) {
  kb_union<<<1, 1024, 0, s>>>(g);
  kb_gather<<<grid, 256, 0, s>>>(g);
  return cudaGetLastError();
}

cudaError_t kb_prox_launch(const BatchArgs& g, cudaStream_t s) {
  kb_step<<<dim3((unsigned)g.S, (unsigned)g.B), kK2Slab, 0, s>>>(g);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const size_t smem = prox_window_smem();
  e = cudaFuncSetAttribute(kb_window, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kb_window<<<(unsigned)g.B, kWinThreads, smem, s>>>(g);
  return cudaGetLastError();
}

}  // namespace l0
