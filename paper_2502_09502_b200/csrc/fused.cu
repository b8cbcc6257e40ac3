// KF: one physical pass over X per FISTA iteration.
//
// Iteration t needs u_t = X beta_t (objective, restart test) and the next
// gradient X^T grad F(u_t + c_{t+1} (u_t - u_{t-1})), whose momentum c_{t+1}
// depends on the restart decision, i.e. on ALL rows of u_t.  KF computes both
// candidates -- c = 1/4 (restart, phi -> 1) and c = (phi+1)/(phi+4) (no
// restart) -- plus X^T zeta_t for the bound check, from ONE read of each X
// tile (kf_fused_s below):
//
//   * a thread-block cluster of fz_cs CTAs spans a full row block; CTA c owns
//     columns [c W, (c+1) W);
//   * row tiles (fz_rows rows x W columns) stream HBM -> shared memory with
//     cp.async.bulk into a ring of fz_stages buffers and stay there until
//     their rows are accumulated into X^T r;
//   * per-row partial dots are pushed to EVERY CTA of the cluster with
//     st.async into a ring of partial slots, each completing a
//     transaction-count mbarrier in the receiving CTA -- no cluster barrier
//     on the per-tile path;
//   * when tile k's partials are complete, u for its rows is the fixed-order
//     sum over the cluster (identical in every CTA), and the tile in shared
//     memory accumulates X^T [r_R | r_N | zeta] in registers;
//   * the last CTA of the grid reduces the per-cluster loss (fixed order) and
//     runs the objective / restart logic (control.cuh).
//
// KR then reduces the per-cluster partials over clusters (fixed order), picks
// the candidate matching the restart decision and runs the slab epilogue
// (gradient step, keys, window candidates, Huber values).

#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "control.cuh"
#include "engine.cuh"
#include "slab_epilogue.cuh"

namespace l0 {


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
// The waits carry a suspend-time hint: a warp whose phase is not complete
// sleeps until the phase completes (or the hint expires) instead of retrying
// every ~50 cycles -- ncu on C5 counted ~150M retries per launch (accumulate
// warps on rfull, producer on empty, gather on the partial slots), issue slots
// taken from the warps doing the work on the same SM sub-partition.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase, uint32_t ns) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(saddr(bar)), "r"(phase), "r"(ns)
        : "memory");
  }
}
// wait for a partial slot filled by st.async from the cluster peers: the
// complete_tx of a remote st.async is a release at cluster scope, so the wait
// acquires at cluster scope (one L1 invalidation per completed wait; measured
// free next to the CTA-scope form on C2).
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t phase, uint32_t ns) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(saddr(bar)), "r"(phase), "r"(ns)
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
__device__ __forceinline__ uint32_t map_rank(const void* local, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(saddr(local)), "r"(rank));
  return ra;
}
// v -> [remote] in CTA `rank`, completing 8 bytes on that CTA's mbarrier
__device__ __forceinline__ void st_async_f64(const double* local_dst, const uint64_t* local_bar,
                                             uint32_t rank, double v) {
  const uint32_t ra = map_rank(local_dst, rank);
  const uint32_t rb = map_rank(local_bar, rank);
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(ra),
               "d"(v), "r"(rb)
               : "memory");
}

template <typename TX> struct FzVec;
template <> struct FzVec<double> {
  using T = double2;
  static constexpr int N = 2;
  __device__ __forceinline__ static void widen(const T& v, double* o) { o[0] = v.x; o[1] = v.y; }
  __device__ __forceinline__ static void widen_s(const T& v, double* o) { widen(v, o); }
};
template <> struct FzVec<float> {
  using T = float4;
  static constexpr int N = 4;
  __device__ __forceinline__ static void widen(const T& v, double* o) {
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
  }
  // x * 2^-896 exactly, for every finite x (normals, zeros and subnormals):
  // the fp32 exponent field lands in the low 8 bits of the fp64 one, so the
  // fp64 bias 1023 reads the fp32 bias 127 as 127 + 896; an fp32 subnormal
  // becomes the fp64 subnormal of the same mantissa.  Three integer ops
  // (shift, mask, shift) instead of an F2F.F64.F32 on the XU pipe.  Paired
  // with the other factor scaled by 2^896, fma(x', b', acc) == fma(x, b, acc)
  // bit for bit as long as b * 2^896 is finite.
  __device__ __forceinline__ static double rebias(float f) {
    const uint32_t u = __float_as_uint(f);
    const uint32_t hi = (uint32_t)((int32_t)u >> 3) & 0x8fffffffu;
    return __hiloint2double((int)hi, (int)(u << 29));
  }
  __device__ __forceinline__ static void widen_s(const T& v, double* o) {
    o[0] = rebias(v.x); o[1] = rebias(v.y); o[2] = rebias(v.z); o[3] = rebias(v.w);
  }
};

constexpr double kRebias = 0x1p896;                // scale paired with FzVec<float>::rebias
constexpr int kFzFwdWarps = 4;                      // forward warps
constexpr int kFzTrWarps = 8;                       // accumulate warps
constexpr int kFzTr = kFzTrWarps * 32;              // 256 accumulate threads

__device__ __forceinline__ double gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return (double)t;
}
// L0_PROBE builds (tools/probe_kfs.py): per-tile globaltimer stamps of CTA 0
// and CTA cs-1 into a.scratch, [cta][tile][which]: 0 forward start, 1 tile
// landed, 2 partials sent, 3 gather start, 4 accumulated, 5 refill issued
#ifdef L0_PROBE
#define FZ_STAMP(a, slotk, which)                                                           \
  do {                                                                                     \
    const int _c = (blockIdx.x == 0) ? 0 : ((int)blockIdx.x == a.fz_cs - 1 ? 1 : -1);     \
    if (_c >= 0 && (slotk) < 1000 && (_c * 1000 + (slotk)) * 6 + 6 <= a.pv)                 \
      a.scratch[(_c * 1000 + (slotk)) * 6 + (which)] = gtimer();                            \
  } while (0)
#else
#define FZ_STAMP(a, slotk, which) do { } while (0)
#endif

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(bar)) : "memory");
}

// Shared tail of the single-pass kernels: per-cluster transpose partials to
// fz_part, per-cluster loss / flags / F* sums to fz_cpart, and in the last CTA
// of the grid the fixed-order reduction over clusters and the objective /
// restart logic.  Transpose thread lt owns columns c0 + v*kFzTr*VE + lt*VE + e.
template <int NA, int VE, bool HASN, bool HASZ>
__device__ __forceinline__ void kf_finish(const EngineArgs& a, int mode, int64_t t, bool want_z, int cid,
                                          uint32_t crank, int64_t c0, bool is_tr, int lt,
                                          const double* accR, const double* accN, const double* accZ,
                                          double loss_acc, const double* f_acc, int bad, int gbad_R,
                                          int gbad_N, int* sbad, double* sred) {
  const int tid = threadIdx.x;
  const int cs = a.fz_cs;
  const int ncl = a.fz_ncl;
  const int64_t pv = a.pv;
  State* st = a.st;
  if (is_tr) {
#pragma unroll
    for (int v = 0; v < NA / VE; ++v) {
#pragma unroll
      for (int e = 0; e < VE; ++e) {
        const int64_t col = c0 + (int64_t)v * kFzTr * VE + lt * VE + e;
        if (col < pv) {
          a.fz_part[(0 * (int64_t)ncl + cid) * pv + col] = accR[v * VE + e];
          if constexpr (HASN) a.fz_part[(1 * (int64_t)ncl + cid) * pv + col] = accN[v * VE + e];
          if constexpr (HASZ) {
            if (want_z) a.fz_part[(2 * (int64_t)ncl + cid) * pv + col] = accZ[v * VE + e];
          }
        }
      }
    }
  }
  if (bad) *sbad = 1;
  if (gbad_R) atomicOr(sbad, 2);
  if (gbad_N) atomicOr(sbad, 4);
  double sums[4] = {loss_acc, f_acc[0], f_acc[1], f_acc[2]};
  block_sum4(sums, sred);
  const double lsum = sums[0], f0 = sums[1], f1 = sums[2], f2 = sums[3];
  if (crank == 0 && tid == 0) {
    double* cp = a.fz_cpart + 8 * (int64_t)cid;
    cp[0] = lsum;
    cp[1] = (double)*sbad;
    cp[2] = f0;
    cp[3] = f1;
    cp[4] = f2;
  }
  if (cs > 1) cluster_barrier();  // no st.async into this CTA is still in flight
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
    st->kf_token = 0;
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

// ---------------------------------------------------------------------------
// kf_fused_s: a row tile stays in its shared-memory stage until it has been
// accumulated into X^T r, so X crosses the SM <-> L2 interface once per
// iteration (round 1's first single-pass kernel re-read every tile from L2
// for the transpose and ran at 0.485 ms on C2, this one at 0.353 ms).  Four
// warp roles, no CTA-wide barrier on the per-tile path:
//   * forward (4 warps): split the tile's columns in quarters, keep their beta
//     quarter in registers, push per-(warp, row) partial dots to every CTA of
//     the cluster (st.async, transaction-count mbarrier per partial slot);
//   * gather (G warps, tiles round-robin): for tile k, sums the
//     cs x 4 partials of each row in a fixed order (identical in every CTA),
//     forms the residuals of the two momentum candidates and zeta (one lane
//     per row), publishes them in the stage's residual slot (rfull[stage]) and
//     re-arms the partial slot;
//   * accumulate (8 warps): each warp on its own, as soon as a stage's
//     residuals are published, accumulates its columns of X^T [r_R | r_N |
//     zeta] from the stage and arrives on empty[stage];
//   * producer (1 warp, one lane): refills a stage with tile k + S once all
//     eight accumulate warps left it.
// The gather of tile k+1 overlaps the accumulation of tile k, and the
// stage refill waits only for the accumulation.
// Slot reuse: a peer writes partial slot j only after its gather consumed my
// partial of tile j - S, i.e. after my forward of j - S, which needed my stage
// refilled after my accumulation (hence my gather, which re-armed the slot) of
// tile j - 2S: a slot ring of 2 S tiles is never written before it is re-armed.
constexpr int kFsMaxStages = 16;
constexpr int kFsMaxSlots = 32;
constexpr int kFsMaxR = 4;
// warps: forward 0..3 | gather 4..4+G-1 | producer | eight accumulate warps.
// G = 4 gather warps for fp64 X (17 warps, 96 registers per thread); fp32 X
// (1.5x the accumulators per thread) takes 2, so the 15-warp CTA keeps 128
// registers per thread without spills (3 spill), and 4-row tiles halve the
// per-tile gather work.
constexpr int kFsGatherWarp = kFzFwdWarps;
template <int G> constexpr int fs_prod_warp() { return kFzFwdWarps + G; }
template <int G> constexpr int fs_acc_warp0() { return kFzFwdWarps + G + 1; }
template <int G> constexpr int fs_block() { return (kFzFwdWarps + G + 1 + kFzTrWarps) * 32; }
// (fp64 X in 1-row tiles: 3 gather warps -- half the rows per tile -- make a
// 16-warp CTA, whose threads get 128 registers instead of 96)
template <typename TX, int R = 2> constexpr int fs_gather() { return sizeof(TX) == 8 ? (R == 1 ? 3 : 4) : 2; }

struct FsShared {
  uint64_t full[kFsMaxStages];        // stage landed (bulk-copy complete_tx)
  uint64_t empty[kFsMaxStages];       // the accumulate warps left the stage
  uint64_t rfull[kFsMaxStages];       // the stage's residuals are published
  uint64_t xb[kFsMaxSlots];           // partial slot complete (st.async from every peer)
  double sy[kFsMaxStages][kFsMaxR];   // y / u_{t-1} of the stage's rows (bulk copies)
  double su[kFsMaxStages][kFsMaxR];
  double rr[kFsMaxStages][3][kFsMaxR];   // r_R, r_N, zeta of the stage's rows
  double red[128];
  int bad;
};

__host__ __device__ constexpr size_t fs_align(size_t b) { return (b + 127) & ~size_t(127); }

// shared memory: FsShared | partial slots [NS][cs][4][R] | stages x (R x W x sizeof(TX))
// F32F (fp32 X only, FistaOptions.fp32_forward): the forward dots X beta use
// fp32 products of fp32 X and fp32-rounded beta in four fp32 chains per lane
// and row (24 products each on C3 / C5), reduced in fp64 from there on --
// BASELINE's "fp32 X with fp64 reductions", within the north star's 1e-5
// fp32-mode tolerance.  The transpose products stay fp64 (the gradient and
// the Fenchel bound are exact for the residuals the forward produced).
//
// LIN (squared error, whose gradient is affine in u): the gradients of both
// momentum candidates and X^T zeta follow from A_t = X^T grad F(u_t) alone,
//   X^T grad F(u_t + c (u_t - u_{t-1})) = A_t + c (A_t - A_{t-1}),  X^T zeta_t = -A_t,
// so the tile accumulates ONE residual vector instead of two or three (KR
// keeps A_{t-1} and forms the chosen candidate; fista.py:161-163, :152).
//
// SPEC (ONE = 2; logistic / squared hinge on fp32 X, where three accumulated
// vectors keep the kernel far from the HBM roofline): the tile accumulates the
// NO-RESTART candidate X^T grad F(u_t + c_N (u_t - u_{t-1})) only.  Iterations
// that restart, and bound checks (X^T zeta_t), take one extra transpose pass
// (the two-pass engine's K2, launched after KR and exiting at entry otherwise):
// ~1 in 6 iterations on C3 against 3x fewer accumulators, clusters of 4
// instead of 8 and a third of the gather's loss evaluations.
template <typename TX, int R, int NV, bool F32F = false, int ONE = 0>
__global__ void __launch_bounds__(fs_block<fs_gather<TX, R>()>(), 1) kf_fused_s(EngineArgs a, int mode) {
  // ONE = 3 is SPEC's bound-check variant: the no-restart candidate AND X^T
  // zeta_t (two vectors).  Both SPEC kernels are launched every iteration;
  // ONE = 2 returns at entry on bound-check iterations, ONE = 3 on all others
  // (EngineArgs::fz_spec2), so the conditional K2 pass is left with restarts.
  constexpr bool LIN = ONE == 1 || ONE == 2;   // one accumulated vector
  constexpr bool HASN = ONE == 0;              // accN: the second momentum candidate
  constexpr bool HASZ = ONE == 0 || ONE == 3;  // accZ: X^T zeta on bound checks
  constexpr int G = fs_gather<TX, R>();
  constexpr int kFsProdWarp = fs_prod_warp<G>();
  constexpr int kFsAccWarp0 = fs_acc_warp0<G>();
  constexpr int kFsBlock = fs_block<G>();
  extern __shared__ __align__(128) unsigned char smem[];
  using V = FzVec<TX>;
  constexpr int VE = V::N;
  constexpr int W = NV * kFzTr * VE;           // columns per CTA
  constexpr int QW = W / kFzFwdWarps;          // columns per forward warp
  constexpr int FV = QW / (32 * VE);           // vectors per forward lane per row
  static_assert(R <= kFsMaxR, "rows per tile");
  static_assert(FV * 32 * VE * kFzFwdWarps == W, "forward column split");
  FsShared& sh = *reinterpret_cast<FsShared*>(smem);
  const int cs = a.fz_cs;
  const int S = a.fz_stages;
  const int NS = a.fz_slots;
  double* part = reinterpret_cast<double*>(smem + fs_align(sizeof(FsShared)));
  const size_t part_bytes = fs_align((size_t)NS * cs * kFzFwdWarps * R * 8);
  TX* tiles = reinterpret_cast<TX*>(reinterpret_cast<unsigned char*>(part) + part_bytes);

  // Everything down to pdl_wait() is independent of the kernels before this
  // one (geometry, barrier init, the first S tiles of X): launched as a
  // programmatic dependent of K3 it runs while the prox is still working.
  pdl_launch();   // KR may become resident (it waits for this grid at its top)
  State* st = a.st;
  // which of the two SPEC kernels owns this iteration (bound check or not)
  auto not_mine = [&]() -> bool {
    if (ONE != 2 && ONE != 3) return false;
    if (ONE == 2 && !a.fz_spec2) return false;
    if (st->kf_token == 0) return true;   // the other kernel ran this iteration (t has advanced)
    const bool z = is_check(st->t + 1, a.prm->bci) || !isfinite(st->best_dual);
    return ONE == 2 ? z : !z;
  };
  if (!a.pdl && mode == MODE_ITER && (st->done || st->dual_only || not_mine())) return;
  const double cR = 0.25;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t crank = cs > 1 ? cluster_rank() : 0;
  const int cid = cs > 1 ? (int)cluster_id() : (int)blockIdx.x;
  const int ncl = a.fz_ncl;
  const int64_t n = a.n, ld = a.ld;
  const int64_t c0 = (int64_t)crank * W;
  const int wvalid = (int)max((int64_t)0, min((int64_t)W, ld - c0));
  const uint32_t row_bytes = (uint32_t)wvalid * (uint32_t)sizeof(TX);

  const int ntiles = (int)a.fz_tiles;
  const int mytiles = cid < ntiles ? (ntiles - cid + ncl - 1) / ncl : 0;
  auto tile_of = [&](int k) -> int64_t { return (int64_t)cid + (int64_t)k * ncl; };
  auto tile_rows = [&](int k) -> int { return (int)min((int64_t)R, n - tile_of(k) * R); };
  auto slot_bytes = [&](int k) -> uint32_t {
    return (uint32_t)(cs * kFzFwdWarps * tile_rows(k) * (int)sizeof(double));
  };
  // y / u_{t-1} ride along with a tile when their segments are 16-byte bulk copies
  const bool side_ok = (n % 2 == 0) && (R % 2 == 0);
  auto side = [&](int k) { return side_ok && (tile_rows(k) % 2 == 0); };

  // columns [wvalid, W) of every stage row are never copied: zero them once
  // so every role can run over full rows
  for (int i = tid; i < S * R * (W - wvalid); i += kFsBlock) {
    const int row = i / (W - wvalid), col = wvalid + i % (W - wvalid);
    tiles[(int64_t)row * W + col] = TX(0);
  }
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&sh.full[i], 1);
      mbar_init(&sh.empty[i], kFzTrWarps);
      mbar_init(&sh.rfull[i], 1);
    }
    for (int i = 0; i < NS; ++i) mbar_init(&sh.xb[i], 1);
    sh.bad = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int k = 0; k < NS && k < mytiles; ++k) mbar_arrive_expect(&sh.xb[k], slot_bytes(k));
  // a stage's transaction count covers the X rows and the side copies; the X
  // rows can be issued before the state of the solve is known
  auto side_bytes = [&](int k) -> uint32_t {
    return side(k) ? (uint32_t)tile_rows(k) * 8u * (mode == MODE_ITER ? 2u : 1u) : 0u;
  };
  auto issue_x = [&](int k, int b) {
    const int64_t tile = tile_of(k);
    const int rows = tile_rows(k);
    TX* dst = tiles + (int64_t)b * R * W;
    mbar_arrive_expect(&sh.full[b], row_bytes * rows + side_bytes(k));
    if (row_bytes > 0)
      for (int r = 0; r < rows; ++r)
        bulk_g2s(dst + (int64_t)r * W, static_cast<const TX*>(a.X) + (tile * R + r) * ld + c0,
                 row_bytes, &sh.full[b]);
  };
  auto issue_side = [&](int k, int b, const double* up) {
    if (side_bytes(k) == 0) return;
    const int64_t tile = tile_of(k);
    const uint32_t rb = (uint32_t)tile_rows(k) * 8u;
    bulk_g2s(&sh.sy[b][0], a.y + tile * R, rb, &sh.full[b]);
    if (mode == MODE_ITER) bulk_g2s(&sh.su[b][0], up + tile * R, rb, &sh.full[b]);
  };
  // the first S tiles only need this CTA's barriers: in flight across the
  // wait for the previous kernel and the cluster barrier (which orders the
  // peers' barrier init before any st.async)
  if (warp == kFsProdWarp && lane == 0)
    for (int k = 0; k < S && k < mytiles; ++k) issue_x(k, k);

  pdl_wait();     // K3's beta_t, the control state and u_{t-1} are complete from here on
  int64_t t = 0;
  double cN = 0.25;
  bool want_z = false;
  if (mode == MODE_ITER) {
    if (st->done || st->dual_only || not_mine()) {
      // nothing to do: complete the stages in flight before the CTA exits
      if (warp == kFsProdWarp && lane == 0) {
        for (int k = 0; k < S && k < mytiles; ++k) issue_side(k, k, a.u);
        for (int k = 0; k < S && k < mytiles; ++k) mbar_wait(&sh.full[k], 0u, a.fz_sleep);
      }
      return;
    }
    t = st->t + 1;
    cN = momentum(st->phi + 1);
    want_z = is_check(t, a.prm->bci) || !isfinite(st->best_dual);
  }
  const double* bsrc = (mode == MODE_ITER) ? a.beta + ring(t) * a.pv : a.beta;
  const double* uprev = a.u + ((mode == MODE_ITER) ? ring(t - 1) * n : 0);
  auto issue = [&](int k, int b) {
    issue_x(k, b);
    issue_side(k, b, uprev);
  };
  if (warp == kFsProdWarp && lane == 0)
    for (int k = 0; k < S && k < mytiles; ++k) issue_side(k, k, uprev);
  if (cs > 1) cluster_barrier();
  else __syncthreads();

  constexpr int NBN = HASN ? NV * VE : 1, NBZ = HASZ ? NV * VE : 1;
  double accR[NV * VE], accN[NBN], accZ[NBZ];
  double loss_acc = 0.0, f_acc[3] = {0.0, 0.0, 0.0};
  int bad = 0, gbad_R = 0, gbad_N = 0;

  if (warp < kFzFwdWarps) {
    // ===================== forward =====================
    const int qc = warp * QW;                  // this warp's column quarter
    double bq[FV * VE];
#pragma unroll
    for (int j = 0; j < FV; ++j)
#pragma unroll
      for (int e = 0; e < VE; ++e) {
        const int64_t col = c0 + qc + (j * 32 + lane) * VE + e;
        bq[j * VE + e] = col < a.p ? bsrc[col] : 0.0;
      }
    if constexpr (F32F) {
      // ---- fp32 mode: fp32 products, fp64 from the lane sums on ----
      float bf[FV * VE];
#pragma unroll
      for (int i = 0; i < FV * VE; ++i) bf[i] = (float)bq[i];
      int buf = 0, q = 0;
      uint32_t ph = 0;
      for (int k = 0; k < mytiles; ++k) {
        const int rows = tile_rows(k);
        mbar_wait(&sh.full[buf], ph, a.fz_sleep);
        const float* tl = reinterpret_cast<const float*>(tiles) + (int64_t)buf * R * W;
        double d[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float s4[4] = {0.f, 0.f, 0.f, 0.f};
          if (r < rows) {
#pragma unroll
            for (int j = 0; j < FV; ++j) {
              const float4 xv = *reinterpret_cast<const float4*>(tl + r * W + qc + (j * 32 + lane) * 4);
              s4[0] = fmaf(xv.x, bf[j * 4 + 0], s4[0]);
              s4[1] = fmaf(xv.y, bf[j * 4 + 1], s4[1]);
              s4[2] = fmaf(xv.z, bf[j * 4 + 2], s4[2]);
              s4[3] = fmaf(xv.w, bf[j * 4 + 3], s4[3]);
            }
          }
          d[r] = ((double)s4[0] + (double)s4[1]) + ((double)s4[2] + (double)s4[3]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int r = 0; r < R; ++r) d[r] += __shfl_xor_sync(0xffffffffu, d[r], o);
        if (lane < cs) {
#pragma unroll
          for (int r = 0; r < R; ++r)
            if (r < rows)
              st_async_f64(part + (((size_t)q * cs + crank) * kFzFwdWarps + warp) * R + r, &sh.xb[q],
                           (uint32_t)lane, d[r]);
        }
        if (++buf == S) { buf = 0; ph ^= 1u; }
        if (++q == NS) q = 0;
      }
    } else {
    // fp32 X: widen by integer rebias against beta * 2^896 (all of this
    // warp's beta finite after scaling; |beta| <= M keeps that true unless M
    // is within 2^-896 of the fp64 range)
    bool fint = sizeof(TX) == 4 && (a.fz_widen & 1);
    if (fint) {
      bool ok = true;
#pragma unroll
      for (int i = 0; i < FV * VE; ++i) ok = ok && isfinite(bq[i] * kRebias);
      fint = __all_sync(0xffffffffu, ok);
      if (fint)
#pragma unroll
        for (int i = 0; i < FV * VE; ++i) bq[i] *= kRebias;
    }
    auto fwd_loop = [&](auto INT) {
      constexpr bool kInt = decltype(INT)::value;
      int buf = 0, q = 0;
      uint32_t ph = 0;
      for (int k = 0; k < mytiles; ++k) {
        const int rows = tile_rows(k);
        if (tid == 0) FZ_STAMP(a, k, 0);
        mbar_wait(&sh.full[buf], ph, a.fz_sleep);
        if (tid == 0) FZ_STAMP(a, k, 1);
        const TX* tl = tiles + (int64_t)buf * R * W;
        double d[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          double d0 = 0.0, d1 = 0.0;
          if (r < rows) {
#pragma unroll
            for (int j = 0; j < FV; ++j) {   // columns >= wvalid are zero in every stage
              const int col = qc + (j * 32 + lane) * VE;
              double x[VE];
              const typename V::T xv = *reinterpret_cast<const typename V::T*>(tl + r * W + col);
              if (kInt) V::widen_s(xv, x);
              else V::widen(xv, x);
#pragma unroll
              for (int e = 0; e < VE; ++e) {
                if (((j * VE + e) & 1) == 0) d0 = fma(x[e], bq[j * VE + e], d0);
                else d1 = fma(x[e], bq[j * VE + e], d1);
              }
            }
          }
          d[r] = d0 + d1;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int r = 0; r < R; ++r) d[r] += __shfl_xor_sync(0xffffffffu, d[r], o);
        if (lane < cs) {
#pragma unroll
          for (int r = 0; r < R; ++r)
            if (r < rows)
              st_async_f64(part + (((size_t)q * cs + crank) * kFzFwdWarps + warp) * R + r, &sh.xb[q],
                           (uint32_t)lane, d[r]);
        }
        if (tid == 0) FZ_STAMP(a, k, 2);
        if (++buf == S) { buf = 0; ph ^= 1u; }
        if (++q == NS) q = 0;
      }
    };
    if (fint) fwd_loop(std::true_type{});
    else fwd_loop(std::false_type{});
    }
  } else if (warp < kFsGatherWarp + G) {
    // ===================== gather =====================
    const int gw = warp - kFsGatherWarp;
    const int np = cs * kFzFwdWarps;           // partials per row
    for (int k = gw; k < mytiles; k += G) {
      const int buf = k % S, q = k % NS;
      const uint32_t ph = (uint32_t)((k / S) & 1), qph = (uint32_t)((k / NS) & 1);
      const int rows = tile_rows(k);
      // y / u_{t-1} that do not ride with the tile (odd n, 1-row tiles): the
      // global loads go out before the waits
      double y_pre = 0.0, up_pre = 0.0;
      if (!side(k) && (lane / (32 / R)) < rows && (lane % (32 / R)) < 4) {
        const int64_t row = tile_of(k) * R + lane / (32 / R);
        y_pre = a.y[row];
        if (mode == MODE_ITER) up_pre = uprev[row];
      }
      mbar_wait_cluster(&sh.xb[q], qph, a.fz_sleep);
      mbar_wait(&sh.full[buf], ph, a.fz_sleep);            // y / u_{t-1} of the stage
      if (lane == 0) FZ_STAMP(a, k, 3);
      double us[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double v = lane < np ? part[((size_t)q * np + lane) * R + r] : 0.0;
        for (int j = lane + 32; j < np; j += 32) v += part[((size_t)q * np + j) * R + r];
        us[r] = v;
      }
      // butterfly that halves the live rows each round while more than one
      // is left: afterwards every lane of the group lane / (32 / R) holds the
      // cluster total u of that row (2R - 2 + 5 - log2 R shuffles, not 5R)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const int nl = (R * o / 16) > 1 ? R * o / 16 : 1;   // live rows before this round
        if (nl > 1) {
          const bool up = (lane & o) != 0;
#pragma unroll
          for (int i = 0; i < nl / 2; ++i) {
            const double keep = up ? us[i + nl / 2] : us[i];
            const double send = up ? us[i] : us[i + nl / 2];
            us[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
        } else {
          us[0] += __shfl_xor_sync(0xffffffffu, us[0], o);
        }
      }
      __syncwarp();
      if (lane == 0 && k + NS < mytiles) mbar_arrive_expect(&sh.xb[q], slot_bytes(k + NS));
      // four lanes per row, one loss evaluation each (the logistic ones are
      // exp / log1p chains; spreading them over lanes cuts the gather's
      // issue slots, which it shares with the forward and accumulate warps):
      //   f = 0: r_R = grad F(u + cR dlt)   f = 1: r_N = grad F(u + cN dlt)
      //   f = 2: zeta = -grad F(u) (+ F*(-zeta) terms)   f = 3: F(u), u out
      constexpr int GL = 32 / R;
      const int r = lane / GL, f = lane % GL;
      if (f < 4 && r < rows) {
        const double u = us[0];
        const int64_t row = tile_of(k) * R + r;
        (void)row;
        double yi, up;
        if (side(k)) {
          yi = sh.sy[buf][r];
          up = (mode == MODE_ITER) ? sh.su[buf][r] : u;
        } else {
          yi = y_pre;
          up = (mode == MODE_ITER) ? up_pre : u;
        }
        if ((ONE == 2 || ONE == 3) && f < 3) {
          // SPEC: the no-restart candidate (fista.py:161-162); ONE = 3 also zeta_t (fista.py:152)
          if (f == 0) {
            const double arg = dadd(u, dmul(cN, dsub(u, up)));
            if (!isfinite(arg)) gbad_N = 1;
            sh.rr[buf][0][r] = F32F ? loss_grad_f32m(a.loss, arg, yi) : loss_grad(a.loss, arg, yi);
          } else if (ONE == 3 && f == 2) {
            const double g = F32F ? loss_grad_f32m(a.loss, u, yi) : loss_grad(a.loss, u, yi);
            sh.rr[buf][2][r] = -g;
            if (crank == 0 && want_z) conj_accumulate(a.loss, -g, yi, f_acc);
          }
        } else if (ONE == 1 && f < 3) {
          // f = 0: grad F(u_t) (= -zeta_t); f = 1, 2: X gamma of the two
          // momenta must be finite (loss_gradient raises otherwise, model.py:215)
          if (f == 0) {
            const double g = F32F ? loss_grad_f32m(a.loss, u, yi) : loss_grad(a.loss, u, yi);
            sh.rr[buf][0][r] = g;
            if (crank == 0 && want_z) conj_accumulate(a.loss, -g, yi, f_acc);
          } else {
            const double arg = dadd(u, dmul(f == 1 ? cR : cN, dsub(u, up)));
            if (f == 1 && !isfinite(arg)) gbad_R = 1;
            if (f == 2 && !isfinite(arg)) gbad_N = 1;
          }
        } else if (f < 3) {
          const double dlt = dsub(u, up);
          // X gamma for the two momenta (fista.py:161-162); zeta_t = -grad F(u_t) (fista.py:152)
          const double arg = f == 0 ? dadd(u, dmul(cR, dlt)) : (f == 1 ? dadd(u, dmul(cN, dlt)) : u);
          if (f == 0 && !isfinite(arg)) gbad_R = 1;
          if (f == 1 && !isfinite(arg)) gbad_N = 1;
          const double g = F32F ? loss_grad_f32m(a.loss, arg, yi) : loss_grad(a.loss, arg, yi);
          sh.rr[buf][f][r] = f == 2 ? -g : g;
          if (f == 2 && crank == 0 && want_z) conj_accumulate(a.loss, -g, yi, f_acc);
        } else if (crank == 0) {
          if (mode == MODE_ITER) {
            a.u[ring(t) * n + row] = u;
          } else {
            a.u[row] = u;
            a.u[2 * n + row] = u;
          }
          if (!isfinite(u)) bad = 1;
          loss_acc += F32F ? loss_term_f32m(a.loss, u, yi) : loss_term(a.loss, u, yi);
        }
      } else if (f < (LIN ? 1 : 3)) {   // rows past n of a partial tile
        sh.rr[buf][f][r] = 0.0;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.rfull[buf]);
    }
  } else if (warp == kFsProdWarp) {
    // ===================== producer =====================
    if (lane == 0) {
      int buf = 0;
      uint32_t ph = 0;
      for (int k = 0; k + S < mytiles; ++k) {
        mbar_wait(&sh.empty[buf], ph, a.fz_sleep);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(k + S, buf);
        if (lane == 0) FZ_STAMP(a, k, 5);
        if (++buf == S) { buf = 0; ph ^= 1u; }
      }
    }
  } else {
    // ===================== accumulate =====================
    const int lt = tid - kFsAccWarp0 * 32;
#pragma unroll
    for (int i = 0; i < NV * VE; ++i) accR[i] = 0.0;
#pragma unroll
    for (int i = 0; i < NBN; ++i) accN[i] = 0.0;
#pragma unroll
    for (int i = 0; i < NBZ; ++i) accZ[i] = 0.0;
    int buf = 0;
    uint32_t ph = 0;
    for (int k = 0; k < mytiles; ++k) {
      const int rows = tile_rows(k);
      mbar_wait(&sh.rfull[buf], ph, a.fz_sleep);
      mbar_wait(&sh.full[buf], ph, a.fz_sleep);
      const TX* tl = tiles + (int64_t)buf * R * W + lt * VE;
      // fp32 X: integer-rebias widening against residuals * 2^896 when they
      // all stay finite after scaling (warp-uniform: every lane reads them)
      bool aint = false;
      if (sizeof(TX) == 4 && (a.fz_widen & 2) && rows == R) {
        aint = true;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          aint = aint && isfinite(sh.rr[buf][0][r] * kRebias);
          if constexpr (HASN) aint = aint && isfinite(sh.rr[buf][1][r] * kRebias);
          if constexpr (HASZ) aint = aint && (!want_z || isfinite(sh.rr[buf][2][r] * kRebias));
        }
      }
      auto acc_full = [&](auto INT) {
        constexpr bool kInt = decltype(INT)::value;
        const double sc = kInt ? kRebias : 1.0;
        // rows in pairs: a pair's loads are issued before its FMAs
        constexpr int RP = R >= 2 ? 2 : 1;
#pragma unroll
        for (int r0 = 0; r0 < R; r0 += RP) {
          typename V::T xv[RP][NV];
#pragma unroll
          for (int h = 0; h < RP; ++h)
#pragma unroll
            for (int v = 0; v < NV; ++v)
              xv[h][v] = *reinterpret_cast<const typename V::T*>(tl + (r0 + h) * W + v * kFzTr * VE);
#pragma unroll
          for (int h = 0; h < RP; ++h) {
            const int r = r0 + h;
            const double rR = sh.rr[buf][0][r] * sc;
            const double rN = HASN ? sh.rr[buf][1][r] * sc : 0.0;
            const double rZ = (HASZ && want_z) ? sh.rr[buf][2][r] * sc : 0.0;
            (void)rN; (void)rZ;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              double x[VE];
              if (kInt) V::widen_s(xv[h][v], x);
              else V::widen(xv[h][v], x);
#pragma unroll
              for (int e = 0; e < VE; ++e) {
                accR[v * VE + e] = fma(x[e], rR, accR[v * VE + e]);
                if constexpr (HASN) accN[v * VE + e] = fma(x[e], rN, accN[v * VE + e]);
              }
              if constexpr (HASZ) {
                if (want_z) {
#pragma unroll
                  for (int e = 0; e < VE; ++e) accZ[v * VE + e] = fma(x[e], rZ, accZ[v * VE + e]);
                }
              }
            }
          }
        }
      };
      if (aint) {
        acc_full(std::true_type{});
      } else if (rows == R) {
        acc_full(std::false_type{});
      } else {
        // the last, partial tile of the grid: rows past n hold stale data
        for (int r = 0; r < rows; ++r) {
          const double rR = sh.rr[buf][0][r];
          const double rN = HASN ? sh.rr[buf][1][r] : 0.0, rZ = HASZ ? sh.rr[buf][2][r] : 0.0;
          (void)rN; (void)rZ;
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            double x[VE];
            V::widen(*reinterpret_cast<const typename V::T*>(tl + r * W + v * kFzTr * VE), x);
#pragma unroll
            for (int e = 0; e < VE; ++e) {
              accR[v * VE + e] = fma(x[e], rR, accR[v * VE + e]);
              if constexpr (HASN) accN[v * VE + e] = fma(x[e], rN, accN[v * VE + e]);
              if constexpr (HASZ) {
                if (want_z) accZ[v * VE + e] = fma(x[e], rZ, accZ[v * VE + e]);
              }
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.empty[buf]);
      if (lt == 0) FZ_STAMP(a, k, 4);
      if (++buf == S) { buf = 0; ph ^= 1u; }
    }
  }
  __syncthreads();
  kf_finish<NV * VE, VE, HASN, HASZ>(a, mode, t, want_z, cid, crank, c0, warp >= kFsAccWarp0,
                         tid - kFsAccWarp0 * 32, accR, accN, accZ, loss_acc, f_acc, bad, gbad_R, gbad_N,
                         &sh.bad, sh.red);
}

// LIN: the chosen candidate from A_t (reduced over clusters / ranks) and the
// kept A_{t-1} (gv's no-restart block, unused in this mode):
//   g = A_t + c (A_t - A_{t-1}),  c = momentum after the restart decision
//   (fista.py:161-163; at the initial pass u_{-1} = u_0, so g = A_0),
//   X^T zeta_t = -A_t (fista.py:152).
__device__ __forceinline__ double lin_candidate(const EngineArgs& a, int mode, int64_t j, double At,
                                                bool wg, double* v) {
  double* keep = a.gv + 2 * a.pv + 8;
  *v = -At;
  if (j >= a.p) return 0.0;
  double g = At;
  if (mode == MODE_ITER) g = dadd(At, dmul(momentum(a.st->phi), dsub(At, keep[j])));
  if (wg) keep[j] = At;   // a bound-only pass re-reduces the same A_t
  return g;
}

// ---------------------------------------------------------------------------
// KR: reduce the per-cluster partials (fixed order), pick the candidate of
// the restart decision, slab epilogue.  One CTA per 256-column slab.
__global__ void __launch_bounds__(kK2Slab) kr_reduce(EngineArgs a, int mode, int epilogue) {
  __shared__ EpiSmem sm;
  pdl_wait();     // KF (programmatic dependent launch: this grid may be resident before KF ends)
  pdl_launch();   // ... and K3 behind this one
  const State* st = a.st;
  if (blockIdx.x == 0 && threadIdx.x == 0) a.st->kf_token = 1;   // next iteration's single pass
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
  if (a.fz_one == 2) {
    // SPEC: KF accumulated the no-restart candidate and, on bound-check
    // iterations (fz_spec2: the ONE = 3 kernel), X^T zeta_t; the restart
    // candidate, bound-only passes and (without fz_spec2) X^T zeta belong to
    // the K2 launch that follows (the two halves of the slab epilogue are
    // independent)
    if (mode == MODE_ITER && st->dual_only) return;
    const bool wg2 = mode != MODE_ITER || !st->last_restarted;
    const bool wz2 = mode == MODE_ITER && a.fz_spec2 && st->dual_pending;
    if (!wg2 && !wz2) return;
    if (j < p) {
      if (wg2) {
        for (int c = 0; c < ncl; ++c) g += __ldcg(a.fz_part + (int64_t)c * pv + j);
        a.gv[j] = g;
      }
      if (wz2) {
        for (int c = 0; c < ncl; ++c) v += __ldcg(a.fz_part + (2 * (int64_t)ncl + c) * pv + j);
        a.gv[pv + j] = v;
      }
    }
    if (wg2 && blockIdx.x == 0 && threadIdx.x == 0 && mode == MODE_ITER && ((int)a.gv[2 * pv + 6] & 4)) {
      State* sw = a.st;   // non-finite X gamma: loss_gradient raises (model.py:215)
      atomicExch(&sw->err, (int)ST_INVALID);
      sw->err_iter = sw->t + 1;
      sw->done = 1;
    }
    slab_epilogue(a, blockIdx.x, st->t + 1, momentum(st->phi), wg2, wz2, g, v, sm);
    return;
  }
  if (a.fz_one == 1) {
    // one partial vector A_t = X^T grad F(u_t) (kf_fused_s LIN)
    if (j < p)
      for (int c = 0; c < ncl; ++c) g += __ldcg(a.fz_part + (int64_t)c * pv + j);
    if (!epilogue) {  // row-sharded: A_t goes through the all-reduce, kr_pick extrapolates
      if (j < p) a.gv[j] = g;
      return;
    }
    const double gsel = lin_candidate(a, mode, j, g, wg, &v);
    if (j < p) {
      a.gv[j] = gsel;
      a.gv[pv + j] = v;
    }
    if (wg && blockIdx.x == 0 && threadIdx.x == 0) {
      const int flags = (int)a.gv[2 * pv + 6];
      if (flags & (use_R ? 2 : 4)) {
        State* sw = a.st;
        atomicExch(&sw->err, (int)ST_INVALID);
        sw->err_iter = sw->t + 1;
        sw->done = 1;
      }
    }
    slab_epilogue(a, blockIdx.x, st->t + 1, momentum(st->phi), wg, wz, gsel, v, sm);
    return;
  }
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
__global__ void __launch_bounds__(kK2Slab) kr_pick(EngineArgs a, int mode) {
  __shared__ EpiSmem sm;
  const State* st = a.st;
  if (st->done) return;
  const bool wg = st->dual_only == 0;
  const bool wz = st->dual_pending != 0;
  if (!wg && !wz) return;
  const int64_t pv = a.pv;
  const int64_t j = (int64_t)blockIdx.x * kK2Slab + threadIdx.x;
  const bool use_R = st->last_restarted != 0;
  const int64_t t = st->t + 1;
  if (a.fz_one == 1) {
    double v = 0.0;
    const double At = j < a.p ? a.gv[j] : 0.0;
    const double g = lin_candidate(a, mode, j, At, wg, &v);
    slab_epilogue(a, blockIdx.x, t, momentum(st->phi), wg, wz, g, v, sm);
    return;
  }
  const double g = j < a.p ? (use_R ? a.gv[j] : a.gv[2 * pv + 8 + j]) : 0.0;
  const double v = (wz && j < a.p) ? a.gv[pv + j] : 0.0;
  slab_epilogue(a, blockIdx.x, t, momentum(st->phi), wg, wz, g, v, sm);
}

// ---------------------------------------------------------------------------
// planning and launch
// ---------------------------------------------------------------------------
static size_t fused_smem(const EngineArgs& a) {
  const size_t es = a.dtype == F64 ? 8 : 4;
  return fs_align(sizeof(FsShared)) + fs_align((size_t)a.fz_slots * a.fz_cs * kFzFwdWarps * a.fz_rows * 8) +
         (size_t)a.fz_stages * (size_t)a.fz_rows * (size_t)a.fz_w * es;
}

using KfFn = void (*)(EngineArgs, int);

template <typename TX, int R, bool F32F, int ONE>
static KfFn kfs_pick_nv(int nv) {
  switch (nv) {
    case 1: return kf_fused_s<TX, R, 1, F32F, ONE>;
    case 2: return kf_fused_s<TX, R, 2, F32F, ONE>;
    case 3: return kf_fused_s<TX, R, 3, F32F, ONE>;
    case 4:
      if constexpr (sizeof(TX) == 8 || ONE != 0) return kf_fused_s<TX, R, 4, F32F, ONE>;
      return nullptr;
    case 5:
      if constexpr ((sizeof(TX) == 4 && ONE != 0 && R == 2) || (sizeof(TX) == 8 && ONE == 1 && R == 1))
        return kf_fused_s<TX, R, 5, F32F, ONE>;
      return nullptr;
    case 6:
      if constexpr ((sizeof(TX) == 4 && ONE != 0 && R == 2) || (sizeof(TX) == 8 && ONE == 1 && R == 1))
        return kf_fused_s<TX, R, 6, F32F, ONE>;
      return nullptr;
    case 7:
      if constexpr (sizeof(TX) == 8 && ONE == 1 && R == 1) return kf_fused_s<TX, R, 7, F32F, ONE>;
      return nullptr;
    case 8:
      if constexpr (sizeof(TX) == 8 && ONE == 1 && R == 1) return kf_fused_s<TX, R, 8, F32F, ONE>;
      return nullptr;
    default: return nullptr;
  }
}

template <typename TX, bool F32F, int ONE>
static KfFn kfs_pick_r(int rows, int nv) {
  if (rows == 1) {
    if constexpr (sizeof(TX) == 8 && ONE == 1) return nv > 4 ? kfs_pick_nv<TX, 1, F32F, ONE>(nv) : nullptr;
    return nullptr;
  }
  if (rows == 2) return kfs_pick_nv<TX, 2, F32F, ONE>(nv);
  if (rows == 4) {
    if constexpr (ONE != 2 && ONE != 3) return kfs_pick_nv<TX, 4, F32F, ONE>(nv);
  }
  return nullptr;
}

template <typename TX, bool F32F>
static KfFn kfs_pick_one(int one, int rows, int nv) {
  if (one == 1) return kfs_pick_r<TX, F32F, 1>(rows, nv);
  if (one == 2) {
    if constexpr (sizeof(TX) == 4) return kfs_pick_r<TX, F32F, 2>(rows, nv);
    return nullptr;
  }
  if (one == 3) {
    if constexpr (sizeof(TX) == 4) return kfs_pick_r<TX, F32F, 3>(rows, nv);
    return nullptr;
  }
  return kfs_pick_r<TX, F32F, 0>(rows, nv);
}

static KfFn kf_pick(const EngineArgs& a) {
  if (a.dtype == F64) return kfs_pick_one<double, false>(a.fz_one, a.fz_rows, a.fz_nv);
  if (a.f32_forward)   // fp32 mode (FistaOptions.fp32_forward)
    return kfs_pick_one<float, true>(a.fz_one, a.fz_rows, a.fz_nv);
  return kfs_pick_one<float, false>(a.fz_one, a.fz_rows, a.fz_nv);
}

static cudaError_t fused_config(const EngineArgs& a, cudaLaunchConfig_t& cfg, cudaLaunchAttribute* at,
                                KfFn* fn, bool pdl = false) {
  *fn = kf_pick(a);
  if (!*fn) return cudaErrorInvalidValue;
  const size_t smem = fused_smem(a);
  cudaError_t e = cudaFuncSetAttribute(*fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (a.fz_cs > 8) {
    e = cudaFuncSetAttribute(*fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cfg = cudaLaunchConfig_t{};
  cfg.gridDim = dim3((unsigned)(a.fz_cs * a.fz_ncl));
  cfg.blockDim = dim3(a.dtype == F64 ? (a.fz_rows == 1 ? fs_block<fs_gather<double, 1>()>()
                                                       : fs_block<fs_gather<double>()>())
                                     : fs_block<fs_gather<float>()>());
  cfg.dynamicSmemBytes = smem;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)a.fz_cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (pdl) {
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs = 2;
  }
  return cudaSuccess;
}

// Cluster size, rows per tile and ring depth: the smallest cluster (override:
// L0_FZ_CS) whose column slice fits the accumulate registers, R = 2 rows per
// tile for fp64 X (C2: 0.352 ms; R = 4 spills at 17 warps: 0.39 ms) and 4 for
// fp32 X with two or three accumulated vectors (C5: 9.96 vs 12.0 ms, C3: 1.18
// vs 1.59 ms; L0_FZ_R overrides); fp32 X in the LIN kernel takes 2-row tiles
// and up to 6 vectors per thread, i.e. half the cluster size (C5 at n = 200k:
// clusters of 2 x 5120 columns, 148 SMs, KF 1.17 ms = 6.85 TB/s against 1.67
// ms with 4-row tiles in clusters of 4 on 132 SMs), and as many stages as the shared memory holds next to the
// partial slots (<= kFsMaxStages; slots = 2 x stages, see the slot-reuse
// argument above; L0_FZ_S caps the stages).
int fused_plan(EngineArgs& a, int sms) {
  (void)sms;
  const int VE = a.dtype == F64 ? 2 : 4;
  const int64_t unit = (int64_t)kFzTr * VE;   // columns per accumulate-thread vector sweep
  const size_t es = a.dtype == F64 ? 8 : 4;
  const char* env = getenv("L0_FZ_CS");
  const int want_cs = env ? atoi(env) : 0;
  const char* renv = getenv("L0_FZ_R");
  const int R0 = renv ? (atoi(renv) == 4 ? 4 : 2) : ((a.dtype == F64 || a.fz_one) ? 2 : 4);
  // vectors per accumulate thread: the accumulator registers bound the column
  // slice (LIN keeps one accumulator per column instead of three); fp64 LIN
  // goes on to 8 vectors (4096 columns) with 1-row tiles, which keeps the
  // tile bytes and the ring depth of the 2-row x 2048-column plan in half
  // the cluster size (L0_FZ_WIDE=0: off)
  const bool wide64 = a.dtype == F64 && a.fz_one == 1 && !renv &&
                      (!getenv("L0_FZ_WIDE") || atoi(getenv("L0_FZ_WIDE")));
  const int maxv0 = a.dtype == F64 ? 4 : (a.fz_one ? (R0 == 2 ? 6 : 4) : 3);
  const int maxv = wide64 ? 8 : maxv0;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t budget = (size_t)(getenv("L0_FZ_KB") ? atoi(getenv("L0_FZ_KB")) * 1024 : std::max(optin, 0));
  for (int cs : {1, 2, 4, 8, 16}) {
    if (want_cs > 0 && cs != want_cs) continue;
    const int64_t need = (a.p + cs - 1) / cs;
    const int64_t W = ((need + unit - 1) / unit) * unit;
    const int nv = (int)(W / unit);
    if (nv > maxv) continue;
    const int R = nv > maxv0 ? 1 : R0;
    // stages S and slots 2S: fixed + 2S*cs*4*R*8 (+ align) + S*R*W*es <= budget
    const size_t fixed = fs_align(sizeof(FsShared)) + 128;
    if (fixed >= budget) continue;
    const size_t per = 2 * (size_t)cs * kFzFwdWarps * R * 8 + (size_t)R * (size_t)W * es;
    int S = (int)((budget - fixed) / per);
    S = std::min(S, std::min(kFsMaxStages, kFsMaxSlots / 2));
    if (getenv("L0_FZ_S")) S = std::min(S, atoi(getenv("L0_FZ_S")));
    if (S < 2) continue;
    a.fz_slots = 2 * S;
    // fp32 X: widen by integer rebias (bit 0 forward warps, bit 1 accumulate
    // warps) instead of F2F on the XU pipe; L0_FZ_WIDEN overrides
    // (LIN: forward warps only -- C5 at n = 200k: 1.168 vs 1.194 ms with both)
    a.fz_widen = getenv("L0_FZ_WIDEN") ? atoi(getenv("L0_FZ_WIDEN")) : (a.fz_one ? 1 : 3);
    a.fz_cs = cs;
    // suspend-time hint of the role waits (ns); L0_FZ_SLEEP overrides
    a.fz_sleep = getenv("L0_FZ_SLEEP") ? (uint32_t)atoi(getenv("L0_FZ_SLEEP")) : 1000u;
    a.fz_w = W;
    a.fz_nv = nv;
    a.fz_rows = R;
    a.fz_stages = S;
    a.fz_tiles = (a.n + R - 1) / R;
    a.fz_ncl = 1;   // grid of one cluster for the occupancy query
    int ncl = 0;
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute at[2];
    KfFn fn = nullptr;
    cudaError_t e = fused_config(a, cfg, at, &fn);
    if (e != cudaSuccess) {
      if (getenv("L0_DEBUG")) fprintf(stderr, "fused_plan: config %s\n", cudaGetErrorString(e));
      cudaGetLastError();
      return 0;
    }
    e = cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg);
    if (getenv("L0_DEBUG"))
      fprintf(stderr, "fused_plan: cs=%d W=%lld nv=%d R=%d S=%d slots=%d smem=%zu ncl=%d (%s)\n", cs,
              (long long)W, nv, R, S, a.fz_slots, fused_smem(a), ncl, cudaGetErrorString(e));
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
  cudaLaunchAttribute at[2];
  KfFn fn = nullptr;
  cudaError_t e = fused_config(a, cfg, at, &fn, a.pdl && mode == MODE_ITER);
  if (e != cudaSuccess) return e;
  cfg.stream = s;
  e = cudaLaunchKernelEx(&cfg, fn, a, mode);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_fused_reduce(const EngineArgs& a, int mode, cudaStream_t s) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3((unsigned)a.k2_slabs);
  cfg.blockDim = dim3(kK2Slab);
  cfg.stream = s;
  pdl_attr(cfg, at, a.pdl && mode == MODE_ITER);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kr_reduce, a, mode, a.multi ? 0 : 1);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_fused_pick(const EngineArgs& a, int mode, cudaStream_t s) {
  kr_pick<<<a.k2_slabs, kK2Slab, 0, s>>>(a, mode);
  return cudaGetLastError();
}

}  // namespace l0
