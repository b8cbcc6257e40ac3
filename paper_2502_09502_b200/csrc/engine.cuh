// Engine-wide kernel arguments and layout constants (shared by all .cu files).
#pragma once

#include "common.cuh"

namespace l0 {

// K1 (forward X.beta): CTA = 8 warps over a column slab of kK1Slab columns
// whose beta slice is staged in shared memory; warps stream rows.
constexpr int kK1Threads = 256;
constexpr int kK1Slab = 2048;
// K2 (transpose X^T r): CTA = 8 warps over one 256-column slab; each lane
// accumulates 8 columns in registers, the warps split the chunk's rows, and a
// fixed-order shared-memory tree combines the 8 warps.  Narrow slabs keep the
// cross-CTA partials small (chunks x p values).
constexpr int kK2Threads = 256;
constexpr int kK2Slab = 256;
constexpr int kK2StageRows = 256;                       // rows of r staged per pass
// 256-column slabs per K2 work item: fp32 items span two slabs so each row
// segment a CTA streams is 2 KB, as for fp64
template <typename TX> constexpr int kK2Cw = sizeof(TX) == 4 ? 2 : 1;
constexpr int kPvAlign = 2048;                          // p-vector stride alignment
constexpr int kTargetCtas = 148 * 4;
constexpr int kHTop = 32;   // per-slab Huber top list (bound checks with k <= 32)

enum KMode : int {
  MODE_ITER = 0,    // FISTA iteration (ring buffers, fused epilogues)
  MODE_INIT = 1,    // initial u_0 / objective
  MODE_PLAIN = 2,   // standalone matvec on explicit vectors
};

struct EngineArgs {
  // problem
  const void* X;
  const double* y;
  int64_t n, p, ld;
  int dtype;
  int loss;
  // launch layout
  int k1_slabs, k1_chunks, k1_grid;   // work items = slabs x chunks, persistent grid
  int k2_slabs, k2_chunks, k2_grid;
  int64_t k1_rows, k2_rows;   // rows per chunk
  int64_t pv;                 // stride of p-vectors (multiple of kPvAlign, >= ld)
  // FISTA vectors
  double* beta;      // ring [3][pv]
  double* u;         // ring [3][n]
  double* gam;       // gamma after the gradient step [pv]
  double* key;       // sort keys |rho*gamma| (or -1 for fixed coords) [pv]
  double* gv;        // [g (pv) | v = X^T zeta (pv) | F* acc (4) | loss, bad (2) | pad (2) | g_norestart (pv)]
  double* k2_part;   // [2][k2_chunks][pv]
  double* k2_fpart;  // [k2_chunks][4]
  double* u_part;    // [k1_slabs][n]
  double* loss_part; // [k1_chunks][2] (sum, non-finite count)
  unsigned* cnt;     // counters, see cnt_* helpers (zeroed once; kernels leave them zeroed)
  // prox
  double* xs;        // sorted keys [pv]
  int* perm;         // sorted coordinate ids [pv]
  int* iota;         // 0..p-1 (device sort path)
  double* tail;      // tail prefix sums [pv]
  double* scratch;   // [pv] scratch (Huber values, |beta|)
  const uint8_t* mask;  // node classes, nullable
  const int* fone;      // fixed-one ids (sorted), Params::n_fone of them
  // per-slab epilogue products (K2 -> K3), slabs of kK2Slab columns
  double* hval;      // Huber values of the bound check (free coords, -1 otherwise) [pv]
  double* cand_key;  // window candidates per slab [k2_slabs][kK2Slab]
  int* cand_idx;
  int* slab_cnt;     // candidates per slab
  double* slab_sum;  // sum |beta+| of non-candidate free coordinates per slab
  double* slab_max;  // max |beta+| of non-candidate free coordinates per slab
  double* slab_below;// largest positive free key below the candidate threshold per slab
  double* slab_hfone;// sum of fixed-one Huber values per slab
  double* slab_htop; // top-kHTop free Huber values per slab [k2_slabs][kHTop]
  // control
  State* st;
  const Params* prm;
  int multi;         // row-sharded: global epilogues run as separate kernels
  int plain_rhs2;    // PLAIN K2: number of RHS columns
  // single-physical-pass kernel (fused.cu): clusters of fz_cs CTAs span a row
  int fused;         // 1: iterations run K3 -> KF -> KR instead of K2 -> K3 -> K1
  int fz_cs, fz_ncl, fz_nv, fz_rows;   // cluster size, clusters, vectors/thread, rows/tile
  int fz_stages;     // shared-memory tile ring depth
  int fz_slots;      // partial-slot ring depth
  int fz_widen;      // fp32 X: bit 0 forward, bit 1 accumulate widen by integer rebias (fused.cu)
  int fz_one;        // single-pass kernel with ONE accumulated vector (fused.cu): 1 squared error
                     // (LIN: candidates by linearity), 2 SPEC (no-restart candidate; restarts
                     // and bound checks through the K2 launch that follows), 0 three vectors
  int pdl;           // single-pass chain launched as programmatic dependents (engine.cuh pdl_*)
  int fz_spec2;      // SPEC: bound-check iterations run the two-vector kernel (ONE = 3) instead of K2
  int k2_cond;       // K2 launched behind the SPEC kernel: runs only for restarts / bound passes
                     // (2: X^T zeta of bound checks comes from the ONE = 3 kernel)
  int f32_forward;   // fp32 X: forward products in fp32 (FistaOptions.fp32_forward; fused.cu)
  uint32_t fz_sleep;  // suspend-time hint (ns) of the single-pass kernel's mbarrier waits
  int64_t fz_w;      // columns per CTA (multiple of 256 * vector width)
  int64_t fz_tiles;  // row tiles
  double* fz_part;   // [3][fz_ncl][pv] transpose partials (restart / no-restart / zeta; LIN: [fz_ncl][pv])
  double* fz_cpart;  // [fz_ncl][8] per-cluster loss, non-finite, F* sums
  int prox_full_sort; // 1: K3 sorts all p keys (reference check path); 0: windowed sort
  // verification ring of K3 decisions (l0_problem_set_prox_record; nullptr: off):
  // per iteration kProxRecHead ints (see ProxRec) + the first prox_rec_w sorted ids
  int* prox_rec;
  int prox_rec_cap, prox_rec_w;
  // PLAIN-mode vectors
  const double* in_vec;
  double* out_vec;
  const double* in_vec2;
  double* out_vec2;
};

// counter block: [k2 work, k2 exit, k2 all | k1 work, k1 exit, k1 all | k2 slabs... | k1 chunks...]
__device__ __forceinline__ unsigned* cnt_k2_work(const EngineArgs& a) { return a.cnt + 0; }
__device__ __forceinline__ unsigned* cnt_k2_exit(const EngineArgs& a) { return a.cnt + 1; }
__device__ __forceinline__ unsigned* cnt_k2_all(const EngineArgs& a) { return a.cnt + 2; }
__device__ __forceinline__ unsigned* cnt_k1_work(const EngineArgs& a) { return a.cnt + 3; }
__device__ __forceinline__ unsigned* cnt_k1_exit(const EngineArgs& a) { return a.cnt + 4; }
__device__ __forceinline__ unsigned* cnt_k1_all(const EngineArgs& a) { return a.cnt + 5; }
__device__ __forceinline__ unsigned* cnt_k2_slab(const EngineArgs& a) { return a.cnt + 8; }
__device__ __forceinline__ unsigned* cnt_k1_chunk(const EngineArgs& a) { return a.cnt + 8 + a.k2_slabs; }
__device__ __forceinline__ unsigned* cnt_fused(const EngineArgs& a) { return a.cnt + 6; }
inline int64_t counter_words(int k2_slabs, int k1_chunks) { return 8 + k2_slabs + k1_chunks; }

__device__ __forceinline__ int64_t ring(int64_t t) { return ((t % 3) + 3) % 3; }

// FISTA momentum coefficient (fista.py:161): phi / (phi + 3.0)
__device__ __forceinline__ double momentum(int64_t phi) {
  double f = (double)phi;
  return ddiv(f, dadd(f, 3.0));
}

// bound check cadence (fista.py:182)
__device__ __forceinline__ bool is_check(int64_t t, int bci) { return t == 1 || (t % bci) == 0; }

// K3 decision record (prox.py:101-116 internals the parity tests compare with
// the oracle's stable argsort and PAVA pool): header fields, then ids
enum ProxRec : int {
  PR_ITER = 0,   // iteration whose beta the prox produced (fista.py:159 t)
  PR_HOW = 1,    // _prox_gstar_core case: 0 copy, 1 elementwise, 2 sort + PAVA
  PR_POOL = 2,   // 1: a merged pool [a*, c*] exists, 0: none
  PR_A = 3, PR_C = 4,   // pool bounds in sorted positions of the free coordinates
  PR_LEN = 5,    // sorted prefix length K3 materialised (all free coords: full sort)
  PR_PATH = 6,   // 0 window fast path, 1 window extensions, 2 full key sort
  PR_NFREE = 7,
  kProxRecHead = 8
};
// All threads of the K3 CTA call this after the pool search (a.perm holds the
// sorted prefix and is visible block-wide).
__device__ __forceinline__ void record_prox(int* rec, int cap, int w, const int* perm,
                                            int64_t iter, int how, int pool, int64_t astar,
                                            int64_t cstar, int64_t len, int path, int64_t nf) {
  if (rec == nullptr || cap <= 0) return;
  int* r = rec + (size_t)(iter % cap) * (size_t)(kProxRecHead + w);
  if (threadIdx.x == 0) {
    r[PR_ITER] = (int)iter;
    r[PR_HOW] = how;
    r[PR_POOL] = pool;
    r[PR_A] = pool ? (int)astar : -1;
    r[PR_C] = pool ? (int)cstar : -1;
    r[PR_LEN] = (int)len;
    r[PR_PATH] = path;
    r[PR_NFREE] = (int)nf;
  }
  const int64_t m = len < w ? len : w;
  for (int64_t i = threadIdx.x; i < w; i += blockDim.x)
    r[kProxRecHead + i] = i < m ? perm[i] : -1;
}

// Programmatic dependent launch (single-pass chain K3 -> KF -> KR -> K3 ...):
// a kernel launched with the attribute may become resident, and run whatever
// does not depend on its predecessor, once every CTA of the predecessor has
// executed pdl_launch(); pdl_wait() returns when the predecessor grid has
// completed and its writes are visible.  Every kernel of the chain waits at
// its top on every path, so completion stays transitive.  Both are no-ops in
// a launch without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
inline void pdl_attr(cudaLaunchConfig_t& cfg, cudaLaunchAttribute* at, bool on) {
  cfg.attrs = at;
  cfg.numAttrs = 0;
  if (on) {
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs = 1;
  }
}

// Launch helpers (defined in gemv.cu / prox.cu)
cudaError_t launch_k1(const EngineArgs& a, int mode, cudaStream_t s);
cudaError_t launch_k2(const EngineArgs& a, int mode, cudaStream_t s);
cudaError_t launch_grad_step(const EngineArgs& a, cudaStream_t s);
int k1_blocks_per_sm(int dtype);
int k2_blocks_per_sm(int dtype);
cudaError_t launch_objective(const EngineArgs& a, int mode, cudaStream_t s);
cudaError_t launch_fused(const EngineArgs& a, int mode, cudaStream_t s);
cudaError_t launch_fused_reduce(const EngineArgs& a, int mode, cudaStream_t s);
cudaError_t launch_fused_pick(const EngineArgs& a, int mode, cudaStream_t s);
int fused_plan(EngineArgs& a, int sms);   // 0: the problem does not fit the fused kernel
cudaError_t launch_prox_iter(const EngineArgs& a, void* sort_tmp, size_t sort_tmp_bytes,
                             cudaStream_t s);
size_t prox_sort_tmp_bytes(int64_t p);
bool prox_block_path(int64_t p);

}  // namespace l0
