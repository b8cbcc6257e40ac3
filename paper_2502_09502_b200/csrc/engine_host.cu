// Host side of the engine: problem layout, workspace carving, the FISTA driver
// loop (CUDA graphs of `chunk` iterations, device-resident control state), and
// NCCL row sharding.  fista.py:76-222 is the behaviour being reproduced.

#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <nccl.h>

#include "control.cuh"
#include "engine.cuh"
#include "prox.cuh"
#include "l0cert_b200.h"

namespace l0 {

thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define L0_CUDA_TRY(expr)                                                            \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess)                                                           \
      return set_error(ST_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

constexpr int L0_ABORTED_CODE = 6;

static inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
static inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// ---------------------------------------------------------------------------
// NCCL, resolved at run time (only row-sharded solves need it)
// ---------------------------------------------------------------------------
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  bool load(std::string* err) {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) { *err = "cannot dlopen libnccl.so.2"; return false; }
    commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
    allReduce = (decltype(allReduce))dlsym(h, "ncclAllReduce");
    commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
    getErrorString = (decltype(getErrorString))dlsym(h, "ncclGetErrorString");
    getUniqueId = (decltype(getUniqueId))dlsym(h, "ncclGetUniqueId");
    if (!commInitRank || !allReduce || !commDestroy) { *err = "NCCL symbols missing"; return false; }
    return true;
  }
};
static NcclApi g_nccl;

// ---------------------------------------------------------------------------
// problem
// ---------------------------------------------------------------------------
struct Graph {
  cudaGraphExec_t exec = nullptr;
  int G = 0;
  int profile = 0;
  int full_sort = 0;   // K3 variant captured (EngineArgs::prox_full_sort)
  int f32f = 0;        // single-pass kernel variant captured (EngineArgs::f32_forward)
  int64_t kernels = 0;
  std::vector<cudaEvent_t> ev;  // profile: [iter][k2b,k2e,k3b,k3e,k1b,k1e]
};

struct Problem {
  EngineArgs a{};
  int sm_count = 148;
  uint64_t ws_bytes = 0;
  void* ws = nullptr;
  void* sort_tmp = nullptr;
  size_t sort_tmp_bytes = 0;
  Params* d_prm = nullptr;
  double* d_small = nullptr;  // 64 doubles of scratch
  double* d_vec_n = nullptr;  // n doubles
  double* d_vec_p = nullptr;  // pv doubles
  uint8_t* d_mask = nullptr;
  int* d_fone = nullptr;
  State* h_st[2] = {nullptr, nullptr};  // pinned mirrors (double-buffered chunks)
  cudaStream_t stream = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr, ev_chunk[2] = {nullptr, nullptr};
  // [profile][K3 variant: windowed / full key sort][double-buffer slot]: every
  // variant stays captured, so a solve that switches K3 variants (C3) does not
  // re-capture its graphs in every call
  Graph graphs[2][2][2];
  Graph* graph = graphs[0][0];
  int fused_planned = 0;
  // single-pass plans: [0] the default kernel of the loss (LIN for squared
  // error, three vectors otherwise), [1] SPEC (one vector; non-linear losses
  // on fp32 X, single-GPU solves only: its conditional K2 launch has no
  // place between the all-reduces of the row-sharded path)
  struct FzPlan {
    int ok = 0, one = 0, cs = 1, ncl = 1, nv = 0, rows = 0, stages = 0, slots = 0, widen = 0;
    uint32_t sleep = 0;
    int64_t w = 0, tiles = 0;
  } plan[2];
  int plan_sel = 0;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  int force_full_sort = 0;      // re-run after a window tie overflow (ST_TIE_OVERFLOW)
  double trace_delivered = -1;  // ... skipping the trace records already delivered
};

}  // namespace l0

struct l0_problem : l0::Problem {};

namespace l0 {

// install a single-pass plan into the kernel arguments (graphs captured with
// another plan are dropped by the caller)
static void select_plan(Problem& P, int which) {
  EngineArgs& a = P.a;
  const Problem::FzPlan& pl = P.plan[which];
  P.plan_sel = which;
  a.fz_one = pl.one;
  a.fz_spec2 = (pl.one == 2 && (!getenv("L0_FZ_SPEC2") || atoi(getenv("L0_FZ_SPEC2")))) ? 1 : 0;
  a.fz_cs = pl.cs; a.fz_ncl = pl.ncl; a.fz_nv = pl.nv; a.fz_rows = pl.rows;
  a.fz_stages = pl.stages; a.fz_slots = pl.slots; a.fz_widen = pl.widen;
  a.fz_sleep = pl.sleep; a.fz_w = pl.w; a.fz_tiles = pl.tiles;
  a.fused = pl.ok;
  P.fused_planned = pl.ok;
  if (!pl.ok) { a.fz_ncl = 1; a.fz_cs = 1; }
}

static int compute_layout(Problem& P) {
  EngineArgs& a = P.a;
  const int64_t n = a.n, p = a.p;
  a.pv = round_up(std::max(p, a.ld), kPvAlign);
  int dev = 0;
  L0_CUDA_TRY(cudaGetDevice(&dev));
  L0_CUDA_TRY(cudaDeviceGetAttribute(&P.sm_count, cudaDevAttrMultiProcessorCount, dev));
  const int sms = P.sm_count > 0 ? P.sm_count : 148;
  // K1: kK1Slab-wide slabs, ~8 items per resident CTA
  a.k1_slabs = (int)ceil_div(p, kK1Slab);
  int64_t k1_res = (int64_t)sms * k1_blocks_per_sm(a.dtype);
  int64_t chunks = std::max<int64_t>(1, ceil_div(k1_res * 8, a.k1_slabs));
  const int64_t k1_min_rows = getenv("L0_K1_ROWS") ? atoi(getenv("L0_K1_ROWS")) : 8;
  chunks = std::min<int64_t>(chunks, std::max<int64_t>(1, ceil_div(n, k1_min_rows)));
  a.k1_rows = ceil_div(n, chunks);
  a.k1_chunks = (int)ceil_div(n, a.k1_rows);
  a.k1_grid = (int)std::min<int64_t>(k1_res, (int64_t)a.k1_slabs * a.k1_chunks);
  // K2: 256-column slabs
  a.k2_slabs = (int)ceil_div(p, kK2Slab);
  const int64_t k2_groups = ceil_div(a.k2_slabs, a.dtype == F32 ? kK2Cw<float> : kK2Cw<double>);
  int64_t k2_res = (int64_t)sms * k2_blocks_per_sm(a.dtype);
  chunks = std::max<int64_t>(1, ceil_div(k2_res * 8, k2_groups));
  // >= 64 rows per K2 item: on small X the cross-chunk reduction of the last
  // CTA per slab dominates (C1: 23.6 -> 17.2 us per K2); large X never hits
  // the cap.  L0_K2_ROWS / L0_K1_ROWS override.
  const int64_t k2_min_rows = getenv("L0_K2_ROWS") ? atoi(getenv("L0_K2_ROWS")) : 64;
  chunks = std::min<int64_t>(chunks, std::max<int64_t>(1, ceil_div(n, k2_min_rows)));
  a.k2_rows = ceil_div(n, chunks);
  a.k2_chunks = (int)ceil_div(n, a.k2_rows);
  a.k2_grid = (int)std::min<int64_t>(k2_res, k2_groups * a.k2_chunks);
  a.prox_full_sort = getenv("L0_FULL_SORT") ? atoi(getenv("L0_FULL_SORT")) : 0;
  // squared error: gradient candidates by linearity from one accumulated
  // vector (fused.cu LIN); L0_FZ_LIN=0 keeps the two-candidate kernel
  auto env_on = [](const char* k) { return !getenv(k) || atoi(getenv(k)) != 0; };
  auto plan_one = [&](int one) {
    Problem::FzPlan pl;
    a.fz_one = one;
    pl.ok = fused_plan(a, sms) ? 1 : 0;
    pl.one = one;
    if (pl.ok) {
      pl.cs = a.fz_cs; pl.ncl = a.fz_ncl; pl.nv = a.fz_nv; pl.rows = a.fz_rows;
      pl.stages = a.fz_stages; pl.slots = a.fz_slots; pl.widen = a.fz_widen;
      pl.sleep = a.fz_sleep; pl.w = a.fz_w; pl.tiles = a.fz_tiles;
    }
    return pl;
  };
  // L0_FZ_SPEC=0 keeps the three-vector kernel for non-linear losses on fp32 X
  if (a.loss != SQUARED_ERROR && a.dtype == F32 && env_on("L0_FZ_SPEC")) P.plan[1] = plan_one(2);
  P.plan[0] = plan_one((a.loss == SQUARED_ERROR && env_on("L0_FZ_LIN")) ? 1 : 0);
  select_plan(P, 0);
  P.sort_tmp_bytes = std::max(prox_sort_tmp_bytes(std::max<int64_t>(p, 1)), (size_t)256);
  size_t keys_only = 0;
  cub::DeviceRadixSort::SortKeysDescending<double>(nullptr, keys_only, (const double*)nullptr,
                                                   (double*)nullptr, (int)std::max<int64_t>(p, 1));
  P.sort_tmp_bytes = std::max(P.sort_tmp_bytes, keys_only);
  return ST_OK;
}

// carve the workspace; returns bytes needed (and assigns pointers when base != null)
static uint64_t carve(Problem& P, char* base) {
  EngineArgs& a = P.a;
  uint64_t off = 0;
  auto take = [&](uint64_t bytes) -> char* {
    off = (off + 255) & ~uint64_t(255);
    char* r = base ? base + off : nullptr;
    off += bytes;
    return r;
  };
  const int64_t n = a.n, pv = a.pv;
  P.d_prm = (Params*)take(sizeof(Params));
  a.st = (State*)take(sizeof(State));
  a.beta = (double*)take(8ull * 3 * pv);
  a.u = (double*)take(8ull * 3 * n);
  a.gam = (double*)take(8ull * pv);
  a.key = (double*)take(8ull * pv);
  a.xs = (double*)take(8ull * pv);
  a.tail = (double*)take(8ull * pv);
  a.scratch = (double*)take(8ull * pv);
  a.gv = (double*)take(8ull * (3 * pv + 8));
  a.k2_part = (double*)take(8ull * 2 * a.k2_chunks * pv);
  a.k2_fpart = (double*)take(8ull * 4 * a.k2_chunks);
  a.u_part = (double*)take(8ull * a.k1_slabs * n);
  a.loss_part = (double*)take(8ull * 2 * a.k1_chunks);
  a.cnt = (unsigned*)take(4ull * counter_words(a.k2_slabs, a.k1_chunks));
  a.perm = (int*)take(4ull * pv);
  a.iota = (int*)take(4ull * pv);
  a.hval = (double*)take(8ull * pv);
  a.cand_key = (double*)take(8ull * pv);
  a.cand_idx = (int*)take(4ull * pv);
  const int64_t S = a.k2_slabs;
  a.slab_cnt = (int*)take(4ull * S);
  a.slab_sum = (double*)take(8ull * S);
  a.slab_max = (double*)take(8ull * S);
  a.slab_below = (double*)take(8ull * S);
  a.slab_hfone = (double*)take(8ull * S);
  a.slab_htop = (double*)take(8ull * S * kHTop);
  const uint64_t ncl_max = (uint64_t)std::max(1, std::max(P.plan[0].ncl, P.plan[1].ncl));
  a.fz_part = (double*)take(8ull * 3 * ncl_max * pv);
  a.fz_cpart = (double*)take(8ull * 8 * ncl_max);
  P.d_mask = (uint8_t*)take(pv);
  P.d_fone = (int*)take(4ull * pv);
  P.sort_tmp = take(P.sort_tmp_bytes);
  P.d_small = (double*)take(8ull * 64);
  P.d_vec_n = (double*)take(8ull * n);
  P.d_vec_p = (double*)take(8ull * pv);
  a.prm = P.d_prm;
  return off + 256;
}

static void destroy_graphs(Problem& P) {
  for (auto& prof : P.graphs)
    for (auto& set : prof)
      for (auto& g : set) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        for (auto e : g.ev) cudaEventDestroy(e);
        g = Graph{};
      }
}

static int fused_tail(Problem& P, int mode, cudaStream_t s) {
  EngineArgs& a = P.a;
  L0_CUDA_TRY(launch_fused_reduce(a, mode, s));
  if (a.multi) {
    if (P.comm) {
      // LIN: A_t, the loss and the flags only (gv's third block keeps A_{t-1})
      ncclResult_t r = g_nccl.allReduce(a.gv, a.gv, (size_t)((a.fz_one == 1 ? 2 : 3) * a.pv + 8),
                                        ncclDouble, ncclSum, P.comm, s);
      if (r != ncclSuccess) return set_error(ST_CUDA, "ncclAllReduce (fused) failed");
    }
    L0_CUDA_TRY(launch_objective(a, mode, s));
    L0_CUDA_TRY(launch_fused_pick(a, mode, s));
  } else if (a.fz_one == 2 && mode == MODE_ITER) {
    // SPEC: restart iterations and bound passes take the two-pass engine's
    // transpose kernel (it exits at entry on every other iteration)
    EngineArgs a2 = a;
    a2.k2_cond = a.fz_spec2 ? 2 : 1;
    L0_CUDA_TRY(launch_k2(a2, MODE_ITER, s));
  }
  return ST_OK;
}

// one FISTA iteration's launches (captured into the chunk graph)
static int launch_iteration(Problem& P, cudaStream_t s, cudaEvent_t* ev) {
  EngineArgs& a = P.a;
  if (a.fused) {
    // K3 (prox of t) -> KF (single pass over X: u_t and both next gradients) -> KR
    if (ev) L0_CUDA_TRY(cudaEventRecordWithFlags(ev[2], s, cudaEventRecordExternal));
    L0_CUDA_TRY(launch_prox_iter(a, P.sort_tmp, P.sort_tmp_bytes, s));
    if (ev) L0_CUDA_TRY(cudaEventRecordWithFlags(ev[3], s, cudaEventRecordExternal));
    if (ev) L0_CUDA_TRY(cudaEventRecordWithFlags(ev[0], s, cudaEventRecordExternal));
    L0_CUDA_TRY(launch_fused(a, MODE_ITER, s));
    if (a.fz_one == 2 && a.fz_spec2) {   // SPEC: the bound-check iterations' two-vector kernel
      EngineArgs a3 = a;
      a3.fz_one = 3;
      L0_CUDA_TRY(launch_fused(a3, MODE_ITER, s));
    }
    if (ev) L0_CUDA_TRY(cudaEventRecordWithFlags(ev[1], s, cudaEventRecordExternal));
    if (ev) L0_CUDA_TRY(cudaEventRecordWithFlags(ev[4], s, cudaEventRecordExternal));
    int rc = fused_tail(P, MODE_ITER, s);
    if (rc) return rc;
    if (ev) L0_CUDA_TRY(cudaEventRecordWithFlags(ev[5], s, cudaEventRecordExternal));
    return ST_OK;
  }
  if (ev) L0_CUDA_TRY(cudaEventRecordWithFlags(ev[0], s, cudaEventRecordExternal));
  L0_CUDA_TRY(launch_k2(a, MODE_ITER, s));
  if (a.multi) {
    if (P.comm) {
      ncclResult_t r = g_nccl.allReduce(a.gv, a.gv, (size_t)(2 * a.pv + 3), ncclDouble, ncclSum,
                                        P.comm, s);
      if (r != ncclSuccess) return set_error(ST_CUDA, "ncclAllReduce (gradient) failed");
    }
    L0_CUDA_TRY(launch_grad_step(a, s));
  }
  if (ev) L0_CUDA_TRY(cudaEventRecordWithFlags(ev[1], s, cudaEventRecordExternal));
  if (ev) L0_CUDA_TRY(cudaEventRecordWithFlags(ev[2], s, cudaEventRecordExternal));
  L0_CUDA_TRY(launch_prox_iter(a, P.sort_tmp, P.sort_tmp_bytes, s));
  if (ev) L0_CUDA_TRY(cudaEventRecordWithFlags(ev[3], s, cudaEventRecordExternal));
  if (ev) L0_CUDA_TRY(cudaEventRecordWithFlags(ev[4], s, cudaEventRecordExternal));
  L0_CUDA_TRY(launch_k1(a, MODE_ITER, s));
  if (a.multi) {
    if (P.comm) {
      ncclResult_t r = g_nccl.allReduce(a.gv + 2 * a.pv + 4, a.gv + 2 * a.pv + 4, 2, ncclDouble,
                                        ncclSum, P.comm, s);
      if (r != ncclSuccess) return set_error(ST_CUDA, "ncclAllReduce (loss) failed");
    }
    L0_CUDA_TRY(launch_objective(a, MODE_ITER, s));
  }
  if (ev) L0_CUDA_TRY(cudaEventRecordWithFlags(ev[5], s, cudaEventRecordExternal));
  return ST_OK;
}

static int build_graph(Problem& P, int which, int G, int profile) {
  Graph& g = P.graph[which];
  if (g.exec && g.G == G && g.profile == profile && g.full_sort == P.a.prox_full_sort &&
      g.f32f == P.a.f32_forward)
    return ST_OK;
  if (g.exec) {
    cudaGraphExecDestroy(g.exec);
    for (auto e : g.ev) cudaEventDestroy(e);
    g = Graph{};
  }
  if (profile) {
    g.ev.resize((size_t)G * 6);
    for (auto& e : g.ev) L0_CUDA_TRY(cudaEventCreate(&e));
  }
  cudaStream_t s = P.stream;
  L0_CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  int rc = ST_OK;
  for (int i = 0; i < G && rc == ST_OK; ++i)
    rc = launch_iteration(P, s, profile ? &g.ev[(size_t)i * 6] : nullptr);
  if (rc == ST_OK) {
    cudaError_t e = cudaMemcpyAsync(P.h_st[which], P.a.st, sizeof(State), cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) rc = set_error(ST_CUDA, cudaGetErrorString(e));
  }
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(s, &graph);
  if (rc != ST_OK) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  if (e != cudaSuccess) return set_error(ST_CUDA, std::string("capture: ") + cudaGetErrorString(e));
  size_t nn = 0;
  L0_CUDA_TRY(cudaGraphGetNodes(graph, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn);
  L0_CUDA_TRY(cudaGraphGetNodes(graph, nodes.data(), &nn));
  int64_t kernels = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType t;
    cudaGraphNodeGetType(nd, &t);
    if (t == cudaGraphNodeTypeKernel) ++kernels;
  }
  e = cudaGraphInstantiate(&g.exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return set_error(ST_CUDA, std::string("instantiate: ") + cudaGetErrorString(e));
  g.G = G;
  g.profile = profile;
  g.full_sort = P.a.prox_full_sort;
  g.f32f = P.a.f32_forward;
  g.kernels = kernels;
  return ST_OK;
}

// g(beta) of an arbitrary vector (standalone path: sort |beta| then the
// envelope kernel), written to *d_out
static int envelope_of(Problem& P, const double* d_beta, int64_t kg, int64_t nf, double M,
                       const uint8_t* d_mask, const int* d_fone, int64_t n_fone, double* d_out,
                       cudaStream_t s, int64_t* launches) {
  EngineArgs& a = P.a;
  const int64_t p = a.p;
  int* flags = reinterpret_cast<int*>(P.d_small);
  L0_CUDA_TRY(cudaMemsetAsync(flags, 0, 8, s));
  const int blocks = (int)std::min<int64_t>(ceil_div(p, 256), 1024);
  k_abs_free<<<blocks, 256, 0, s>>>(d_beta, p, d_mask, M, a.scratch, flags);
  L0_CUDA_TRY(cudaGetLastError());
  size_t bytes = P.sort_tmp_bytes;
  L0_CUDA_TRY(cub::DeviceRadixSort::SortKeysDescending(P.sort_tmp, bytes, a.scratch, P.d_vec_p,
                                                       (int)p, 0, 64, s));
  k_g_value_final<<<1, 1024, 0, s>>>(P.d_vec_p, p, nf, kg, M, d_beta, d_fone, n_fone, flags,
                                     d_out);
  L0_CUDA_TRY(cudaGetLastError());
  if (launches) *launches += 4;
  return ST_OK;
}

static int auto_chunk(const Problem& P, int bci) {
  const EngineArgs& a = P.a;
  const double bytes = 2.0 * (double)a.n * (double)a.ld * (a.dtype == F64 ? 8.0 : 4.0);
  const double t_it = bytes / 6.0e12 + 40e-6;  // seconds, rough
  // ~16 ms of work per replay (L0_CHUNK_MS overrides): the loop is host-driven
  // -- every replay boundary needs the host thread within one chunk time to
  // keep two in flight -- and on a busy host 4 ms chunks lost up to 25-40% of a
  // C3 solve (C3 run-to-run); the bench's 20-iteration C2 solve
  // becomes a single replay
  const double chunk_s = getenv("L0_CHUNK_MS") ? std::max(0.5, atof(getenv("L0_CHUNK_MS"))) * 1e-3 : 16e-3;
  int G = (int)std::ceil(chunk_s / t_it);
  G = std::max(4, std::min(G, 100));
  (void)bci;
  return G;
}

}  // namespace l0

using namespace l0;

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* l0_last_error(void) { return g_last_error.c_str(); }
int32_t l0_abi_version(void) { return 1; }

int32_t l0_problem_create(const void* d_X, int32_t dtype, int64_t n, int64_t p, int64_t ld,
                          const double* d_y, int32_t loss, l0_problem** out) {
  if (!out) return set_error(ST_INVALID, "out is null");
  *out = nullptr;
  if (!d_X || !d_y) return set_error(ST_INVALID, "X and y must be device pointers");
  if (dtype != F64 && dtype != F32) return set_error(ST_INVALID, "dtype must be L0_F64 or L0_F32");
  if (n < 1 || p < 1) return set_error(ST_INVALID, "n and p must be positive");
  if (p > (int64_t)INT32_MAX - 4096) return set_error(ST_INVALID, "p too large");
  const int64_t es = dtype == F64 ? 8 : 4;
  if (ld < p || (ld * es) % 16 != 0) return set_error(ST_INVALID, "ld must be >= p and a multiple of 16 bytes");
  if (((uintptr_t)d_X) % 16 != 0) return set_error(ST_INVALID, "X must be 16-byte aligned");
  if (loss < 0 || loss > 4)
    return set_error(ST_UNSUPPORTED, "loss must be squared_error, logistic, squared_hinge, poisson or gamma");
  l0_problem* P = new l0_problem();
  P->a.X = d_X;
  P->a.y = d_y;
  P->a.n = n;
  P->a.p = p;
  P->a.ld = ld;
  P->a.dtype = dtype;
  P->a.loss = loss;
  int rc = compute_layout(*P);
  if (rc != ST_OK) { delete P; return rc; }
  P->ws_bytes = carve(*P, nullptr);
  cudaError_t e = cudaStreamCreateWithFlags(&P->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&P->ev_in, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&P->ev_out, cudaEventDisableTiming);
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&P->ev_chunk[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMallocHost((void**)&P->h_st[i], sizeof(State));
  }
  if (e != cudaSuccess) {
    l0_problem_destroy(P);
    return set_error(ST_CUDA, cudaGetErrorString(e));
  }
  *out = P;
  return ST_OK;
}

int32_t l0_problem_workspace_bytes(const l0_problem* prob, uint64_t* bytes) {
  if (!prob || !bytes) return set_error(ST_INVALID, "null argument");
  *bytes = prob->ws_bytes;
  return ST_OK;
}

int32_t l0_problem_set_workspace(l0_problem* P, void* d_ws, uint64_t bytes) {
  if (!P || !d_ws) return set_error(ST_INVALID, "null argument");
  if (bytes < P->ws_bytes) return set_error(ST_INVALID, "workspace too small");
  destroy_graphs(*P);
  P->ws = d_ws;
  carve(*P, (char*)d_ws);
  EngineArgs& a = P->a;
  L0_CUDA_TRY(cudaMemsetAsync(a.cnt, 0, 4 * counter_words(a.k2_slabs, a.k1_chunks), P->stream));
  L0_CUDA_TRY(cudaMemsetAsync(a.gv, 0, 8 * (3 * a.pv + 8), P->stream));
  k_iota<<<(int)std::min<int64_t>(ceil_div(a.pv, 256), 1024), 256, 0, P->stream>>>(a.iota, a.pv);
  L0_CUDA_TRY(cudaGetLastError());
  L0_CUDA_TRY(cudaStreamSynchronize(P->stream));
  return ST_OK;
}

int32_t l0_problem_destroy(l0_problem* P) {
  if (!P) return ST_OK;
  destroy_graphs(*P);
  if (P->comm && g_nccl.commDestroy) g_nccl.commDestroy(P->comm);
  for (int i = 0; i < 2; ++i) {
    if (P->h_st[i]) cudaFreeHost(P->h_st[i]);
    if (P->ev_chunk[i]) cudaEventDestroy(P->ev_chunk[i]);
  }
  if (P->ev_in) cudaEventDestroy(P->ev_in);
  if (P->ev_out) cudaEventDestroy(P->ev_out);
  if (P->stream) cudaStreamDestroy(P->stream);
  delete P;
  return ST_OK;
}

int32_t l0_debug_probe(l0_problem* P, int64_t* out16) {
  if (!P || !out16) return set_error(ST_INVALID, "null argument");
  for (int i = 0; i < 16; ++i) out16[i] = P->h_st[0]->probe[i];
  return ST_OK;
}

int32_t l0_problem_set_prox_record(l0_problem* P, int32_t* d_ring, int32_t cap, int32_t width) {
  if (!P) return set_error(ST_INVALID, "null argument");
  if (d_ring != nullptr && (cap < 1 || width < 0))
    return set_error(ST_INVALID, "prox record ring needs cap >= 1 and width >= 0");
  destroy_graphs(*P);   // the ring pointer is baked into the captured K3 launches
  P->a.prox_rec = d_ring;
  P->a.prox_rec_cap = d_ring ? cap : 0;
  P->a.prox_rec_w = d_ring ? width : 0;
  return ST_OK;
}

int32_t l0_debug_scratch(l0_problem* P, double* h_out, int64_t count) {
  if (!P || !h_out || !P->ws) return set_error(ST_INVALID, "null argument");
  count = std::min<int64_t>(count, P->a.pv);
  L0_CUDA_TRY(cudaStreamSynchronize(P->stream));
  L0_CUDA_TRY(cudaMemcpy(h_out, P->a.scratch, 8 * (size_t)count, cudaMemcpyDeviceToHost));
  return ST_OK;
}

int32_t l0_problem_set_comm(l0_problem* P, const void* h_id, int32_t nranks, int32_t rank) {
  if (!P) return set_error(ST_INVALID, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return set_error(ST_INVALID, "bad rank");
  destroy_graphs(*P);
  if (P->comm && g_nccl.commDestroy) g_nccl.commDestroy(P->comm);
  P->comm = nullptr;
  if (nranks == 1) {
    // h_id == NULL: run the row-sharded code path on one rank with the
    // all-reduces elided (tests the sharded kernels on a single GPU)
    P->a.multi = h_id == nullptr ? 1 : 0;
    P->nranks = 1;
    P->rank = 0;
    return ST_OK;
  }
  if (!h_id) return set_error(ST_INVALID, "NCCL unique id required for nranks > 1");
  std::string err;
  if (!g_nccl.load(&err)) return set_error(ST_CUDA, err);
  ncclUniqueId id;
  std::memcpy(&id, h_id, sizeof(id));
  ncclComm_t comm = nullptr;
  ncclResult_t r = g_nccl.commInitRank(&comm, nranks, id, rank);
  if (r != ncclSuccess)
    return set_error(ST_CUDA, std::string("ncclCommInitRank: ") +
                                  (g_nccl.getErrorString ? g_nccl.getErrorString(r) : "error"));
  P->comm = comm;
  P->nranks = nranks;
  P->rank = rank;
  P->a.multi = 1;
  return ST_OK;
}

int32_t l0_nccl_unique_id(void* h_out128) {
  if (!h_out128) return set_error(ST_INVALID, "null argument");
  std::string err;
  if (!g_nccl.load(&err)) return set_error(ST_CUDA, err);
  if (!g_nccl.getUniqueId) return set_error(ST_CUDA, "ncclGetUniqueId missing");
  ncclUniqueId id;
  if (g_nccl.getUniqueId(&id) != ncclSuccess) return set_error(ST_CUDA, "ncclGetUniqueId failed");
  std::memcpy(h_out128, &id, sizeof(id));
  return ST_OK;
}

static int check_ready(const l0_problem* P) {
  if (!P) return set_error(ST_INVALID, "null problem");
  if (!P->ws) return set_error(ST_INVALID, "problem has no workspace (l0_problem_set_workspace)");
  return ST_OK;
}

int32_t l0_fista_solve(l0_problem* P, int64_t k, double M, double lambda2,
                       const l0_fista_opts* o, const l0_node* node, const double* d_warm,
                       double* d_beta_out, l0_report* rep, l0_trace_cb cb, void* user,
                       void* stream) {
  int rc = check_ready(P);
  if (rc) return rc;
  if (!o || !rep || !d_beta_out) return set_error(ST_INVALID, "null argument");
  std::memset(rep, 0, sizeof(*rep));
  EngineArgs& a = P->a;
  const int64_t p = a.p;
  // ---- validation (model.py:102-107, fista.py:55-61, perspective.py:36-47) ----
  if (a.loss > SQUARED_HINGE)   // fista.py:92-95: the solver needs a Lipschitz-smooth loss
    return set_error(ST_UNSUPPORTED, "bound-grade loss: the relaxation solver needs a solver-grade loss");
  if (!(k >= 1 && k <= p)) return set_error(ST_INVALID, "k must satisfy 1 <= k <= p");
  if (!(M > 0 && std::isfinite(M))) return set_error(ST_INVALID, "M must be a positive finite real");
  if (!(lambda2 > 0 && std::isfinite(lambda2)))
    return set_error(ST_INVALID, "lambda2 must be a positive finite real");
  if (!(o->gap_tolerance > 0)) return set_error(ST_INVALID, "gap_tolerance must be positive");
  if (o->bound_check_interval < 1) return set_error(ST_INVALID, "bound_check_interval must be >= 1");
  if (o->max_iterations < 1) return set_error(ST_INVALID, "max_iterations must be >= 1");
  // fista.py:101 clamps any L to max(L, 1e-12) (an all-zero X gives L = 0);
  // only NaN is rejected
  if (std::isnan(o->lipschitz)) return set_error(ST_INVALID, "lipschitz constant is NaN");
  // row sharding over NCCL: every rank must replay the same number of chunks
  // (each holds all-reduces), so no rank may stop on its own host clock
  if (a.multi && P->comm && std::isfinite(o->time_limit))
    return set_error(ST_UNSUPPORTED, "time_limit is not available with row sharding over NCCL "
                                     "(ranks would stop after different chunks)");

  std::vector<uint8_t> mask;
  std::vector<int> fone;
  int64_t n1 = 0, n0 = 0;
  double parent_bound = -INFINITY;
  if (node) {
    parent_bound = node->parent_bound;
    n1 = node->n_fixed_one;
    n0 = node->n_fixed_zero;
    if (n1 + n0 > 0) {
      mask.assign((size_t)p, (uint8_t)FREE);
      for (int64_t i = 0; i < n1; ++i) {
        int64_t j = node->h_fixed_one[i];
        if (j < 0 || j >= p) return set_error(ST_INVALID, "fixed_one index out of range");
        if (mask[j] != FREE) return set_error(ST_INVALID, "duplicate fixed index");
        mask[j] = FIXED_ONE;
        fone.push_back((int)j);
      }
      for (int64_t i = 0; i < n0; ++i) {
        int64_t j = node->h_fixed_zero[i];
        if (j < 0 || j >= p) return set_error(ST_INVALID, "fixed_zero index out of range");
        if (mask[j] != FREE) return set_error(ST_INVALID, "fixed_one and fixed_zero must be disjoint");
        mask[j] = FIXED_ZERO;
      }
      std::sort(fone.begin(), fone.end());
    }
  }
  if (n1 > k) return set_error(ST_INFEASIBLE, "|fixed_one| exceeds the budget k");
  const bool node_mode = (n1 + n0) > 0;
  const int64_t nfree = p - n1 - n0;

  Params hp{};
  hp.L = std::max(o->lipschitz, 1e-12);   // fista.py:101
  hp.two_l2 = 2.0 * lambda2;              // fista.py:98
  hp.rho = hp.L / hp.two_l2;              // fista.py:102
  hp.M = M;
  hp.gap_tol = o->gap_tolerance;
  hp.gap_tol_rel = o->gap_tolerance_rel;
  hp.early_primal = o->early_primal_cutoff;
  hp.early_dual = o->early_dual_cutoff;
  hp.parent_bound = parent_bound;
  hp.max_iter = o->max_iterations;
  hp.k = k;
  hp.k_g = k - n1;
  hp.k_rem = std::min(k - n1, nfree);
  hp.n_free = nfree;
  hp.n_fone = n1;
  hp.bci = o->bound_check_interval;
  hp.restart = o->restart ? 1 : 0;
  hp.stop_on_gap = o->stop_on_gap ? 1 : 0;
  hp.node_mode = node_mode ? 1 : 0;
  hp.loss = a.loss;
  // engine path: auto = the single physical pass where it is measured faster
  // (X far beyond L2 with a 4..8-CTA cluster per row block: C2 2322 vs 1442
  // it/s, C5 73.6 vs 64.3, C3 even), the two-pass engine otherwise (small X:
  // L2 serves the second pass)
  const double x_bytes = (double)a.n * (double)a.ld * (a.dtype == F64 ? 8.0 : 4.0);
  {
    const int which = (P->plan[1].ok && !a.multi) ? 1 : 0;
    if (which != P->plan_sel) {
      destroy_graphs(*P);
      select_plan(*P, which);
    }
  }
  // (the one-vector kernels win from X just beyond L2 and without clusters as
  // well: a C4 node solve, 400 MB fp32, 5800 vs 3430 it/s)
  const int auto_fused = P->fused_planned && a.fz_cs >= (a.fz_one ? 1 : 4) && a.fz_cs <= 8 &&
                         x_bytes > (a.fz_one ? 128e6 : 512e6);   // L2-resident X (C1): the second pass hits L2
  const int want_fused = (o->engine_path == 2) ? P->fused_planned
                         : (o->engine_path == 1) ? 0 : auto_fused;
  if (o->engine_path == 2 && !P->fused_planned)
    return set_error(ST_UNSUPPORTED, "the single-pass kernel does not fit this problem");
  if (want_fused != a.fused) destroy_graphs(*P);
  a.fused = want_fused;
  a.f32_forward = (o->fp32_forward && a.dtype == F32 && a.fused) ? 1 : 0;
  // L0_PDL=1: the single-pass chain as programmatic dependent launches (KF's
  // first X tiles load while the prox runs; KR / K3 resident before their
  // predecessor ends); not with per-kernel events or NCCL kernels between the
  // launches.  Off by default: measured 1.3% slower on C2 (2814 vs 2850 it/s
  // at K = 200, profiles/r2_ab_pdl.txt), equal on C3 / C5
  {
    const int pdl = (a.fused && !a.multi && !o->profile && getenv("L0_PDL") &&
                     atoi(getenv("L0_PDL"))) ? 1 : 0;
    if (pdl != a.pdl) destroy_graphs(*P);
    a.pdl = pdl;
  }
  // K3 variant: the windowed top-of-order sort, switched to the full key sort
  // for the rest of the solve once most iterations of a chunk needed window
  // extensions (a PAVA pool spanning much of p, as on C3: K3 0.34 -> 0.19 ms);
  // L0_FULL_SORT=0/1 pins either variant
  const char* full_env = getenv("L0_FULL_SORT");
  a.prox_full_sort = full_env ? atoi(full_env) : P->force_full_sort;
  const bool auto_full = full_env == nullptr && !P->force_full_sort;
  // the captured graphs always see the node buffers; Params::node_mode gates their use
  a.mask = P->d_mask;
  a.fone = P->d_fone;
  const uint8_t* h_mask_ptr = node_mode ? P->d_mask : nullptr;
  const int* h_fone_ptr = node_mode ? P->d_fone : nullptr;

  auto t0 = std::chrono::steady_clock::now();
  cudaStream_t user_s = (cudaStream_t)stream;
  cudaStream_t s = P->stream;
  L0_CUDA_TRY(cudaEventRecord(P->ev_in, user_s));
  L0_CUDA_TRY(cudaStreamWaitEvent(s, P->ev_in, 0));
  L0_CUDA_TRY(cudaMemcpyAsync(P->d_prm, &hp, sizeof(Params), cudaMemcpyHostToDevice, s));
  if (node_mode) {
    L0_CUDA_TRY(cudaMemcpyAsync(P->d_mask, mask.data(), (size_t)p, cudaMemcpyHostToDevice, s));
    if (!fone.empty())
      L0_CUDA_TRY(cudaMemcpyAsync(P->d_fone, fone.data(), 4 * fone.size(), cudaMemcpyHostToDevice, s));
  }
  int64_t launches = 0;
  k_state_init<<<1, 1, 0, s>>>(a.st, parent_bound);
  ++launches;
  const size_t vb = 8ull * (size_t)p;
  if (d_warm) {
    L0_CUDA_TRY(cudaMemcpyAsync(a.beta, d_warm, vb, cudaMemcpyDeviceToDevice, s));
    L0_CUDA_TRY(cudaMemcpyAsync(a.beta + 2 * a.pv, d_warm, vb, cudaMemcpyDeviceToDevice, s));
    // g(beta_0) for the initial composite objective (fista.py:143)
    rc = envelope_of(*P, a.beta, hp.k_g, nfree, M, h_mask_ptr, h_fone_ptr, n1, &a.st->g_next, s,
                     &launches);
    if (rc) return rc;
  } else {
    L0_CUDA_TRY(cudaMemsetAsync(a.beta, 0, vb, s));
    L0_CUDA_TRY(cudaMemsetAsync(a.beta + 2 * a.pv, 0, vb, s));
  }
  if (a.fused) {
    // u_0 = X beta_0, F(u_0), objective, and the first gradient (fista.py:141-143, :162)
    L0_CUDA_TRY(launch_fused(a, MODE_INIT, s));
    rc = fused_tail(*P, MODE_INIT, s);
    if (rc) return rc;
    launches += a.multi ? 4 : 2;
  } else {
    L0_CUDA_TRY(launch_k1(a, MODE_INIT, s));  // u_0 = X beta_0, F(u_0), objective
    ++launches;
    if (a.multi) {
      if (P->comm && g_nccl.allReduce(a.gv + 2 * a.pv + 4, a.gv + 2 * a.pv + 4, 2, ncclDouble,
                                      ncclSum, P->comm, s) != ncclSuccess)
        return set_error(ST_CUDA, "ncclAllReduce (initial loss) failed");
      L0_CUDA_TRY(launch_objective(a, MODE_INIT, s));
      ++launches;
    }
  }

  // ---- chunked iteration: graph replays, double-buffered state mirrors ------
  // iterations that can ever run: max_iterations plus one bound-only pass
  // (fista.py:208-209); no chunk is launched past them, and the chunk size is
  // trimmed so that they tile into whole chunks (no trailing empty launches)
  const int64_t need = o->max_iterations + 1;
  int G = o->chunk_iterations > 0 ? std::min(o->chunk_iterations, 100)
                                  : auto_chunk(*P, o->bound_check_interval);
  if (o->chunk_iterations <= 0 && need < (int64_t)G * 64) {
    const int64_t nch = (need + G - 1) / G;
    G = (int)std::max<int64_t>(1, (need + nch - 1) / nch);
  }
  int64_t launched_its = 0;
  P->graph = P->graphs[o->profile ? 1 : 0][a.prox_full_sort ? 1 : 0];
  int64_t trace_seen = 0;
  int64_t chunks = 0;
  bool aborted = false, stop_sent = false, abort_deferred = false;
  int64_t t_before[2] = {0, 0};
  int64_t t_prev = 0, ext_prev = 0;
  State* last = nullptr;
  int inflight = 0;
  int next = 0;
  auto launch_chunk = [&](int w) -> int {
    // captured on first use (a solve that fits one replay never builds the second slot)
    int brc = build_graph(*P, w, G, o->profile ? 1 : 0);
    if (brc) return brc;
    L0_CUDA_TRY(cudaGraphLaunch(P->graph[w].exec, s));
    L0_CUDA_TRY(cudaEventRecord(P->ev_chunk[w], s));
    launched_its += G;
    return ST_OK;
  };
  // keep two chunks in flight
  for (int w = 0; w < 2 && launched_its < need; ++w) {
    rc = launch_chunk(w);
    if (rc) return rc;
    ++inflight;
  }
  while (inflight > 0) {
    const int w = next;
    next ^= 1;
    L0_CUDA_TRY(cudaEventSynchronize(P->ev_chunk[w]));
    --inflight;
    ++chunks;
    launches += P->graph[w].kernels;
    State* h = P->h_st[w];
    last = h;
    // profile: accumulate the kernel times of the iterations this chunk executed
    if (o->profile) {
      const int64_t did = std::max<int64_t>(0, std::min<int64_t>(G, h->t - t_prev));
      Graph& g = P->graph[w];
      // (right after a K3-variant switch this slot of the new set may not be
      // captured yet: the chunk that just finished belonged to the other set)
      for (int64_t i = 0; i < did && (size_t)(i * 6 + 5) < g.ev.size(); ++i) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, g.ev[i * 6 + 0], g.ev[i * 6 + 1]) == cudaSuccess) { rep->k2_ms += ms; rep->k2_count++; }
        if (cudaEventElapsedTime(&ms, g.ev[i * 6 + 2], g.ev[i * 6 + 3]) == cudaSuccess) { rep->k3_ms += ms; rep->k3_count++; }
        if (cudaEventElapsedTime(&ms, g.ev[i * 6 + 4], g.ev[i * 6 + 5]) == cudaSuccess) { rep->k1_ms += ms; rep->k1_count++; }
      }
    }
    // window extensions in this chunk -> full key sort from the next launch on
    const int64_t did_chunk = h->t - t_prev;
    const int64_t ext_now = (int64_t)h->win_ext + h->slow_prox;
    if (auto_full && !a.prox_full_sort && did_chunk >= 4 && 2 * (ext_now - ext_prev) >= did_chunk)
      a.prox_full_sort = 1;
    ext_prev = ext_now;
    t_prev = h->t;
    (void)t_before;
    // trace records, in order (fista.py:185-194)
    if (cb && !aborted) {
      for (; trace_seen < h->trace_count; ++trace_seen) {
        const TraceRec& r = h->trace[trace_seen % kTraceCap];
        if (r.iteration <= P->trace_delivered) continue;   // delivered before a re-run
        l0_trace_record rec{r.iteration, r.primal, r.dual, r.gap, r.restarted};
        if (cb(&rec, user) != 0) {
          if (a.multi && P->comm) {
            // sharded: keep replaying in step with the other ranks (their
            // all-reduces wait for ours); report the abort after the solve
            abort_deferred = true;
            cb = nullptr;
            break;
          }
          aborted = true;
          break;
        }
      }
    }
    if (h->done || aborted) {
      // drain the other in-flight chunk (all no-ops or the tail)
      if (inflight > 0) {
        L0_CUDA_TRY(cudaEventSynchronize(P->ev_chunk[next]));
        --inflight;
        ++chunks;
        launches += P->graph[next].kernels;
        if (P->h_st[next]->t >= h->t) last = P->h_st[next];
      }
      break;
    }
    const double elapsed = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (!stop_sent && elapsed > o->time_limit) {  // fista.py:204-206 (checked per chunk)
      k_request_stop<<<1, 1, 0, s>>>(a.st, P->d_prm, TERM_TIME_LIMIT);
      L0_CUDA_TRY(cudaGetLastError());
      ++launches;
      if (a.fused) {  // the final bound pass needs the Huber values of zeta_t
        rc = fused_tail(*P, MODE_ITER, s);
        if (rc) return rc;
        launches += a.fz_one == 2 ? 2 : 1;
      }
      stop_sent = true;
    }
    // nothing left that could run (the in-flight chunk finishes the solve);
    // with nothing in flight a chunk is launched anyway (never strand a solve)
    if (launched_its >= need && !stop_sent && inflight > 0) continue;
    if (P->graph[w].full_sort != a.prox_full_sort) {
      // (the chunk still in flight was launched from the other variant's set;
      // its kernel count is the same up to the sort kernels -- a statistic only)
      P->graph = P->graphs[o->profile ? 1 : 0][a.prox_full_sort ? 1 : 0];
    }
    rc = launch_chunk(w);
    if (rc) return rc;
    ++inflight;
  }
  const State* h = last;
  if (!aborted && h->err == ST_TIE_OVERFLOW && !a.prox_full_sort) {
    // an exact tie group larger than the prox window (prox_window.cu select_window):
    // the same deterministic solve on the full key sort, whose trajectory is
    // identical (test_k3_variants_agree); trace records already delivered are skipped
    L0_CUDA_TRY(cudaStreamSynchronize(s));
    double delivered = -1;
    for (int64_t i = std::max<int64_t>(0, trace_seen - kTraceCap); i < trace_seen; ++i)
      delivered = std::max(delivered, h->trace[i % kTraceCap].iteration);
    P->force_full_sort = 1;
    P->trace_delivered = cb ? delivered : -1;
    const int rc2 = l0_fista_solve(P, k, M, lambda2, o, node, d_warm, d_beta_out, rep, cb, user, stream);
    P->force_full_sort = 0;
    P->trace_delivered = -1;
    rep->gpu_launches += launches;
    return rc2;
  }
  if (aborted) {
    L0_CUDA_TRY(cudaStreamSynchronize(s));
    rep->status = L0_ABORTED_CODE;
    return set_error(L0_ABORTED_CODE, "aborted by the trace callback");
  }
  // ---- report (fista.py:213-222) -------------------------------------------
  rep->primal_value = h->obj;
  rep->dual_bound = h->best_dual;
  rep->gap = h->gap;
  rep->iterations = h->t;
  rep->restarts = h->restarts;
  rep->termination = h->termination;
  rep->status = h->err;
  rep->error_iteration = h->err_iter;
  rep->topk_fallbacks = h->topk_fallbacks;
  rep->prox_full_passes = h->slow_prox;
  rep->single_pass = a.fused;
  rep->cluster_size = a.fused ? a.fz_cs : 0;
  L0_CUDA_TRY(cudaMemcpyAsync(d_beta_out, a.beta + ((h->t % 3)) * a.pv, vb,
                              cudaMemcpyDeviceToDevice, s));
  L0_CUDA_TRY(cudaEventRecord(P->ev_out, s));
  L0_CUDA_TRY(cudaStreamWaitEvent(user_s, P->ev_out, 0));
  L0_CUDA_TRY(cudaStreamSynchronize(s));
  rep->gpu_launches = launches;
  rep->wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (abort_deferred) {
    rep->status = L0_ABORTED_CODE;
    return set_error(L0_ABORTED_CODE, "aborted by the trace callback (after the sharded solve)");
  }
  if (h->err != ST_OK) {
    if (h->err == ST_NUMERICAL)
      return set_error(ST_NUMERICAL, "composite objective became non-finite at iteration " +
                                         std::to_string(h->err_iter) +
                                         "; the step-size constant is likely too small");
    if (h->err == ST_INVALID) return set_error(ST_INVALID, "u contains non-finite entries");
    if (h->err == ST_UNSUPPORTED)
      return set_error(ST_UNSUPPORTED, "budget k exceeds the envelope kernel's top-k capacity (2048)");
    if (h->err == ST_TIE_OVERFLOW)
      return set_error(ST_UNSUPPORTED, "exact tie group larger than the prox window (4096 keys)");
    return set_error(h->err, "solve failed");
  }
  return ST_OK;
}

}  // extern "C"
