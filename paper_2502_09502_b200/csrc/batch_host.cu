// Host side of the batched node engine (SURVEY.md §8(a) a6 batched, north
// star item 4): many branch-and-bound node relaxations on one shared X,
// advanced in lockstep by CUDA graphs of G iterations; the two X passes of an
// iteration are tcgen05 contractions over all nodes (tc_gemm.cu).
#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "batch_ops.cuh"
#include "tc_gemm.cuh"
#include "l0cert_b200.h"

namespace l0 {

struct Batch {
  const l0_problem* prob = nullptr;
  BatchArgs g{};
  int64_t n = 0, p = 0, B = 0;
  int sms = 148;
  uint64_t ws_bytes = 0;
  void* ws = nullptr;
  __half *xh = nullptr, *xl = nullptr, *xth = nullptr, *xtl = nullptr;   // 3xFP16 splits of X (scaled)
  unsigned* xmax = nullptr;      // max |X| (float bits) for the X scale
  TcGemmArgs gf{}, gt{}, gfs{};   // forward (dense: MODE_INIT), transpose, forward (support-compacted)
  CUtensorMap m_xh{}, m_xl{}, m_xth{}, m_xtl{}, m_bh{}, m_bl{}, m_rh{}, m_rl{};
  CUtensorMap m_xuh{}, m_xul{}, m_bsh{}, m_bsl{};
  int sparse = 1;                // support-compacted forward contraction (L0_SPARSE_FWD=0: dense)
  int* h_flags = nullptr;   // pinned mirror of flags[0..8)
  cudaStream_t stream = nullptr;
  cudaEvent_t ev_in = nullptr, ev_chunk = nullptr;
  cudaGraphExec_t exec = nullptr;
  int G = 0;
  int profile = 0;
  std::vector<cudaEvent_t> ev;   // profile: [iter][gemm_t b,e | step+window b,e | gemm_f b,e]
  int64_t graph_kernels = 0;
  int sf_cap = 1, sct_cap = 1;   // split-K partial capacity carved for the measured choice
  int streamk = 0;               // stream-K contractions (L0_TC_SK=1; default: tuned split-K)
  float* sk_part = nullptr;      // stream-K partials [sms][kTcBN][kTcBM]
  int* sk_flag = nullptr;        // [sms]
};

static uint64_t batch_carve(Batch& Bt, char* base) {
  BatchArgs& g = Bt.g;
  uint64_t off = 0;
  auto take = [&](uint64_t bytes) -> char* {
    off = (off + 1023) & ~uint64_t(1023);
    char* r = base ? base + off : nullptr;
    off += bytes;
    return r;
  };
  const int64_t n = g.n, p = g.p, B = g.B, pv = g.pv, pp = g.pp, nn = g.nn;
  Bt.xh = (__half*)take(2ull * n * pp);
  Bt.xl = (__half*)take(2ull * n * pp);
  Bt.xth = (__half*)take(2ull * p * nn);
  Bt.xtl = (__half*)take(2ull * p * nn);
  Bt.xmax = (unsigned*)take(4ull);
  g.bh = (__half*)take(2ull * B * pp);
  g.bl = (__half*)take(2ull * B * pp);
  g.rh = (__half*)take(2ull * 2 * B * nn);
  g.rl = (__half*)take(2ull * 2 * B * nn);
  g.rinv = (float*)take(4ull * 2 * B);
  g.binv = (float*)take(4ull * B);
  g.gbound = (double*)take(8ull * B * g.rblocks);
  g.cf = (float*)take(4ull * Bt.sf_cap * B * nn);
  g.ct = (float*)take(4ull * Bt.sct_cap * 2 * B * pp);
  g.u = (double*)take(8ull * 3 * B * nn);
  g.st = (State*)take(sizeof(State) * B);
  g.prm = (Params*)take(sizeof(Params) * B);
  g.beta = (double*)take(8ull * 3 * B * pv);
  g.gam = (double*)take(8ull * B * pv);
  g.key = (double*)take(8ull * B * pv);
  g.xs = (double*)take(8ull * B * pv);
  g.tail = (double*)take(8ull * B * pv);
  g.scratch = (double*)take(8ull * B * pv);
  g.perm = (int*)take(4ull * B * pv);
  g.gv = (double*)take(8ull * B * (3 * pv + 8));
  g.mask = (uint8_t*)take(1ull * B * pv);
  g.fone = (int*)take(4ull * B * g.fone_stride);
  g.fpart = (double*)take(8ull * 4 * B * g.rblocks);
  g.lpart = (double*)take(8ull * 2 * B * g.rblocks);
  g.cnt = (unsigned*)take(4ull * B);
  g.hval = (double*)take(8ull * B * pv);
  g.cand_key = (double*)take(8ull * B * pv);
  g.cand_idx = (int*)take(4ull * B * pv);
  g.slab_cnt = (int*)take(4ull * B * g.S);
  g.slab_sum = (double*)take(8ull * B * g.S);
  g.slab_max = (double*)take(8ull * B * g.S);
  g.slab_below = (double*)take(8ull * B * g.S);
  g.slab_hfone = (double*)take(8ull * B * g.S);
  g.slab_htop = (double*)take(8ull * B * g.S * kHTop);
  g.flags = (int*)take(4ull * 8);
  g.slot = (int*)take(4ull * B);
  Bt.sk_part = Bt.streamk ? (float*)take(4ull * Bt.sms * kTcBN * kTcBM) : nullptr;
  Bt.sk_flag = Bt.streamk ? (int*)take(4ull * Bt.sms) : nullptr;
  g.sparse_fwd = Bt.sparse;
  if (Bt.sparse) {
    g.umask = (int*)take(4ull * pp);
    g.slot_of = (int*)take(4ull * pp);
    g.col_of = (int*)take(4ull * pp);
    g.uctl = (int*)take(4ull * 8);
    g.xuh = (__half*)take(2ull * n * pp);
    g.xul = (__half*)take(2ull * n * pp);
    g.bsh = (__half*)take(2ull * B * pp);
    g.bsl = (__half*)take(2ull * B * pp);
    g.fx_n = (int*)take(4ull * B);
    g.fx_j = (int*)take(4ull * B * kFoneDirect);
    g.fx_v = (double*)take(8ull * B * kFoneDirect);
    g.xth = Bt.xth;
    g.xtl = Bt.xtl;
  }
  return off + 1024;
}

static void batch_destroy_graph(Batch& Bt) {
  if (Bt.exec) cudaGraphExecDestroy(Bt.exec);
  for (auto e : Bt.ev) cudaEventDestroy(e);
  Bt.ev.clear();
  Bt.exec = nullptr;
  Bt.G = 0;
  Bt.profile = 0;
}

#define L0_B_TRY(expr)                                                                \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess)                                                            \
      return set_error(ST_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

static int batch_iteration(Batch& Bt, cudaStream_t s, cudaEvent_t* ev) {
  BatchArgs& g = Bt.g;
  const dim3 rgrid((unsigned)g.rblocks, (unsigned)g.B);
  auto rec = [&](int i) -> cudaError_t {
    return ev ? cudaEventRecordWithFlags(ev[i], s, cudaEventRecordExternal) : cudaSuccess;
  };
  kb_compact<<<1, 1024, 0, s>>>(g);
  kb_rhs<<<rgrid, kRowThreads, 0, s>>>(g);
  kb_plan<<<1, 1, 0, s>>>(g);
  L0_B_TRY(cudaGetLastError());
  L0_B_TRY(rec(0));
  L0_B_TRY(tc_gemm_launch(Bt.m_xth, Bt.m_xtl, Bt.m_rh, Bt.m_rl, Bt.gt, std::min(Bt.gt.units, Bt.sms), s));
  L0_B_TRY(rec(1));
  L0_B_TRY(rec(2));
  L0_B_TRY(kb_prox_launch(g, s));
  L0_B_TRY(rec(3));
  L0_B_TRY(rec(4));
  if (Bt.sparse) {
    // union of the operand supports -> X column cache, then the compacted contraction
    L0_B_TRY(kb_sparse_fwd_prep(g, Bt.sms * 4, s));
    L0_B_TRY(tc_gemm_launch(Bt.m_xuh, Bt.m_xul, Bt.m_bsh, Bt.m_bsl, Bt.gfs, std::min(Bt.gfs.units, Bt.sms), s));
  } else {
    L0_B_TRY(tc_gemm_launch(Bt.m_xh, Bt.m_xl, Bt.m_bh, Bt.m_bl, Bt.gf, std::min(Bt.gf.units, Bt.sms), s));
  }
  L0_B_TRY(rec(5));
  kb_obj<<<rgrid, kRowThreads, 0, s>>>(g, MODE_ITER);
  L0_B_TRY(cudaGetLastError());
  return ST_OK;
}

static int batch_build_graph(Batch& Bt, int G, int profile) {
  if (Bt.exec && Bt.G == G && Bt.profile == profile) return ST_OK;
  batch_destroy_graph(Bt);
  if (profile) {
    Bt.ev.resize((size_t)G * 6);
    for (auto& e : Bt.ev) L0_B_TRY(cudaEventCreate(&e));
  }
  cudaStream_t s = Bt.stream;
  L0_B_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  int rc = ST_OK;
  for (int i = 0; i < G && rc == ST_OK; ++i) rc = batch_iteration(Bt, s, profile ? &Bt.ev[(size_t)i * 6] : nullptr);
  if (rc == ST_OK) {
    kb_count<<<1, 256, 0, s>>>(Bt.g);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(Bt.h_flags, Bt.g.flags, 8 * sizeof(int), cudaMemcpyDeviceToHost, s);
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
  L0_B_TRY(cudaGraphGetNodes(graph, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn);
  L0_B_TRY(cudaGraphGetNodes(graph, nodes.data(), &nn));
  int64_t kernels = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType t;
    cudaGraphNodeGetType(nd, &t);
    if (t == cudaGraphNodeTypeKernel) ++kernels;
  }
  e = cudaGraphInstantiate(&Bt.exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return set_error(ST_CUDA, std::string("instantiate: ") + cudaGetErrorString(e));
  Bt.G = G;
  Bt.profile = profile;
  Bt.graph_kernels = kernels;
  return ST_OK;
}

__global__ void kb_gather_beta(BatchArgs g, double* out) {
  const int64_t b = blockIdx.y;
  const int64_t slot = ring(g.st[b].t);
  const double* src = g.beta + (b * 3 + slot) * g.pv;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < g.p; j += (int64_t)gridDim.x * blockDim.x)
    out[b * g.p + j] = src[j];
}

}  // namespace l0

struct l0_batch : l0::Batch {};

using namespace l0;

// Split-K of the forward contraction, measured: every split count up to the
// carved capacity is timed on the real operands (all node rows live; two
// launches each after a warm-up) and the fastest kept (C4: 8 splits, 0.42 ms,
// vs the model's 2, 0.50 ms -- the model underrates the wave quantisation of
// splits x tiles over the SMs).  The transpose keeps the model's choice.
static cudaError_t tune_one(Batch& Bt, TcGemmArgs& gm, const CUtensorMap& ah, const CUtensorMap& al,
                            const CUtensorMap& bh, const CUtensorMap& bl, int cap, cudaStream_t s) {
  if (cap <= 1) return cudaSuccess;
  cudaEvent_t e0, e1;
  cudaError_t e = cudaEventCreate(&e0);
  if (e != cudaSuccess) return e;
  e = cudaEventCreate(&e1);
  if (e != cudaSuccess) return e;
  int best = gm.S;
  float best_ms = 1e30f;
  for (int S = 1; S <= cap; ++S) {
    if (S > 1 && gm.kb_total / S < 4) break;
    TcGemmArgs g = gm;
    g.S = S;
    g.units = S * g.m_tiles * g.n_tiles;
    const int grid = std::min(g.units, Bt.sms);
    e = tc_gemm_launch(ah, al, bh, bl, g, grid, s);
    if (e != cudaSuccess) break;
    cudaEventRecord(e0, s);
    for (int r = 0; r < 2; ++r) tc_gemm_launch(ah, al, bh, bl, g, grid, s);
    cudaEventRecord(e1, s);
    e = cudaEventSynchronize(e1);
    if (e != cudaSuccess) break;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (getenv("L0_DEBUG")) fprintf(stderr, "tune M=%lld N=%lld K=%lld S=%d: %.4f ms\n", (long long)g.M,
                                    (long long)g.N, (long long)g.K, S, ms / 2);
    if (ms < best_ms * 0.98f) { best_ms = ms; best = S; }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  gm.S = best;
  gm.units = best * gm.m_tiles * gm.n_tiles;
  return e;
}

static cudaError_t tune_splits(Batch& Bt, cudaStream_t s) {
  BatchArgs& g = Bt.g;
  // every node row live during the timing
  int h[8] = {0, 0, (int)g.B, (int)g.B, 0, 0, 0, 0};
  cudaError_t e = cudaMemcpyAsync(g.flags, h, sizeof(h), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  e = tune_one(Bt, Bt.gf, Bt.m_xh, Bt.m_xl, Bt.m_bh, Bt.m_bl, Bt.sf_cap, s);
  if (e != cudaSuccess) return e;
  e = tune_one(Bt, Bt.gt, Bt.m_xth, Bt.m_xtl, Bt.m_rh, Bt.m_rl, Bt.sct_cap, s);
  if (e != cudaSuccess) return e;
  g.sf_init = Bt.gf.S;
  g.sf = Bt.sparse ? Bt.gfs.S : Bt.gf.S;
  g.sct = Bt.gt.S;
  return cudaMemsetAsync(g.flags, 0, 4ull * 8, s);
}

extern "C" {

// operands (hi/lo splits) | stream-K partials and flags for up to 256 CTAs
static constexpr int kSkMaxCtas = 256;
uint64_t l0_tc_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  const int64_t ldk = (K + 31) / 32 * 32;
  return (uint64_t)(2 * (M + N) * ldk) * 4 + 1024 + 4ull * kSkMaxCtas * (kTcBN * kTcBM + 1) + 256 + 64;
}

static int32_t tc_gemm_abi(int f16, const void* d_A, int32_t a_dtype, int64_t M, int64_t K, int64_t lda,
                           const void* d_B, int32_t b_dtype, int64_t N, int64_t ldb, float* d_C, int64_t ldc,
                           int32_t splits, int32_t* h_splits_out, void* d_ws, uint64_t ws_bytes, void* stream) {
  if (!d_A || !d_B || !d_C || !d_ws) return set_error(L0_INVALID, "null argument");
  if (M < 1 || N < 1 || K < 1 || lda < K || ldb < K || ldc < M)
    return set_error(L0_INVALID, "bad GEMM shape");
  if (ws_bytes < l0_tc_gemm_workspace_bytes(M, N, K)) return set_error(L0_INVALID, "workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  // operand regions sized for fp32 rows of ldk (the fp16 rows of ldk16 fit in them)
  const int64_t ldk = (K + 31) / 32 * 32;
  const int64_t ldk16 = (K + 63) / 64 * 64;
  char* base = (char*)(((uintptr_t)d_ws + 255) & ~uintptr_t(255));
  float* ah = (float*)base;
  float* al = ah + M * ldk;
  float* bh = al + M * ldk;
  float* bl = bh + N * ldk;
  double sa = 1.0, sb = 1.0;
  if (f16) {
    // power-of-two scales from max |A|, max |B| (3xFP16, tc_gemm.cuh)
    unsigned* mx = (unsigned*)(bl + N * ldk + (int64_t)kSkMaxCtas * (kTcBN * kTcBM + 1));   // after the stream-K flags
    if (cudaMemsetAsync(mx, 0, 8, s) != cudaSuccess) return set_error(L0_CUDA, "memset failed");
    auto amax = [&](const void* src, int dt, int64_t rows, int64_t ld, unsigned* o) {
      if (dt == L0_F64) k_absmax<double><<<148, 256, 0, s>>>((const double*)src, rows, K, ld, o);
      else k_absmax<float><<<148, 256, 0, s>>>((const float*)src, rows, K, ld, o);
    };
    amax(d_A, a_dtype, M, lda, mx);
    amax(d_B, b_dtype, N, ldb, mx + 1);
    unsigned hb[2] = {0, 0};
    if (cudaMemcpyAsync(hb, mx, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
      return set_error(L0_CUDA, "operand maxima failed");
    float fa, fb;
    std::memcpy(&fa, &hb[0], 4);
    std::memcpy(&fb, &hb[1], 4);
    sa = std::ldexp(1.0, f16_exp(fa));
    sb = std::ldexp(1.0, f16_exp(fb));
  }
  auto split = [&](const void* src, int dt, int64_t rows, int64_t ld, float* h, float* l, double sc) {
    if (f16) {
      const int blocks = (int)std::min<int64_t>((rows * ldk16 + 255) / 256, 148 * 16);
      if (dt == L0_F64)
        k_split_rows_h<double><<<blocks, 256, 0, s>>>((const double*)src, rows, K, ld, sc, (__half*)h, (__half*)l, ldk16);
      else
        k_split_rows_h<float><<<blocks, 256, 0, s>>>((const float*)src, rows, K, ld, sc, (__half*)h, (__half*)l, ldk16);
      return;
    }
    const int blocks = (int)std::min<int64_t>((rows * ldk + 255) / 256, 148 * 16);
    if (dt == L0_F64)
      k_split_rows<double><<<blocks, 256, 0, s>>>((const double*)src, rows, K, ld, h, l, ldk);
    else
      k_split_rows<float><<<blocks, 256, 0, s>>>((const float*)src, rows, K, ld, h, l, ldk);
  };
  split(d_A, a_dtype, M, lda, ah, al, sa);
  split(d_B, b_dtype, N, ldb, bh, bl, sb);
  if (cudaGetLastError() != cudaSuccess) return set_error(L0_CUDA, "split kernel launch failed");
  const int64_t ld_op = f16 ? ldk16 : ldk;
  CUtensorMap m_ah, m_al, m_bh, m_bl;
  if (tc_make_map(&m_ah, ah, M, K, ld_op, kTcBM, f16) || tc_make_map(&m_al, al, M, K, ld_op, kTcBM, f16) ||
      tc_make_map(&m_bh, bh, N, K, ld_op, kTcBN, f16) || tc_make_map(&m_bl, bl, N, K, ld_op, kTcBN, f16))
    return set_error(L0_CUDA, "cuTensorMapEncodeTiled failed");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  TcGemmArgs g{};
  g.M = M;
  g.N = N;
  g.K = K;
  g.ldc = ldc;
  g.c_split = N * ldc;
  g.C = d_C;
  g.n_active = nullptr;
  g.f16 = f16;
  g.a_inv_scale = (float)(1.0 / (sa * sb));
  tc_gemm_plan(g, sms, splits > 0 ? splits : 32);
  if (splits > 0) {
    g.S = splits;
    g.units = g.S * g.m_tiles * g.n_tiles;
  } else if (splits < 0) {   // stream-K: one output, partials only for tiles that straddle CTAs
    sms = std::min(sms, kSkMaxCtas);
    g.S = 1;
    g.units = g.m_tiles * g.n_tiles;
    g.streamk = 1;
    g.sk_part = bl + N * ldk;
    g.sk_flag = (int*)(g.sk_part + (int64_t)kSkMaxCtas * kTcBN * kTcBM);
    if (cudaMemsetAsync(g.sk_flag, 0, 4ull * kSkMaxCtas, s) != cudaSuccess)
      return set_error(L0_CUDA, "memset failed");
  }
  if (h_splits_out) *h_splits_out = g.S;
  const int grid = std::min(g.units, sms);
  cudaError_t e = tc_gemm_launch(m_ah, m_al, m_bh, m_bl, g, grid, s);
  if (e != cudaSuccess) return set_error(L0_CUDA, std::string("tc_gemm: ") + cudaGetErrorString(e));
  return L0_OK;
}

int32_t l0_tc_gemm_3xtf32(const void* d_A, int32_t a_dtype, int64_t M, int64_t K, int64_t lda,
                          const void* d_B, int32_t b_dtype, int64_t N, int64_t ldb, float* d_C,
                          int64_t ldc, int32_t splits, int32_t* h_splits_out, void* d_ws,
                          uint64_t ws_bytes, void* stream) {
  return tc_gemm_abi(0, d_A, a_dtype, M, K, lda, d_B, b_dtype, N, ldb, d_C, ldc, splits, h_splits_out, d_ws,
                     ws_bytes, stream);
}

int32_t l0_tc_gemm_3xf16(const void* d_A, int32_t a_dtype, int64_t M, int64_t K, int64_t lda,
                         const void* d_B, int32_t b_dtype, int64_t N, int64_t ldb, float* d_C,
                         int64_t ldc, int32_t splits, int32_t* h_splits_out, void* d_ws,
                         uint64_t ws_bytes, void* stream) {
  return tc_gemm_abi(1, d_A, a_dtype, M, K, lda, d_B, b_dtype, N, ldb, d_C, ldc, splits, h_splits_out, d_ws,
                     ws_bytes, stream);
}

int32_t l0_batch_create(const l0_problem* prob, int64_t n_nodes, l0_batch** out) {
  if (!out || !prob) return set_error(L0_INVALID, "null argument");
  *out = nullptr;
  if (n_nodes < 1 || n_nodes > 65535) return set_error(L0_INVALID, "n_nodes must be in [1, 65535]");
  const EngineArgs& a = prob->a;
  if (a.p > kb_prox_capacity())
    return set_error(L0_UNSUPPORTED, "batched nodes support p <= 131072 (per-node window kernel)");
  if (a.n >= (int64_t)INT32_MAX || a.p >= (int64_t)INT32_MAX)
    return set_error(L0_INVALID, "n and p must fit the tensor-map coordinates");
  l0_batch* Bt = new l0_batch();
  Bt->prob = prob;
  Bt->n = a.n;
  Bt->p = a.p;
  Bt->B = n_nodes;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&Bt->sms, cudaDevAttrMultiProcessorCount, dev);
  BatchArgs& g = Bt->g;
  g.n = a.n;
  g.p = a.p;
  g.B = n_nodes;
  g.pv = (a.p + kK2Slab - 1) / kK2Slab * kK2Slab;   // slab arrays index slab * 256 + pos
  g.pp = g.pv;
  g.nn = (a.n + 31) / 32 * 32;
  g.loss = a.loss;
  g.y = a.y;
  g.fone_stride = g.pv;
  g.rblocks = (int)((a.n + kRowsPerBlock - 1) / kRowsPerBlock);
  g.S = (int)((a.p + kK2Slab - 1) / kK2Slab);
  // contraction plans: forward M = n, N = B, K = p; transpose M = p, N = 2B
  // (the zeta rows only on bound checks), K = n, split count planned for N = B
  TcGemmArgs& gf = Bt->gf;
  gf.M = a.n; gf.N = n_nodes; gf.K = a.p;
  gf.f16 = 1;
  tc_gemm_plan(gf, Bt->sms, 32);
  if (const char* e = getenv("L0_TC_SF")) {   // tuning override
    gf.S = std::max(1, atoi(e));
    gf.units = gf.S * gf.m_tiles * gf.n_tiles;
  }
  TcGemmArgs& gt = Bt->gt;
  gt.M = a.p; gt.N = n_nodes; gt.K = a.n;
  gt.f16 = 1;
  tc_gemm_plan(gt, Bt->sms, 32);
  if (const char* e = getenv("L0_TC_ST")) gt.S = std::max(1, atoi(e));
  gt.N = 2 * n_nodes;
  gt.n_tiles = (int)((gt.N + kTcBN - 1) / kTcBN);
  gt.units = gt.S * gt.m_tiles * gt.n_tiles;
  // stream-K (L0_TC_SK=1): one output per contraction from even (tile,
  // K-block) shares.  Measured on C4: no faster end to end (1.52 vs 1.47-1.52
  // ms per batched iteration) and each output is one fp32 TMEM accumulation
  // over all of K (5000 / 20000) instead of eight ~625-deep chunks summed in
  // fp64 by the consumers -- so the tuned split-K stays the default
  Bt->streamk = getenv("L0_TC_SK") ? atoi(getenv("L0_TC_SK")) : 0;
  if (Bt->streamk) {
    for (TcGemmArgs* t : {&gf, &gt}) {
      t->S = 1;
      t->units = t->m_tiles * t->n_tiles;
      t->streamk = 1;
    }
  }
  // support-compacted forward (K = the cached columns, read on the device):
  // ~8 fp16 K blocks per tile at steady state on C4, one split (measured: 1
  // split 0.958 ms per batched iteration, 2 splits 0.991, 3 splits 1.049 --
  // the partials' HBM round trip costs more than the wave quantisation)
  Bt->sparse = getenv("L0_SPARSE_FWD") ? atoi(getenv("L0_SPARSE_FWD")) : 1;
  TcGemmArgs& gfs = Bt->gfs;
  gfs = gf;
  gfs.S = getenv("L0_TC_SFS") ? std::max(1, atoi(getenv("L0_TC_SFS"))) : 1;
  gfs.units = gfs.S * gfs.m_tiles * gfs.n_tiles;
  gfs.streamk = 0;
  g.sf_init = gf.S;
  g.sf = Bt->sparse ? gfs.S : gf.S;
  g.sct = gt.S;
  // partial capacity for the measured split choice (l0_batch_set_workspace)
  Bt->sf_cap = std::max(gf.S, std::min(8, std::max(1, gf.kb_total / 8)));
  // the transpose keeps the model's split: timed alone more splits look
  // faster (C4: 9 vs 5), but kb_step's re-read of the extra partials costs
  // more than they save (end to end 1.565 vs 1.510 ms per batched iteration)
  Bt->sct_cap = gt.S;
  if (getenv("L0_TC_SF")) Bt->sf_cap = gf.S;
  if (getenv("L0_TC_ST")) Bt->sct_cap = gt.S;
  if (Bt->sparse) Bt->sf_cap = std::max(Bt->sf_cap, gfs.S);
  if (Bt->streamk) Bt->sf_cap = Bt->sct_cap = std::max(1, Bt->sparse ? gfs.S : 1);
  Bt->ws_bytes = batch_carve(*Bt, nullptr);
  cudaError_t e = cudaStreamCreateWithFlags(&Bt->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&Bt->ev_in, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&Bt->ev_chunk, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaMallocHost((void**)&Bt->h_flags, 8 * sizeof(int));
  if (e != cudaSuccess) {
    l0_batch_destroy(Bt);
    return set_error(L0_CUDA, cudaGetErrorString(e));
  }
  *out = Bt;
  return L0_OK;
}

int32_t l0_batch_workspace_bytes(const l0_batch* Bt, uint64_t* bytes) {
  if (!Bt || !bytes) return set_error(L0_INVALID, "null argument");
  *bytes = Bt->ws_bytes;
  return L0_OK;
}

int32_t l0_batch_set_workspace(l0_batch* Bt, void* d_ws, uint64_t bytes) {
  if (!Bt || !d_ws) return set_error(L0_INVALID, "null argument");
  if (bytes < Bt->ws_bytes) return set_error(L0_INVALID, "workspace too small");
  batch_destroy_graph(*Bt);
  Bt->ws = d_ws;
  char* base = (char*)(((uintptr_t)d_ws + 1023) & ~uintptr_t(1023));
  batch_carve(*Bt, base);
  BatchArgs& g = Bt->g;
  const EngineArgs& a = Bt->prob->a;
  cudaStream_t s = Bt->stream;
  const int64_t n = g.n, p = g.p;
  // X -> hi/lo 3xFP16 operands scaled by 2^sx (|X 2^sx| < 2^14), row-major
  // (forward) and transposed (transpose pass)
  const int blocks = (int)std::min<int64_t>((n * g.pp + 255) / 256, (int64_t)Bt->sms * 16);
  const dim3 tgrid((unsigned)((p + 31) / 32), (unsigned)((g.nn + 31) / 32));
  L0_B_TRY(cudaMemsetAsync(Bt->xmax, 0, 4, s));
  if (a.dtype == F64) k_absmax<double><<<Bt->sms * 4, 256, 0, s>>>((const double*)a.X, n, p, a.ld, Bt->xmax);
  else k_absmax<float><<<Bt->sms * 4, 256, 0, s>>>((const float*)a.X, n, p, a.ld, Bt->xmax);
  L0_B_TRY(cudaGetLastError());
  unsigned xm_bits = 0;
  L0_B_TRY(cudaMemcpyAsync(&xm_bits, Bt->xmax, 4, cudaMemcpyDeviceToHost, s));
  L0_B_TRY(cudaStreamSynchronize(s));
  float xm = 0.f;
  std::memcpy(&xm, &xm_bits, 4);
  if (!std::isfinite(xm)) return set_error(L0_INVALID, "X contains non-finite entries");
  const int sx = f16_exp((double)xm);
  g.xsc = std::ldexp(1.0, sx);
  if (a.dtype == F64) {
    k_split_rows_h<double><<<blocks, 256, 0, s>>>((const double*)a.X, n, p, a.ld, g.xsc, Bt->xh, Bt->xl, g.pp);
    k_split_transpose_h<double><<<tgrid, dim3(32, 8), 0, s>>>((const double*)a.X, n, p, a.ld, g.xsc, Bt->xth, Bt->xtl, g.nn);
  } else {
    k_split_rows_h<float><<<blocks, 256, 0, s>>>((const float*)a.X, n, p, a.ld, g.xsc, Bt->xh, Bt->xl, g.pp);
    k_split_transpose_h<float><<<tgrid, dim3(32, 8), 0, s>>>((const float*)a.X, n, p, a.ld, g.xsc, Bt->xth, Bt->xtl, g.nn);
  }
  L0_B_TRY(cudaGetLastError());
  L0_B_TRY(cudaMemsetAsync(g.rh, 0, 2ull * 2 * g.B * g.nn, s));
  L0_B_TRY(cudaMemsetAsync(g.rl, 0, 2ull * 2 * g.B * g.nn, s));
  L0_B_TRY(cudaMemsetAsync(g.rinv, 0, 4ull * 2 * g.B, s));
  L0_B_TRY(cudaMemsetAsync(g.binv, 0, 4ull * g.B, s));
  L0_B_TRY(cudaMemsetAsync(g.cnt, 0, 4ull * g.B, s));
  L0_B_TRY(cudaMemsetAsync(g.flags, 0, 4ull * 8, s));
  int rc = 0;
  rc |= tc_make_map(&Bt->m_xh, Bt->xh, n, p, g.pp, kTcBM, 1);
  rc |= tc_make_map(&Bt->m_xl, Bt->xl, n, p, g.pp, kTcBM, 1);
  rc |= tc_make_map(&Bt->m_xth, Bt->xth, p, n, g.nn, kTcBM, 1);
  rc |= tc_make_map(&Bt->m_xtl, Bt->xtl, p, n, g.nn, kTcBM, 1);
  rc |= tc_make_map(&Bt->m_bh, g.bh, g.B, p, g.pp, kTcBN, 1);
  rc |= tc_make_map(&Bt->m_bl, g.bl, g.B, p, g.pp, kTcBN, 1);
  rc |= tc_make_map(&Bt->m_rh, g.rh, 2 * g.B, n, g.nn, kTcBN, 1);
  rc |= tc_make_map(&Bt->m_rl, g.rl, 2 * g.B, n, g.nn, kTcBN, 1);
  if (Bt->sparse) {
    rc |= tc_make_map(&Bt->m_xuh, g.xuh, n, p, g.pp, kTcBM, 1);
    rc |= tc_make_map(&Bt->m_xul, g.xul, n, p, g.pp, kTcBM, 1);
    rc |= tc_make_map(&Bt->m_bsh, g.bsh, g.B, p, g.pp, kTcBN, 1);
    rc |= tc_make_map(&Bt->m_bsl, g.bsl, g.B, p, g.pp, kTcBN, 1);
    L0_B_TRY(cudaMemsetAsync(g.umask, 0, 4ull * g.pp, s));
    L0_B_TRY(cudaMemsetAsync(g.slot_of, 0xff, 4ull * g.pp, s));
    L0_B_TRY(cudaMemsetAsync(g.col_of, 0xff, 4ull * g.pp, s));
    L0_B_TRY(cudaMemsetAsync(g.uctl, 0, 4ull * 8, s));
    L0_B_TRY(cudaMemsetAsync(g.xuh, 0, 2ull * n * g.pp, s));
    L0_B_TRY(cudaMemsetAsync(g.xul, 0, 2ull * n * g.pp, s));
    L0_B_TRY(cudaMemsetAsync(g.bsh, 0, 2ull * g.B * g.pp, s));
    L0_B_TRY(cudaMemsetAsync(g.bsl, 0, 2ull * g.B * g.pp, s));
    TcGemmArgs& gfs = Bt->gfs;
    gfs.ldc = g.nn;
    gfs.c_split = g.B * g.nn;
    gfs.C = g.cf;
    gfs.n_active = g.flags + 3;
    gfs.k_active = g.uctl + 3;
    gfs.a_inv_scale = (float)(1.0 / g.xsc);
    gfs.b_inv_scale = g.binv;
  }
  if (rc) return set_error(L0_CUDA, "cuTensorMapEncodeTiled failed");
  TcGemmArgs& gf = Bt->gf;
  gf.ldc = g.nn;
  gf.c_split = g.B * g.nn;
  gf.C = g.cf;
  gf.n_active = g.flags + 3;
  gf.a_inv_scale = (float)(1.0 / g.xsc);
  gf.b_inv_scale = g.binv;
  TcGemmArgs& gt = Bt->gt;
  gt.ldc = g.pp;
  gt.c_split = 2 * g.B * g.pp;
  gt.C = g.ct;
  gt.n_active = g.flags + 2;
  gt.a_inv_scale = (float)(1.0 / g.xsc);
  gt.b_inv_scale = g.rinv;
  if (Bt->streamk) {
    for (TcGemmArgs* t : {&gf, &gt}) {
      t->sk_part = Bt->sk_part;
      t->sk_flag = Bt->sk_flag;
    }
    L0_B_TRY(cudaMemsetAsync(Bt->sk_flag, 0, 4ull * Bt->sms, s));
  } else {
    L0_B_TRY(tune_splits(*Bt, s));
  }
  L0_B_TRY(cudaStreamSynchronize(s));
  return L0_OK;
}

int32_t l0_batch_destroy(l0_batch* Bt) {
  if (!Bt) return L0_OK;
  batch_destroy_graph(*Bt);
  if (Bt->h_flags) cudaFreeHost(Bt->h_flags);
  if (Bt->ev_in) cudaEventDestroy(Bt->ev_in);
  if (Bt->ev_chunk) cudaEventDestroy(Bt->ev_chunk);
  if (Bt->stream) cudaStreamDestroy(Bt->stream);
  delete Bt;
  return L0_OK;
}

int32_t l0_batch_solve(l0_batch* Bt, int64_t k, double M, double lambda2, const l0_fista_opts* o,
                       const l0_node* nodes, const double* d_warm, const double* h_g0,
                       double* d_beta_out, l0_report* reps, void* stream) {
  if (!Bt || !o || !reps || !d_beta_out) return set_error(L0_INVALID, "null argument");
  if (!Bt->ws) return set_error(L0_INVALID, "batch has no workspace (l0_batch_set_workspace)");
  BatchArgs& g = Bt->g;
  const int64_t p = g.p, B = g.B, pv = g.pv;
  const bool dbg = getenv("L0_DEBUG") != nullptr;
  auto tq = std::chrono::steady_clock::now();
  auto tick = [&](const char* what) {
    if (!dbg) return;
    auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "  batch_solve %-28s %8.3f ms\n", what, std::chrono::duration<double>(now - tq).count() * 1e3);
    tq = now;
  };
  std::memset(reps, 0, sizeof(l0_report) * (size_t)B);
  if (g.loss > SQUARED_HINGE) return set_error(L0_UNSUPPORTED, "bound-grade loss: the relaxation solver needs a solver-grade loss");
  if (!(k >= 1 && k <= p)) return set_error(L0_INVALID, "k must satisfy 1 <= k <= p");
  if (!(M > 0 && std::isfinite(M))) return set_error(L0_INVALID, "M must be a positive finite real");
  if (!(lambda2 > 0 && std::isfinite(lambda2))) return set_error(L0_INVALID, "lambda2 must be a positive finite real");
  if (!(o->gap_tolerance > 0)) return set_error(L0_INVALID, "gap_tolerance must be positive");
  if (o->bound_check_interval < 1) return set_error(L0_INVALID, "bound_check_interval must be >= 1");
  if (o->max_iterations < 1) return set_error(L0_INVALID, "max_iterations must be >= 1");
  if (std::isnan(o->lipschitz))   // fista.py:101: any other L is clamped to >= 1e-12
    return set_error(L0_INVALID, "lipschitz constant is NaN");
  // ---- per-node classes and parameters (model.py:119-149, perspective.py:36-73) ----
  // compact per-node index lists (fixed-one ascending, then fixed-zero); the
  // device expands them into the [B][pv] class rows (kb_fill_nodes) -- no
  // B x p host arrays to build and upload per solve
  std::vector<int64_t> off((size_t)B + 1, 0);
  std::vector<int> idx;
  std::vector<uint8_t> cls;
  std::vector<Params> prm((size_t)B);
  std::vector<uint8_t> seen((size_t)p, 0);
  for (int64_t b = 0; b < B; ++b) {
    const l0_node* nd = nodes ? &nodes[b] : nullptr;
    int64_t n1 = 0, n0 = 0;
    double parent = -INFINITY;
    const size_t first = idx.size();
    if (nd) {
      parent = nd->parent_bound;
      n1 = nd->n_fixed_one;
      n0 = nd->n_fixed_zero;
      int err = ST_OK;
      std::string msg;
      for (int64_t i = 0; i < n1 && !err; ++i) {
        const int64_t j = nd->h_fixed_one[i];
        if (j < 0 || j >= p) { err = L0_INVALID; msg = "fixed_one index out of range"; break; }
        if (seen[j]) { err = L0_INVALID; msg = "duplicate fixed index"; break; }
        seen[j] = 1;
        idx.push_back((int)j);
        cls.push_back((uint8_t)FIXED_ONE);
      }
      std::sort(idx.begin() + first, idx.end());
      for (int64_t i = 0; i < n0 && !err; ++i) {
        const int64_t j = nd->h_fixed_zero[i];
        if (j < 0 || j >= p) { err = L0_INVALID; msg = "fixed_zero index out of range"; break; }
        if (seen[j]) { err = L0_INVALID; msg = "fixed_one and fixed_zero must be disjoint"; break; }
        seen[j] = 1;
        idx.push_back((int)j);
        cls.push_back((uint8_t)FIXED_ZERO);
      }
      for (size_t e = first; e < idx.size(); ++e) seen[(size_t)idx[e]] = 0;
      if (err) return set_error(err, msg);
    }
    off[(size_t)b + 1] = (int64_t)idx.size();
    if (n1 > k) return set_error(L0_INFEASIBLE, "|fixed_one| exceeds the budget k (node " + std::to_string(b) + ")");
    const int64_t nfree = p - n1 - n0;
    Params& hp = prm[(size_t)b];
    hp = Params{};
    hp.L = std::max(o->lipschitz, 1e-12);   // fista.py:101
    hp.two_l2 = 2.0 * lambda2;              // fista.py:98
    hp.rho = hp.L / hp.two_l2;              // fista.py:102
    hp.M = M;
    hp.gap_tol = o->gap_tolerance;
    hp.gap_tol_rel = o->gap_tolerance_rel;
    hp.early_primal = o->early_primal_cutoff;
    hp.early_dual = o->early_dual_cutoff;
    hp.parent_bound = parent;
    hp.max_iter = o->max_iterations;
    hp.k = k;
    hp.k_g = k - n1;
    hp.k_rem = std::min(k - n1, nfree);
    hp.n_free = nfree;
    hp.n_fone = n1;
    hp.bci = o->bound_check_interval;
    hp.restart = o->restart ? 1 : 0;
    hp.stop_on_gap = o->stop_on_gap ? 1 : 0;
    hp.node_mode = (n1 + n0) > 0 ? 1 : 0;
    hp.loss = g.loss;
  }
  tick("host node lists + params");
  auto t0 = std::chrono::steady_clock::now();
  cudaStream_t user_s = (cudaStream_t)stream;
  cudaStream_t s = Bt->stream;
  L0_B_TRY(cudaEventRecord(Bt->ev_in, user_s));
  L0_B_TRY(cudaStreamWaitEvent(s, Bt->ev_in, 0));
  L0_B_TRY(cudaMemcpyAsync(g.prm, prm.data(), sizeof(Params) * B, cudaMemcpyHostToDevice, s));
  int64_t launches = 0;
  L0_B_TRY(cudaMemsetAsync(g.mask, (int)FREE, (size_t)(B * pv), s));
  if (!idx.empty()) {
    // the list rides in the (not yet used) candidate-index scratch: off | idx | cls
    char* lst = reinterpret_cast<char*>(g.cand_idx);
    const size_t ob = 8 * off.size(), ib = 4 * idx.size();
    if (ob + ib + cls.size() > 4ull * B * pv) return set_error(L0_INVALID, "node lists exceed the scratch");
    L0_B_TRY(cudaMemcpyAsync(lst, off.data(), ob, cudaMemcpyHostToDevice, s));
    L0_B_TRY(cudaMemcpyAsync(lst + ob, idx.data(), ib, cudaMemcpyHostToDevice, s));
    L0_B_TRY(cudaMemcpyAsync(lst + ob + ib, cls.data(), cls.size(), cudaMemcpyHostToDevice, s));
    kb_fill_nodes<<<(unsigned)B, 128, 0, s>>>(g, reinterpret_cast<const int64_t*>(lst),
                                              reinterpret_cast<const int*>(lst + ob),
                                              reinterpret_cast<const uint8_t*>(lst + ob + ib));
    L0_B_TRY(cudaGetLastError());
    ++launches;
  }
  double* d_g0 = nullptr;
  if (h_g0) {
    // g(beta_0) per node rides in the per-node gv scratch until the state init reads it
    d_g0 = g.gv;   // [B][3 pv + 8] doubles: the first B doubles are free at this point
    L0_B_TRY(cudaMemcpyAsync(d_g0, h_g0, 8ull * B, cudaMemcpyHostToDevice, s));
  } else if (d_warm) {
    if (k > kCandCap)
      return set_error(L0_UNSUPPORTED, "warm starts with k > 2048 need g(beta_0) per node (h_g0)");
    // g(beta_0) of every warm start on the device (kb_g0: one CTA per node)
    d_g0 = g.gv;
    kb_g0<<<(unsigned)B, 512, 0, s>>>(g, d_warm, d_g0);
    L0_B_TRY(cudaGetLastError());
    ++launches;
  }
  kb_state_init<<<(unsigned)((B + 127) / 128), 128, 0, s>>>(g, d_g0);
  ++launches;
  if (d_warm) {
    // warm starts (fista.py:130-137): beta_0 -> ring slots, split for u_0 = X beta_0
    kb_warm_scale<<<(unsigned)B, 256, 0, s>>>(g, d_warm);
    kb_warm<<<dim3((unsigned)std::min<int64_t>((g.pp + 255) / 256, 64), (unsigned)B), 256, 0, s>>>(g, d_warm);
    L0_B_TRY(cudaGetLastError());
    launches += 2;
  } else {
    // cold start: beta_0 = 0 (fista.py:130-137); u_0 = X beta_0 through the forward contraction
    L0_B_TRY(cudaMemsetAsync(g.beta, 0, 8ull * 3 * B * pv, s));
    L0_B_TRY(cudaMemsetAsync(g.bh, 0, 2ull * B * g.pp, s));
    L0_B_TRY(cudaMemsetAsync(g.bl, 0, 2ull * B * g.pp, s));
    L0_B_TRY(cudaMemsetAsync(g.binv, 0, 4ull * B, s));
  }
  Bt->gf.n_active = nullptr;
  L0_B_TRY(tc_gemm_launch(Bt->m_xh, Bt->m_xl, Bt->m_bh, Bt->m_bl, Bt->gf, std::min(Bt->gf.units, Bt->sms), s));
  Bt->gf.n_active = g.flags + 3;
  kb_obj<<<dim3((unsigned)g.rblocks, (unsigned)B), kRowThreads, 0, s>>>(g, MODE_INIT);
  L0_B_TRY(cudaGetLastError());
  launches += 2;
  tick("uploads + init launches");
  const int G = o->chunk_iterations > 0 ? std::min(o->chunk_iterations, 100) : 10;
  int rc = batch_build_graph(*Bt, G, o->profile ? 1 : 0);
  if (rc) return rc;
  tick("graph (cached or built)");
  int64_t chunks = 0;
  bool stop_sent = false;
  double prof_ms[3] = {0.0, 0.0, 0.0}, prof_gap[3] = {0.0, 0.0, 0.0};
  int64_t prof_n = 0, prof_gn = 0;
  for (;;) {
    L0_B_TRY(cudaGraphLaunch(Bt->exec, s));
    L0_B_TRY(cudaEventRecord(Bt->ev_chunk, s));
    L0_B_TRY(cudaEventSynchronize(Bt->ev_chunk));
    ++chunks;
    if (o->profile) {
      for (int i = 0; i < G; ++i) {
        float ms;
        for (int k2 = 0; k2 < 3; ++k2)
          if (cudaEventElapsedTime(&ms, Bt->ev[(size_t)i * 6 + 2 * k2], Bt->ev[(size_t)i * 6 + 2 * k2 + 1]) == cudaSuccess)
            prof_ms[k2] += ms;
        // gaps: transpose end -> prox begin, prox end -> forward begin, and
        // forward end -> next transpose begin (kb_obj, kb_compact, kb_rhs, kb_plan)
        if (cudaEventElapsedTime(&ms, Bt->ev[(size_t)i * 6 + 1], Bt->ev[(size_t)i * 6 + 2]) == cudaSuccess)
          prof_gap[0] += ms;
        if (cudaEventElapsedTime(&ms, Bt->ev[(size_t)i * 6 + 3], Bt->ev[(size_t)i * 6 + 4]) == cudaSuccess)
          prof_gap[1] += ms;
        if (i + 1 < G &&
            cudaEventElapsedTime(&ms, Bt->ev[(size_t)i * 6 + 5], Bt->ev[(size_t)(i + 1) * 6]) == cudaSuccess) {
          prof_gap[2] += ms;
          ++prof_gn;
        }
        ++prof_n;
      }
    }
    if (Bt->h_flags[4] >= B) break;
    const double elapsed = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (!stop_sent && elapsed > o->time_limit) {  // fista.py:204-206 (checked per chunk)
      kb_request_stop<<<(unsigned)((B + 127) / 128), 128, 0, s>>>(g, TERM_TIME_LIMIT);
      L0_B_TRY(cudaGetLastError());
      ++launches;
      stop_sent = true;
    }
  }
  launches += chunks * Bt->graph_kernels;
  tick("chunks (device)");
  if (o->profile && getenv("L0_DEBUG") && prof_n > 0)
    fprintf(stderr, "batch profile (ms per iteration): gemm_t %.4f | gap %.4f | prox %.4f | gap %.4f | gemm_f %.4f | "
            "obj+compact+rhs+plan %.4f\n", prof_ms[0] / prof_n, prof_gap[0] / prof_n, prof_ms[1] / prof_n,
            prof_gap[1] / prof_n, prof_ms[2] / prof_n, prof_gn ? prof_gap[2] / prof_gn : 0.0);
  // ---- reports and iterates ----------------------------------------------------
  // the report fields only (the states' probe stamps and trace rings are not read)
  std::vector<State> hs((size_t)B);
  L0_B_TRY(cudaMemcpy2DAsync(hs.data(), sizeof(State), g.st, sizeof(State), offsetof(State, probe), (size_t)B,
                             cudaMemcpyDeviceToHost, s));
  kb_gather_beta<<<dim3((unsigned)std::min<int64_t>((p + 255) / 256, 64), (unsigned)B), 256, 0, s>>>(g, d_beta_out);
  L0_B_TRY(cudaGetLastError());
  ++launches;
  cudaEvent_t ev_out;
  L0_B_TRY(cudaEventCreateWithFlags(&ev_out, cudaEventDisableTiming));
  cudaEventRecord(ev_out, s);
  cudaStreamWaitEvent(user_s, ev_out, 0);
  L0_B_TRY(cudaStreamSynchronize(s));
  cudaEventDestroy(ev_out);
  tick("state D2H + beta gather");
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  int first_err = ST_OK;
  int64_t err_node = -1;
  for (int64_t b = 0; b < B; ++b) {
    const State& h = hs[(size_t)b];
    l0_report& r = reps[b];
    r.primal_value = h.obj;
    r.dual_bound = h.best_dual;
    r.gap = h.gap;
    r.iterations = h.t;
    r.restarts = h.restarts;
    r.termination = h.termination;
    r.status = h.err;
    r.error_iteration = h.err_iter;
    r.wall_time = wall;
    r.gpu_launches = launches;
    r.topk_fallbacks = h.topk_fallbacks;
    r.prox_full_passes = h.slow_prox;
    // profile: contraction / prox times summed over the executed chunk iterations
    r.k2_ms = prof_ms[0];   // transpose contraction X^T [R | Z]
    r.k3_ms = prof_ms[1];   // slab epilogue + windowed prox
    r.k1_ms = prof_ms[2];   // forward contraction X (beta step)
    r.k1_count = r.k2_count = r.k3_count = prof_n;
    // a window tie overflow has no full-sort re-run in batched mode
    const int err = h.err == ST_TIE_OVERFLOW ? (int)ST_UNSUPPORTED : h.err;
    r.status = err;
    if (err != ST_OK && first_err == ST_OK) { first_err = err; err_node = b; }
  }
  if (first_err != ST_OK)
    return set_error(first_err, "node " + std::to_string(err_node) + " failed (status " +
                                    std::to_string(first_err) + " at iteration " +
                                    std::to_string(hs[(size_t)err_node].err_iter) + ")");
  return L0_OK;
}

}  // extern "C"
