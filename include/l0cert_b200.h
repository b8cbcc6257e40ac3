/*
 * l0cert_b200.h — C ABI of the B200-native dual-bound engine.
 *
 * The reference (`l0cert`, pure Python) has no FFI of its own; its hot path is
 * the in-process API listed below.  Each entry point here is what a binding of
 * that API would call (ctypes from Python).  Reference
 * interfaces replaced, by /root/reference/pkg/src/l0cert file:line:
 *
 *   l0_fista_solve        fista.py:76-222   solve_relaxation (+ FistaOptions :43-61,
 *                                           RelaxationReport :64-73, Termination :35-40,
 *                                           NodeState model.py:119-149)
 *   l0_prox               prox.py:101-201   _prox_gstar_core / prox_gstar / prox_g /
 *                                           prox_gstar_node / prox_g_node
 *   l0_g_value            perspective.py:114-132   g_value
 *   l0_g_conjugate        perspective.py:143-159   g_conjugate
 *   l0_safe_lower_bound   perspective.py:162-190   safe_lower_bound
 *   l0_safe_lower_bound_batched  perspective.py:162-190, once per node of a
 *                                branch-and-bound batch (SPEC.md:330 bounding)
 *   l0_loss_value         model.py:159-181 / :208-218  loss_value, loss_gradient
 *   l0_loss_conjugate     model.py:226-280          loss_conjugate_at_neg
 *   l0_power_iteration    model.py:283-306          _power_iteration_lambda_max
 *   l0_standardize_stats / l0_standardize_apply  data.py:224-242  standardize
 *   l0_matvec/rmatvec     the numpy X @ v / X.T @ r call sites fista.py:141,156,162,165,209
 *
 * Conventions
 *   - Every pointer named d_* is DEVICE memory owned by the caller; h_* is host.
 *   - X is row-major (n rows, leading dimension ld >= p elements, ld*elem a
 *     multiple of 16 bytes, base 16-byte aligned, padding columns finite),
 *     dtype L0_F64 or L0_F32 (fp32 storage, fp64 arithmetic).  All vectors fp64.
 *   - `stream` is a cudaStream_t.  Calls are asynchronous unless they return a
 *     host value (h_*), in which case they synchronise the stream.
 *   - Return value: L0_OK or an l0_status; l0_last_error() describes the last
 *     failure of the calling thread.
 *   - Workspaces are caller-provided device buffers (size from the *_bytes
 *     queries); a workspace must not be shared by concurrent calls.
 */
#ifndef L0CERT_B200_H
#define L0CERT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum l0_status {
  L0_OK = 0,
  L0_INVALID = 1,      /* InvalidInputError (errors.py:8-10)          */
  L0_NUMERICAL = 2,    /* NumericalError (errors.py:18-24)             */
  L0_INFEASIBLE = 3,   /* InfeasibleNodeError (errors.py:27-29)        */
  L0_UNSUPPORTED = 4,  /* UnsupportedOperationError (errors.py:13-15) */
  L0_CUDA = 5,         /* CUDA runtime failure                          */
  L0_ABORTED = 6       /* the trace callback asked to stop              */
};
/* solver-grade losses 0..2; Poisson and gamma (model.py:174-177) are bound-grade:
 * l0_loss_value / l0_loss_conjugate / l0_safe_lower_bound accept them, the
 * solver rejects them with L0_UNSUPPORTED (no global Lipschitz constant) */
enum l0_loss { L0_SQUARED_ERROR = 0, L0_LOGISTIC = 1, L0_SQUARED_HINGE = 2, L0_POISSON = 3,
               L0_GAMMA = 4 };
enum l0_dtype { L0_F64 = 0, L0_F32 = 1 };
enum l0_termination {
  L0_CONVERGED = 0, L0_ITERATION_LIMIT = 1, L0_TIME_LIMIT = 2,
  L0_PRIMAL_BELOW_INCUMBENT = 3, L0_DUAL_ABOVE_INCUMBENT = 4
};
/* per-coordinate node class: free / fixed to one / fixed to zero */
enum l0_node_class { L0_FREE = 0, L0_FIXED_ONE = 1, L0_FIXED_ZERO = 2 };

typedef struct l0_problem l0_problem;

/* FistaOptions (fista.py:43-61) plus engine extensions. */
typedef struct l0_fista_opts {
  int64_t max_iterations;       /* fista.py:45 */
  double gap_tolerance;         /* fista.py:46, absolute */
  double time_limit;            /* fista.py:47, seconds (INFINITY: none) */
  double early_primal_cutoff;   /* fista.py:48, NaN = None */
  double early_dual_cutoff;     /* fista.py:49, NaN = None */
  int32_t bound_check_interval; /* fista.py:50 */
  int32_t restart;              /* fista.py:51 */
  double lipschitz;             /* fista.py:52; L = max(L, 1e-12) is applied (fista.py:101); NaN rejected */
  /* extensions */
  double gap_tolerance_rel;     /* also stop when gap <= rel * |primal| (0: off) */
  int32_t stop_on_gap;          /* 0: fixed-iteration mode (no gap stop) */
  int32_t chunk_iterations;     /* iterations per captured CUDA graph (0: auto) */
  int32_t profile;              /* 1: time the kernels with CUDA events (report fields) */
  int32_t engine_path;          /* 0 auto (single pass when X is beyond L2 and fits a <= 8-CTA
                                   cluster plan: from 128 MB for the one-vector kernels -- squared
                                   error, or another loss on fp32 X -- and from 512 MB with
                                   clusters of 4-8 otherwise; else two-pass), 1 two-pass,
                                   2 single pass */
  int32_t fp32_forward;         /* fp32 X, single pass: X beta with fp32 products and fp64
                                   reductions (the fp32 mode, 1e-5 relative); 0: fp64 products */
} l0_fista_opts;

/* NodeState (model.py:119-149): host index arrays, sorted unique, disjoint. */
typedef struct l0_node {
  const int64_t* h_fixed_one;
  int64_t n_fixed_one;
  const int64_t* h_fixed_zero;
  int64_t n_fixed_zero;
  double parent_bound;          /* model.py:132 (-INFINITY default) */
} l0_node;

/* RelaxationReport (fista.py:64-73) plus engine metrics. */
typedef struct l0_report {
  double primal_value;
  double dual_bound;
  double gap;
  int64_t iterations;
  int64_t restarts;
  int32_t termination;          /* l0_termination */
  int32_t status;               /* l0_status of the solve */
  int64_t error_iteration;      /* NumericalError.iteration (errors.py:22-24) */
  double wall_time;             /* fista.py:73 */
  int64_t gpu_launches;         /* kernels launched by the solve */
  int64_t topk_fallbacks;       /* envelope top-k window misses (diagnostic) */
  double k1_ms, k2_ms, k3_ms;   /* profile: summed kernel time (CUDA events); single-pass
                                   engine: k2 = the fused pass, k1 = reduce + epilogue */
  int64_t k1_count, k2_count, k3_count;
  int64_t prox_full_passes;     /* iterations whose prox window needed full key passes */
  int32_t single_pass;          /* 1: iterations read X once (fused kernel) */
  int32_t cluster_size;         /* CTAs per thread-block cluster of the fused kernel */
} l0_report;

typedef struct l0_trace_record {
  double iteration, primal, dual, gap, restarted;   /* fista.py:186-192 */
} l0_trace_record;

/* Called at every bound check, in order (fista.py:185-194).  A nonzero
 * return aborts the solve (the caller re-raises its own exception). */
typedef int (*l0_trace_cb)(const l0_trace_record* rec, void* user);

const char* l0_last_error(void);
int32_t l0_abi_version(void);

/* ---- problem (ProblemInstance minus k/M/lambda2, model.py:75-116) ---------- */
int32_t l0_problem_create(const void* d_X, int32_t dtype, int64_t n, int64_t p, int64_t ld,
                          const double* d_y, int32_t loss, l0_problem** out);
int32_t l0_problem_workspace_bytes(const l0_problem* prob, uint64_t* bytes);
int32_t l0_problem_set_workspace(l0_problem* prob, void* d_ws, uint64_t bytes);
int32_t l0_problem_destroy(l0_problem* prob);
/* Row-sharded mode: this rank's problem holds a contiguous block of rows of
 * the global X; every iteration all-reduces [X^T r | X^T zeta | F* terms] and
 * the loss over NCCL (h_nccl_unique_id: 128 bytes from l0_nccl_unique_id on
 * rank 0, broadcast by the caller).  nranks == 1 with a NULL id runs the
 * sharded kernels with the all-reduces elided (single-GPU test of that path). */
int32_t l0_problem_set_comm(l0_problem* prob, const void* h_nccl_unique_id, int32_t nranks,
                            int32_t rank);
int32_t l0_nccl_unique_id(void* h_out128);

/* diagnostics: clock64 phase stamps of the last prox kernel (L0_PROBE builds) */
int32_t l0_debug_probe(l0_problem* prob, int64_t* h_out16);
/* verification: record, for every iteration of later l0_fista_solve calls, the
 * prox's decisions into a device ring of cap records of (8 + width) int32:
 * [iteration, case (0 copy / 1 elementwise / 2 sort+PAVA), pool found,
 *  a*, c* (sorted positions of the merged PAVA pool), sorted prefix length,
 *  path (0 window, 1 window extended, 2 full key sort), free count]
 * then the first `width` coordinate ids of the stable descending order of
 * |rho gamma| over the free coordinates (-1 past the prefix).  Record of
 * iteration t sits at slot t % cap.  prox.py:111 (argsort) and :46-98 (pool).
 * d_ring = NULL turns recording off. */
int32_t l0_problem_set_prox_record(l0_problem* prob, int32_t* d_ring, int32_t cap, int32_t width);
/* diagnostics: copy the engine's p-length scratch vector (per-tile timestamps of
 * the single-pass kernel in L0_PROBE builds) */
int32_t l0_debug_scratch(l0_problem* prob, double* h_out, int64_t count);

/* ---- ingest ------------------------------------------------------------------
 * Copy `rows` rows of `row_bytes` from host memory (pitch h_pitch; pageable is
 * fine, e.g. a numpy array) to device rows of pitch d_pitch, through a ring of
 * pinned staging slots filled by `threads` host threads while the copy engine
 * drains the previous slot.  Synchronous (returns after the data is in HBM).
 * Replaces the host copy ProblemInstance makes of X (model.py:92) on the way
 * to the device. */
int32_t l0_upload_rows(void* d_dst, int64_t d_pitch, const void* h_src, int64_t h_pitch,
                       int64_t row_bytes, int64_t rows, int32_t threads, void* stream);

/* ---- hot path ----------------------------------------------------------------- */
int32_t l0_fista_solve(l0_problem* prob, int64_t k, double M, double lambda2,
                       const l0_fista_opts* opts, const l0_node* node /* nullable */,
                       const double* d_warm_start /* nullable, p */, double* d_beta_out /* p */,
                       l0_report* report, l0_trace_cb cb /* nullable */, void* user,
                       void* stream);

/* ---- operators ---------------------------------------------------------------- */
int32_t l0_matvec(l0_problem* prob, const double* d_v, double* d_out, void* stream);
int32_t l0_rmatvec(l0_problem* prob, const double* d_r, double* d_out, void* stream);
int32_t l0_power_iteration(l0_problem* prob, const double* d_v0, double tol, int64_t max_iter,
                           double* h_lambda, int64_t* h_iterations, void* stream);
int32_t l0_safe_lower_bound(l0_problem* prob, const double* d_beta, int64_t k_free, double M,
                            double lambda2, const uint8_t* d_node_class /* nullable */,
                            double* h_out, void* stream);
/* The same bound for nb nodes in one call (fp64 throughout): d_betas is nb x p
 * (node-major), h_k_free[j] the free budget of node j, d_node_class nb x p
 * (node-major, nullable: every coordinate free), h_out[nb] the bounds (-inf
 * where F*(-zeta) is +inf).  Each X tile is read once per pass for all nodes.
 * Workspace (device, caller-owned) from l0_safe_lower_bound_batched_workspace. */
int32_t l0_safe_lower_bound_batched_workspace(l0_problem* prob, int64_t nb, uint64_t* bytes);
int32_t l0_safe_lower_bound_batched(l0_problem* prob, const double* d_betas, int64_t nb,
                                    const int64_t* h_k_free, double M, double lambda2,
                                    const uint8_t* d_node_class /* nullable */, double* h_out,
                                    void* d_ws, uint64_t ws_bytes, void* stream);

/* ---- instance ingest (data.py:224-242 standardize), bit-identical to numpy ---- */
/* d_X row-major fp64 (n x ld); per-column mean, centred norm and max |x| (p each) */
int32_t l0_standardize_stats(const double* d_X, int64_t n, int64_t p, int64_t ld, double* d_mean,
                             double* d_norm, double* d_scale, void* stream);
/* d_out (n x m, row-major) = (X[:, kept] - mean[kept]) / norm[kept] */
int32_t l0_standardize_apply(const double* d_X, int64_t n, int64_t ld, const int64_t* d_kept, int64_t m,
                             const double* d_mean, const double* d_norm, double* d_out, void* stream);

/* ---- branch and bound: batched exact ridge refits ---------
 * C supports of width s <= 48 (device int32, -1 = padding): d_beta (C x s) =
 * (X_S^T X_S + lambda2 I)^{-1} X_S^T y and d_obj (C) = |y - X_S b|^2 +
 * lambda2 |b|^2 (yty = y^T y), squared-error refits without the box. */
int32_t l0_refit_ridge(l0_problem* prob, const int32_t* d_supports, int64_t C, int32_t s, double lambda2,
                       double yty, double* d_beta, double* d_obj, void* stream);

int32_t l0_ops_workspace_bytes(int64_t len, uint64_t* bytes);
/* g_mode=0: out = prox_{rho g*}(in) (prox_gstar[_node]); g_mode=1: out =
 * prox_{g/rho}(in) = in - prox_{rho g*}(rho in)/rho (prox_g[_node]).  k is the
 * budget of the free coordinates.  perm/pool report the stable descending
 * sort and the merged PAVA pool [a*, c*] in sorted positions (-1: none). */
int32_t l0_prox(const double* d_in, int64_t p, double rho, int64_t k, double M,
                const uint8_t* d_node_class, int32_t g_mode, double* d_out,
                int32_t* d_perm_out, int64_t* h_pool_out, void* d_ws, uint64_t ws_bytes,
                void* stream);
int32_t l0_g_value(const double* d_beta, int64_t p, int64_t k_free, double M,
                   const uint8_t* d_node_class, const int32_t* d_fixed_one, int64_t n_fixed_one,
                   double* h_out, void* d_ws, uint64_t ws_bytes, void* stream);
int32_t l0_g_conjugate(const double* d_alpha, int64_t p, int64_t k_free, double M,
                       const uint8_t* d_node_class, double* h_out, void* d_ws, uint64_t ws_bytes,
                       void* stream);
/* prox=0: out = H_M(x) (prox.py:27-32); prox=1: out = hprox(x, w, M) (prox.py:35-43) */
int32_t l0_huber(const double* d_x, int64_t n, double w, double M, int32_t prox, double* d_out,
                 void* stream);
int32_t l0_loss_value(int32_t loss, const double* d_u, const double* d_y, int64_t n,
                      double* h_value, double* d_grad /* nullable */, int32_t* h_nonfinite,
                      void* d_ws, uint64_t ws_bytes, void* stream);
int32_t l0_loss_conjugate(int32_t loss, const double* d_zeta, const double* d_y, int64_t n,
                          double* h_out, void* d_ws, uint64_t ws_bytes, void* stream);
int32_t l0_all_finite(const void* d_x, int32_t dtype, int64_t rows, int64_t cols, int64_t ld,
                      int32_t* h_ok, void* d_ws, uint64_t ws_bytes, void* stream);

/* ---- batched node contraction (tcgen05 tensor cores) ----------------------
 * The batched engine's GEMM, exposed for verification: C_s = A B^T over K
 * split s (s = 0..S-1), A M x K (pitch lda), B N x K (pitch ldb), fp64 or fp32
 * inputs, computed as 3xTF32 (hi/lo TF32 operand split, fp32 accumulation in
 * TMEM).  C is S x N x ldc fp32 (ldc >= M; partial sums per split).  splits=0
 * lets the engine choose S (returned in *h_splits).  Replaces the numpy
 * X @ Gamma / X.T @ R products of a batch of node solves (fista.py:162, :165). */
/* Batched node relaxations on one shared X (the BnB caller's node batches,
 * SPEC.md:294-357; per node exactly l0_fista_solve / fista.py:76-222 with that
 * node's NodeState, cold start).  The two X passes of an iteration are tcgen05
 * contractions over all nodes in 3xTF32, so per-node results carry fp32-class
 * rounding (tolerance 1e-5 relative) whatever the problem's dtype.
 * l0_batch_set_workspace pre-splits X (and X^T) into TF32 hi/lo operands, so
 * X must not change while the batch exists.  Nodes advance in lockstep; a
 * finished node is frozen and leaves the contractions.  Warm starts (the
 * parent's beta, fista.py:130-137) come with g(beta_0) per node.  d_beta_out is n_nodes x p (row per node); reps
 * has n_nodes entries.  Trace callbacks are not available in batched mode. */
typedef struct l0_batch l0_batch;
int32_t l0_batch_create(const l0_problem* prob, int64_t n_nodes, l0_batch** out);
int32_t l0_batch_workspace_bytes(const l0_batch* batch, uint64_t* bytes);
int32_t l0_batch_set_workspace(l0_batch* batch, void* d_ws, uint64_t bytes);
int32_t l0_batch_solve(l0_batch* batch, int64_t k, double M, double lambda2,
                       const l0_fista_opts* opts, const l0_node* nodes /* n_nodes, nullable */,
                       const double* d_warm /* nullable, n_nodes x p warm starts */,
                       const double* h_g0 /* nullable: g(beta_0) per node; with d_warm and
                                             h_g0 NULL the engine evaluates it (kb_g0) */,
                       double* d_beta_out, l0_report* reps, void* stream);
int32_t l0_batch_destroy(l0_batch* batch);

/* C_s = A B^T in 3xTF32 on tcgen05 (the batched engine's contraction):
 * splits > 0: that many K splits (C holds S partials, S x N x ldc); 0: planned
 * split count; < 0: stream-K (one output C, N x ldc).  *h_splits gets S. */
uint64_t l0_tc_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K);
int32_t l0_tc_gemm_3xtf32(const void* d_A, int32_t a_dtype, int64_t M, int64_t K, int64_t lda,
                          const void* d_B, int32_t b_dtype, int64_t N, int64_t ldb, float* d_C,
                          int64_t ldc, int32_t splits, int32_t* h_splits, void* d_ws,
                          uint64_t ws_bytes, void* stream);
/* The same contraction in 3xFP16 (kind::f16, twice the TF32 tensor rate): A
 * and B scaled by powers of two below 2^14, split into fp16 hi + lo, three
 * products accumulated in fp32, C unscaled exactly (the batched engine's
 * contraction; tc_gemm.cuh).  Same arguments and workspace as above. */
int32_t l0_tc_gemm_3xf16(const void* d_A, int32_t a_dtype, int64_t M, int64_t K, int64_t lda,
                         const void* d_B, int32_t b_dtype, int64_t N, int64_t ldb, float* d_C,
                         int64_t ldc, int32_t splits, int32_t* h_splits, void* d_ws,
                         uint64_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* L0CERT_B200_H */
