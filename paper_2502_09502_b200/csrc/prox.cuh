// Shared-memory layouts and argument packs of the prox / envelope kernels.
#pragma once

#include <cub/block/block_scan.cuh>

#include "engine.cuh"

namespace l0 {

constexpr int kCandCap = 2048;  // top-k window / fallback list capacity

struct SelectSmem {
  unsigned hist[256];
  unsigned long long prefix, pmask;
  int64_t remaining;
};

struct ProxSmem {
  union {
    typename cub::BlockScan<double, 1024>::TempStorage scan;
    double gen[1024];
  } u;
  SelectSmem sel;
  double red[32];
  int found;
  int done;
  int ncand;
  int pad_;
  int64_t astar, cstar;
  double vstar;
  double gfree;
  int wvalid[32];
  int64_t wc[32];
  double wv[32];
  double cand[kCandCap];
  double cand2[kCandCap];
};

// Inputs of the post-sort stage (PAVA, scatter, envelope).
struct PostArgs {
  int64_t p;       // coordinates
  int64_t nf;      // free coordinates (sorted first)
  int64_t kk;      // prox budget over the free coordinates
  int64_t kg;      // envelope budget over the free coordinates
  double rho, M;
  const double* xs;
  const int* perm;
  double* tail;
  const double* in;   // gamma (gmode) or mu
  double* out;        // beta+ (gmode) or prox_gstar(mu)
  double* absb;       // |out| per sorted position (-1 for non-free)
  const uint8_t* mask;
  const int* fone;    // fixed-one ids for the envelope (nullptr: trivial node)
  int64_t n_fone;
  int gmode;          // 1: prox of g/rho via Moreau (fista.py:107); 0: prox of rho g*
  int want_g;         // also evaluate g(out) into *g_out
  double* g_out;
  State* st;          // diagnostics / error reporting (nullable)
  int* rec;           // K3 decision ring (EngineArgs::prox_rec; nullptr: off)
  int rec_cap, rec_w;
  int64_t rec_iter;
};

template <int T>
__device__ void prox_post_sort(const PostArgs& q, ProxSmem& sm);
__device__ int dual_step(const EngineArgs& a, ProxSmem& sm);
__device__ void block_kth_largest(const double* vals, int64_t m, int64_t kk, SelectSmem& sm,
                                  double* tau_out, int64_t* cnt_gt_out);
__device__ double block_topk_sum(const double* vals, int64_t m, int64_t kk, int64_t count,
                                 SelectSmem& sm, double* red);
__device__ double envelope_from_top(const double* top, int64_t kkg, double total);

}  // namespace l0
