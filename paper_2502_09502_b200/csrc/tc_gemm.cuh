// tcgen05 (5th-gen tensor core) split-K GEMM for the batched node engine.
//
//   C_s[r][m] = sum_{k in split s} A[m][k] * B[r][k]          (s = 0..S-1)
//
// as three products of split operands, A = Ah + Al and B = Bh + Bl:
//   A B^T ~= Ah Bh^T + Ah Bl^T + Al Bh^T
// accumulated in fp32 in TMEM.  Two operand kinds:
//   * 3xTF32 (kind::tf32, fp32 operands): Ah, Bh exactly representable in
//     TF32, Al, Bl the fp32 remainders; relative error ~2^-21 per product;
//   * 3xFP16 (kind::f16, fp16 operands, twice the tensor rate): the operands
//     pre-scaled by powers of two so that |A sa|, |B sb| < 2^14, hi the nearest
//     fp16 and lo the nearest fp16 of the remainder (~22 significant bits;
//     below |.| ~ 4 the remainder is an fp16 subnormal, an absolute error of
//     2^-25 against a scale of 2^14); the epilogue multiplies by 1 / (sa sb)
//     (per B row), exactly.  This is the batched engine's contraction.
// Both operands are K-major in HBM (128 bytes = 32 fp32 or 64 fp16 per
// swizzle row), staged by TMA with
// the 128-byte swizzle into a 2-stage shared-memory ring; one elected thread
// issues tcgen05.mma (M=128, N=BN, K=8) into a double-buffered TMEM
// accumulator; four epilogue warps drain TMEM with tcgen05.ld and store the
// fp32 split-K partial transposed ([r][m], coalesced along m).  Persistent
// CTAs walk (split, m-tile, n-tile) units, n fastest, so the n-tiles of one
// A block run back to back and A is read from HBM once -- or, in stream-K
// mode, an even share of the (tile, K-block) steps each, which keeps every SM
// busy without split-K partials of every tile in HBM.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace l0 {

constexpr int kTcBM = 128;      // UMMA M (rows of A per tile = TMEM lanes)
constexpr int kTcBK = 32;       // fp32 elements per 128-byte swizzle row
constexpr int kTcThreads = 256; // warp 0 TMA, warp 1 MMA + TMEM, warps 4..7 epilogue

struct TcGemmArgs {
  int64_t M, N, K;      // C is N x M per split
  int64_t ldc;          // row pitch of C (elements)
  int64_t c_split;      // elements between consecutive split partials
  float* C;
  int S;                // K splits
  int units;            // S * m_tiles * n_tiles
  int m_tiles, n_tiles;
  int kb_total;         // K blocks of kTcBK
  const int* n_active;  // nullable: rows of B actually needed (<= N), read on device
  const int* k_active = nullptr;  // nullable: K extent actually used (<= K), read on device; the
                        // split-K units divide the live K blocks, empty units write zeros
  // stream-K mode (streamk = 1): one output C (S = 1), the (tile, K-block)
  // steps split evenly over the persistent CTAs; a tile that straddles CTAs
  // is finished by the CTA holding its first K block, which adds the other
  // CTAs' fp32 partials (sk_part[cta], flagged in sk_flag[cta]) in CTA order.
  int streamk;
  float* sk_part;       // [grid][kTcBN][kTcBM]
  int* sk_flag;         // [grid], zero between launches (the finishing CTA resets it)
  int f16 = 0;          // 1: fp16 operands (kind::f16), K blocks of 64; 0: fp32 (kind::tf32), 32
  float a_inv_scale = 1.f;   // output factor 1 / sa (f16; 1 for tf32)
  const float* b_inv_scale = nullptr;   // nullable: output factor 1 / sb per B row (read on device)
};

// Host: tensor map for a K-major fp32 (f16 = 0) or fp16 (f16 = 1) matrix (rows
// x K, row pitch ld elements) with a box of box_rows x 128 bytes and the
// 128-byte swizzle.
int tc_make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t K, int64_t ld,
                int box_rows, int f16 = 0);
inline int tc_bk(int f16) { return f16 ? 64 : kTcBK; }   // K elements per block

// Launch C = A B^T in 3xTF32.  maps: Ah, Al (box 128 rows), Bh, Bl (box BN rows).
cudaError_t tc_gemm_launch(const CUtensorMap& ah, const CUtensorMap& al, const CUtensorMap& bh,
                           const CUtensorMap& bl, const TcGemmArgs& g, int grid, cudaStream_t s);

// Plan the split count / grid for an (M, N, K) problem on `sms` SMs (g.f16 set).
void tc_gemm_plan(TcGemmArgs& g, int sms, int max_splits);

constexpr int kTcBN = 256;      // UMMA N (rows of B per tile)

}  // namespace l0
