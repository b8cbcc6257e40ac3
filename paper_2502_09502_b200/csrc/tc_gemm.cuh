// tcgen05 (5th-gen tensor core) split-K GEMM for the batched node engine.
//
//   C_s[r][m] = sum_{k in split s} A[m][k] * B[r][k]          (s = 0..S-1)
//
// in "3xTF32": A = Ah + Al and B = Bh + Bl with Ah, Bh exactly representable
// in TF32 and Al, Bl the fp32 remainders, and
//   A B^T ~= Ah Bh^T + Ah Bl^T + Al Bh^T
// accumulated in fp32 in TMEM (relative error ~2^-21 per product instead of
// TF32's 2^-11).  Both operands are K-major fp32 in HBM, staged by TMA with
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
  const int* k_active;  // nullable: K extent actually used (<= K), read on device; the
                        // split-K units divide the live K blocks, empty units write zeros
  // stream-K mode (streamk = 1): one output C (S = 1), the (tile, K-block)
  // steps split evenly over the persistent CTAs; a tile that straddles CTAs
  // is finished by the CTA holding its first K block, which adds the other
  // CTAs' fp32 partials (sk_part[cta], flagged in sk_flag[cta]) in CTA order.
  int streamk;
  float* sk_part;       // [grid][kTcBN][kTcBM]
  int* sk_flag;         // [grid], zero between launches (the finishing CTA resets it)
};

// Host: tensor map for a K-major fp32 matrix (rows x K, row pitch ld elements)
// with a box of box_rows x 32 and the 128-byte swizzle.
int tc_make_map(CUtensorMap* map, const float* base, int64_t rows, int64_t K, int64_t ld,
                int box_rows);

// Launch C = A B^T in 3xTF32.  maps: Ah, Al (box 128 rows), Bh, Bl (box BN rows).
cudaError_t tc_gemm_launch(const CUtensorMap& ah, const CUtensorMap& al, const CUtensorMap& bh,
                           const CUtensorMap& bl, const TcGemmArgs& g, int grid, cudaStream_t s);

// Plan the split count / grid for an (M, N, K) problem on `sms` SMs.
void tc_gemm_plan(TcGemmArgs& g, int sms, int max_splits);

constexpr int kTcBN = 256;      // UMMA N (rows of B per tile)

}  // namespace l0
