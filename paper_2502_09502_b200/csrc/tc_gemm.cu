// tcgen05 split-K 3xTF32 GEMM (see tc_gemm.cuh for the contract).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>

#include "tc_gemm.cuh"

namespace l0 {

namespace {

constexpr int kTcStages = 2;
constexpr uint32_t kTileA = kTcBM * kTcBK * 4;             // 16 KB
constexpr uint32_t kTileB = kTcBN * kTcBK * 4;             // 32 KB
constexpr uint32_t kStageBytes = 2 * kTileA + 2 * kTileB;  // 96 KB
constexpr uint32_t kTmemCols = 2 * kTcBN;                  // double-buffered accumulator
constexpr size_t kTcSmem = (size_t)kTcStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;

__device__ __forceinline__ uint32_t sm_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_addr(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sm_addr(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(sm_addr(b)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          sm_addr(dst)),
      "l"(map), "r"(x), "r"(y), "r"(sm_addr(b))
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sm_addr(b))
               : "memory");
}
// K-major operand, 128-byte swizzle: 8-row atoms of 128 B, atoms 1024 B apart
__device__ __forceinline__ uint64_t kmajor_sw128_desc(const void* p) {
  const uint64_t start = (sm_addr(p) & 0x3FFFFu) >> 4;
  return start | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
        "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
        "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// A run of K blocks [kb0, kb1) of one output tile.  kind: 0 = the whole K
// range of a split-K unit or of a stream-K tile (written to C), 1 = a
// stream-K piece that does not start at K block 0 (fp32 partial to
// sk_part[cta], flagged), 2 = a stream-K piece starting at K block 0 of a
// tile that other CTAs finish (waits for their partials, adds, writes C).
struct Seg {
  int s, mt, nt, kb0, kb1, kind;
};
// stream-K: the steps (tile, K block), tiles in (m-tile, n-tile) order with n
// fastest, split into gridDim.x contiguous ranges
__device__ __forceinline__ int64_t sk_start(int64_t total, int c, int G) { return total * c / G; }

struct SegIter {
  const TcGemmArgs& g;
  int nt_live, units, kbt;
  int64_t step, end, total;   // stream-K
  int u;                      // split-K
  __device__ SegIter(const TcGemmArgs& g_, int ntl, int kbt_) : g(g_), nt_live(ntl), kbt(kbt_) {
    units = g.S * g.m_tiles * nt_live;
    total = (int64_t)g.m_tiles * nt_live * kbt;
    step = sk_start(total, blockIdx.x, gridDim.x);
    end = sk_start(total, blockIdx.x + 1, gridDim.x);
    u = blockIdx.x;
  }
  __device__ bool next(Seg& r) {
    if (g.streamk) {
      if (step >= end) return false;
      const int64_t tile = step / kbt;
      r.s = 0;
      r.nt = (int)(tile % nt_live);
      r.mt = (int)(tile / nt_live);
      r.kb0 = (int)(step - tile * kbt);
      r.kb1 = (int)min((int64_t)kbt, (int64_t)r.kb0 + (end - step));
      r.kind = r.kb0 > 0 ? 1 : (r.kb1 < kbt ? 2 : 0);
      step += r.kb1 - r.kb0;
      return true;
    }
    if (u >= units) return false;
    r.nt = u % nt_live;
    const int rest = u / nt_live;
    r.mt = rest % g.m_tiles;
    r.s = rest / g.m_tiles;
    r.kb0 = (int)(((int64_t)kbt * r.s) / g.S);
    r.kb1 = (int)(((int64_t)kbt * (r.s + 1)) / g.S);
    r.kind = 0;
    u += gridDim.x;
    return true;
  }
};

// instruction descriptors: D f32, both K-major, M = 128, N = kTcBN; A/B tf32
// (format 2, kind::tf32, K = 8 per MMA) or f16 (format 0, kind::f16, K = 16);
// either way one MMA consumes 32 bytes of each operand's 128-byte row
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kTcBN >> 3) << 17) |
                            ((uint32_t)(kTcBM >> 4) << 24);
constexpr uint32_t kIdescF16 = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(kTcBN >> 3) << 17) |
                               ((uint32_t)(kTcBM >> 4) << 24);
__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__global__ void __launch_bounds__(kTcThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap map_ah, const __grid_constant__ CUtensorMap map_al,
                   const __grid_constant__ CUtensorMap map_bh, const __grid_constant__ CUtensorMap map_bl,
                   TcGemmArgs g) {
  extern __shared__ unsigned char tc_smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kTcStages * kStageBytes);
  uint64_t* full = bars;                     // [kTcStages]
  uint64_t* empty = bars + kTcStages;        // [kTcStages]
  uint64_t* tfull = bars + 2 * kTcStages;    // [2]
  uint64_t* tempty = bars + 2 * kTcStages + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kTcStages + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_act = g.n_active ? (int64_t)*g.n_active : g.N;
  const int nt_live = (int)min((int64_t)g.n_tiles, (n_act + kTcBN - 1) / kTcBN);
  const int bke = g.f16 ? 64 : kTcBK;   // K elements per 128-byte block
  const int kbt = g.k_active ? (int)min((int64_t)g.kb_total, ((int64_t)*g.k_active + bke - 1) / bke)
                             : g.kb_total;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_ah) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_al) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_bh) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_bl) : "memory");
    for (int i = 0; i < kTcStages; ++i) {
      bar_init(&full[i], 1);
      bar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      bar_init(&tfull[i], 1);
      bar_init(&tempty[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sm_addr(tmem_slot)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===== TMA producer =====
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      SegIter it(g, nt_live, kbt);
      Seg w;
      while (it.next(w)) {
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          bar_wait(&empty[stage], phase ^ 1u);
          unsigned char* st = smem + stage * kStageBytes;
          bar_expect(&full[stage], kStageBytes);
          const int x = kb * bke;
          tma_load_2d(st, &map_ah, x, w.mt * kTcBM, &full[stage]);
          tma_load_2d(st + kTileA, &map_al, x, w.mt * kTcBM, &full[stage]);
          tma_load_2d(st + 2 * kTileA, &map_bh, x, w.nt * kTcBN, &full[stage]);
          tma_load_2d(st + 2 * kTileA + kTileB, &map_bl, x, w.nt * kTcBN, &full[stage]);
          if (++stage == kTcStages) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (one thread) =====
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int li = 0;
      SegIter it(g, nt_live, kbt);
      Seg w;
      while (it.next(w)) {
        const int acc = li & 1;
        bar_wait(&tempty[acc], ((li >> 1) & 1) ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * kTcBN);
        const int kb0 = w.kb0, kb1 = w.kb1;
        if (kb0 == kb1) {   // empty split-K unit (dynamic K): the epilogue writes zeros
          bar_arrive(&tfull[acc]);
          ++li;
          continue;
        }
        for (int kb = kb0; kb < kb1; ++kb) {
          bar_wait(&full[stage], phase);
          tc_fence_after();
          unsigned char* st = smem + stage * kStageBytes;
          const uint64_t ah = kmajor_sw128_desc(st), al = kmajor_sw128_desc(st + kTileA);
          const uint64_t bh = kmajor_sw128_desc(st + 2 * kTileA);
          const uint64_t bl = kmajor_sw128_desc(st + 2 * kTileA + kTileB);
          if (g.f16) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t o = (uint64_t)(2 * k);   // +32 bytes per K=16 step (>> 4)
              mma_f16(d, ah + o, bh + o, kIdescF16, (kb > kb0 || k > 0) ? 1u : 0u);
              mma_f16(d, ah + o, bl + o, kIdescF16, 1u);
              mma_f16(d, al + o, bh + o, kIdescF16, 1u);
            }
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t o = (uint64_t)(2 * k);   // +32 bytes per K=8 step (>> 4)
              mma_tf32(d, ah + o, bh + o, kIdesc, (kb > kb0 || k > 0) ? 1u : 0u);
              mma_tf32(d, ah + o, bl + o, kIdesc, 1u);
              mma_tf32(d, al + o, bh + o, kIdesc, 1u);
            }
          }
          tc_commit(&empty[stage]);
          if (++stage == kTcStages) { stage = 0; phase ^= 1u; }
        }
        tc_commit(&tfull[acc]);
        ++li;
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue: TMEM -> registers -> C (transposed, coalesced along m) =====
    const int q = warp & 3;
    const int et = threadIdx.x - 128;          // 0..127 over the four epilogue warps
    int li = 0;
    SegIter it(g, nt_live, kbt);
    Seg w;
    while (it.next(w)) {
      const int acc = li & 1;
      bar_wait(&tfull[acc], (li >> 1) & 1);
      tc_fence_after();
      const int64_t m = (int64_t)w.mt * kTcBM + q * 32 + lane;
      if (w.kind == 1) {
        // stream-K piece without K block 0: fp32 partial for the finishing CTA
        float* part = g.sk_part + (int64_t)blockIdx.x * kTcBN * kTcBM;
#pragma unroll 1
        for (int c = 0; c < kTcBN / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * kTcBN + c * 32), v);
#pragma unroll
          for (int j = 0; j < 32; ++j) part[(c * 32 + j) * kTcBM + q * 32 + lane] = __uint_as_float(v[j]);
        }
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (et == 0) asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(g.sk_flag + blockIdx.x), "r"(1) : "memory");
      } else {
        // CTAs holding the later K blocks of this tile (stream-K kind 2)
        int c_first = 0, c_last = -1;
        if (w.kind == 2) {
          const int64_t total = (int64_t)g.m_tiles * nt_live * kbt;
          const int64_t tile_end = ((int64_t)w.mt * nt_live + w.nt + 1) * kbt;
          c_first = blockIdx.x + 1;
          c_last = blockIdx.x;
          while (c_last + 1 < (int)gridDim.x && sk_start(total, c_last + 1, gridDim.x) < tile_end) ++c_last;
          if (et <= c_last - c_first) {
            int f = 0;
            while (!f) asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(f) : "l"(g.sk_flag + c_first + et) : "memory");
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
        }
        float* cbase = g.C + (int64_t)w.s * g.c_split;
        const bool empty_unit = w.kb0 == w.kb1;
#pragma unroll 1
        for (int c = 0; c < kTcBN / 32; ++c) {
          uint32_t v[32];
          if (!empty_unit) {
            tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * kTcBN + c * 32), v);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = 0u;
          }
          float f[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
          for (int cc = c_first; cc <= c_last; ++cc) {   // fixed CTA order
            const float* part = g.sk_part + (int64_t)cc * kTcBN * kTcBM;
#pragma unroll
            for (int j = 0; j < 32; ++j) f[j] += __ldcg(part + (c * 32 + j) * kTcBM + q * 32 + lane);
          }
          const int64_t r0 = (int64_t)w.nt * kTcBN + c * 32;
          if (m < g.M) {
            const float as = g.a_inv_scale;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              if (r0 + j < n_act) {
                const float sc = g.b_inv_scale ? as * __ldg(g.b_inv_scale + r0 + j) : as;
                cbase[(r0 + j) * g.ldc + m] = f[j] * sc;
              }
            }
          }
        }
        if (w.kind == 2) {
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (et <= c_last - c_first) g.sk_flag[c_first + et] = 0;   // consumed: clean for the next launch
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) bar_arrive(&tempty[acc]);
      ++li;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kTmemCols)
                 : "memory");
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

}  // namespace

int tc_make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t K, int64_t ld, int box_rows,
                int f16) {
  auto fn = encode_fn();
  if (!fn) return 1;
  const int es = f16 ? 2 : 4;
  if ((ld * es) % 16 != 0 || ((uintptr_t)base) % 16 != 0) return 2;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * es)};
  cuuint32_t box[2] = {(cuuint32_t)tc_bk(f16), (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                  const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : 3;
}

void tc_gemm_plan(TcGemmArgs& g, int sms, int max_splits) {
  g.m_tiles = (int)((g.M + kTcBM - 1) / kTcBM);
  g.n_tiles = (int)((g.N + kTcBN - 1) / kTcBN);
  g.kb_total = (int)((g.K + tc_bk(g.f16) - 1) / tc_bk(g.f16));
  const double t_kb = 0.85e-6;   // one K block (32 tf32 / 64 f16), 3 MMA groups
  const double part_bytes = 8.0 * (double)g.N * (double)g.M;   // write + read of one split
  int best = 1;
  double best_t = 1e30;
  for (int S = 1; S <= std::max(1, max_splits); ++S) {
    if (S > 1 && g.kb_total / S < 4) break;
    const int64_t units = (int64_t)S * g.m_tiles * g.n_tiles;
    const double waves = std::ceil((double)units / sms);
    const double t = waves * std::ceil((double)g.kb_total / S) * t_kb + S * part_bytes / 6.0e12;
    if (t < best_t * 0.98) { best_t = t; best = S; }
  }
  g.S = best;
  g.units = g.S * g.m_tiles * g.n_tiles;
}

cudaError_t tc_gemm_launch(const CUtensorMap& ah, const CUtensorMap& al, const CUtensorMap& bh,
                           const CUtensorMap& bl, const TcGemmArgs& g, int grid, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  tc_gemm_kernel<<<grid, kTcThreads, kTcSmem, s>>>(ah, al, bh, bl, g);
  return cudaGetLastError();
}

}  // namespace l0
