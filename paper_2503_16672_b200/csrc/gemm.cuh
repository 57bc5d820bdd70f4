// Persistent, warp-specialised tcgen05 GEMM for sm_100a, dense or 2:4-sparse A.
//
//   D[M,N] = A[M,K] * B[K,N]      (bf16 operands, fp32 accumulation in TMEM)
//
// One CTA per SM (grid = min(#tiles, #SMs)), 256 threads:
//   warp 0  : TMA producer (A/B tiles via cp.async.bulk.tensor, 2:4 metadata
//             atoms via cp.async.bulk) into a STAGES-deep smem ring
//   warp 1  : MMA issuer (single thread): tcgen05.cp metadata smem->TMEM, then
//             tcgen05.mma(.sp) into one of NUM_ACC TMEM accumulators
//   warp 2  : TMEM allocator
//   warps 4-7: epilogue (TMEM -> registers -> fused epilogue functor -> HBM);
//             warp w owns TMEM lanes 32*(w%4) .. +31, i.e. tile rows.
// Tile = 128 x BN; K step per stage = 64 (dense) or 128 logical (sparse, i.e.
// 64 stored values per row + one 2048-byte metadata atom).
//
// Operand layouts (smem, SWIZZLE_128B, as TMA writes them):
//   K-major  : rows of 128 bytes (64 bf16 along K), 8-row groups 1024 B apart
//   MN-major : boxes of 64 (M or N) elements x BK rows of K, box stride BK*128 B
// Descriptors follow the canonical tcgen05 forms: K-major SBO = 1024;
// MN-major LBO = box stride, SBO = 1024 (8 K rows).
#pragma once
#include "meta.cuh"
#include "ptx.cuh"

namespace s24 {

struct GemmShape {
  int M, N, K;         // logical sizes (K = logical K for sparse A)
  int tiles_m, tiles_n;
  int group_m;         // tile rasterisation: group_m M-blocks share a B sweep
  const uint8_t* meta; // sparse only: hw-layout metadata, rows padded to 128
};

template <bool SPARSE_, bool A_MN_, bool B_MN_, int BN_, int STAGES_, int NUM_ACC_>
struct GemmCfg {
  static constexpr bool SPARSE = SPARSE_;
  static constexpr bool A_MN = A_MN_;
  static constexpr bool B_MN = B_MN_;
  static constexpr int BM = 128;
  static constexpr int BN = BN_;
  static constexpr int STAGES = STAGES_;
  static constexpr int NUM_ACC = NUM_ACC_;
  static constexpr int BK = SPARSE ? 128 : 64;       // logical K per stage
  static constexpr int A_COLS = SPARSE ? 64 : 64;    // stored A elements per row per stage
  static constexpr int KSTEPS = 4;                   // MMAs per stage (K16 dense / K32 sparse)
  static constexpr uint32_t A_BYTES = BM * A_COLS * 2;
  static constexpr uint32_t B_BYTES = BN * BK * 2;
  static constexpr uint32_t E_BYTES = SPARSE ? 2048 : 0;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES + E_BYTES;
  static constexpr uint32_t TMEM_E_COL = NUM_ACC * BN;
  static constexpr uint32_t TMEM_NEED = NUM_ACC * BN + (SPARSE ? STAGES * 4 : 0);
  static constexpr uint32_t TMEM_COLS = TMEM_NEED <= 32 ? 32 : TMEM_NEED <= 64 ? 64 : TMEM_NEED <= 128 ? 128
                                       : TMEM_NEED <= 256 ? 256 : 512;
  static_assert(TMEM_NEED <= 512, "TMEM budget");
  static_assert(!(SPARSE && A_MN), "sparse A must be K-major");
  static_assert(BN % 64 == 0 && BN <= 256, "BN");
  static constexpr uint32_t BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr uint32_t SMEM_BYTES = BAR_OFF + (2 * STAGES + 2 * NUM_ACC) * 8 + 16 + 1024;
  static constexpr uint32_t IDESC = make_idesc_bf16(BM, BN, A_MN, B_MN, SPARSE);
};

__device__ __forceinline__ void tile_coords(const GemmShape& s, int t, int& mb, int& nb) {
  const int group_tiles = s.group_m * s.tiles_n;
  const int g = t / group_tiles;
  const int first_m = g * s.group_m;
  const int gm = min(s.group_m, s.tiles_m - first_m);
  const int local = t - g * group_tiles;
  mb = first_m + local % gm;
  nb = local / gm;
}

// Epilogue contract: Epi::Params ep; per 32-column chunk of one row
//   Epi::chunk(ep, st, row, row_ok, col0, v[32], lane)   (all 32 lanes call it)
// and Epi::finish(ep, st, lane) once at the end (per-thread state reductions).
template <class Cfg, class Epi>
__global__ void __launch_bounds__(256, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const GemmShape shape, const typename Epi::Params ep) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Cfg::BAR_OFF);
  uint64_t* empty_bar = full_bar + Cfg::STAGES;
  uint64_t* tfull_bar = empty_bar + Cfg::STAGES;
  uint64_t* tempty_bar = tfull_bar + Cfg::NUM_ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + Cfg::NUM_ACC);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const int total_tiles = shape.tiles_m * shape.tiles_n;
  const int num_kb = (shape.K + Cfg::BK - 1) / Cfg::BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < Cfg::NUM_ACC; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 128);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(shape, t, mb, nb);
        const int m0 = mb * Cfg::BM, n0 = nb * Cfg::BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          mbar_arrive_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
          if constexpr (Cfg::A_MN) {
            // A stored [K][M]: two boxes of {64 M, 64 K}
            tma_load_2d(sa, &tmA, &full_bar[stage], m0, kb * Cfg::BK);
            tma_load_2d(sa + Cfg::A_BYTES / 2, &tmA, &full_bar[stage], m0 + 64, kb * Cfg::BK);
          } else {
            // A stored [M][Kstored]: one box {64, 128}
            tma_load_2d(sa, &tmA, &full_bar[stage], kb * Cfg::A_COLS, m0);
          }
          if constexpr (Cfg::B_MN) {
            // B stored [K][N]: BN/64 boxes of {64 N, BK K}
#pragma unroll
            for (int j = 0; j < Cfg::BN / 64; ++j)
              tma_load_2d(sb + j * (Cfg::BK * 128), &tmB, &full_bar[stage], n0 + 64 * j, kb * Cfg::BK);
          } else {
            // B stored [N][K]: BK/64 boxes of {64 K, BN rows}
#pragma unroll
            for (int j = 0; j < Cfg::BK / 64; ++j)
              tma_load_2d(sb + j * (Cfg::BN * 128), &tmB, &full_bar[stage], kb * Cfg::BK + 64 * j, n0);
          }
          if constexpr (Cfg::SPARSE) {
            const uint8_t* src = shape.meta + (static_cast<size_t>(mb) * num_kb + kb) * 2048u;
            bulk_load(sb + Cfg::B_BYTES, src, 2048u, &full_bar[stage]);
          }
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int iter = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++iter) {
        const int acc = iter % Cfg::NUM_ACC;
        const uint32_t acc_phase = (iter / Cfg::NUM_ACC) & 1;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * Cfg::BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * Cfg::STAGE_BYTES);
          const uint32_t sb = sa + Cfg::A_BYTES;
          uint32_t e_tmem = 0;
          if constexpr (Cfg::SPARSE) {
            e_tmem = tmem_base + Cfg::TMEM_E_COL + stage * 4;
            tmem_cp_128x128b(e_tmem, make_sdesc(sb + Cfg::B_BYTES, 0, 128, kLayoutNone));
          }
#pragma unroll
          for (int j = 0; j < Cfg::KSTEPS; ++j) {
            uint64_t adesc, bdesc;
            if constexpr (Cfg::A_MN) {
              adesc = make_sdesc(sa + j * 2048, Cfg::A_BYTES / 2, 1024, kLayoutSw128);
            } else {
              adesc = make_sdesc(sa + j * 32, 16, 1024, kLayoutSw128);
            }
            if constexpr (Cfg::B_MN) {
              // dense: 16 K rows per step; sparse: 32 K rows per step
              bdesc = make_sdesc(sb + j * (Cfg::SPARSE ? 4096 : 2048), Cfg::BK * 128, 1024, kLayoutSw128);
            } else if constexpr (Cfg::SPARSE) {
              bdesc = make_sdesc(sb + (j >> 1) * (Cfg::BN * 128) + (j & 1) * 64, 16, 1024, kLayoutSw128);
            } else {
              bdesc = make_sdesc(sb + j * 32, 16, 1024, kLayoutSw128);
            }
            const uint32_t accum = (kb > 0 || j > 0) ? 1u : 0u;
            if constexpr (Cfg::SPARSE) {
              // metadata address must be 2-column aligned; the odd column is
              // selected by the descriptor's sparse-id2 field (bits 0-1)
              mma_sp_bf16(d_tmem, adesc, bdesc, e_tmem + (j & ~1), Cfg::IDESC | static_cast<uint32_t>(j & 1),
                          accum);
            } else {
              mma_bf16(d_tmem, adesc, bdesc, Cfg::IDESC, accum);
            }
          }
          mma_commit(&empty_bar[stage]);
          if (kb == num_kb - 1) mma_commit(&tfull_bar[acc]);
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;  // TMEM lane quarter
    typename Epi::State st;
    Epi::init(ep, st);
    int iter = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++iter) {
      int mb, nb;
      tile_coords(shape, t, mb, nb);
      const int acc = iter % Cfg::NUM_ACC;
      const uint32_t acc_phase = (iter / Cfg::NUM_ACC) & 1;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row = mb * Cfg::BM + q * 32 + static_cast<int>(lane);
      const bool row_ok = row < shape.M;
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * Cfg::BN;
#pragma unroll 1
      for (int c = 0; c < Cfg::BN / 32; ++c) {
        const int col0 = nb * Cfg::BN + c * 32;
        if (col0 >= shape.N) break;  // uniform across the warp
        uint32_t r[32];
        tmem_ld32(t_row + c * 32, r);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        Epi::chunk(ep, st, row, row_ok, col0, v, lane);
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
    }
    Epi::finish(ep, st, lane);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
  }
#endif
}

}  // namespace s24
