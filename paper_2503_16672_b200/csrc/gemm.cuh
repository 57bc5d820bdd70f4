// Persistent, warp-specialised tcgen05 GEMM for sm_100a, dense or 2:4-sparse A.
//
//   D[M,N] = A[M,K] * B[K,N]      (bf16 or e4m3 operands, fp32 accumulation in TMEM)
//
// CG = 1: one CTA per tile of 128 x BN.
// CG = 2: a CTA pair (cluster of 2 on one TPC) per tile of 256 x BN, issued as
//         tcgen05.mma.cta_group::2 by the leader CTA: each CTA stages its own
//         128 rows of A and BN/2 columns of B; the pair's tensor cores read
//         both halves of B, halving smem operand traffic per SM.
// 128 + 32*EPI_WARPS threads per CTA:
//   warps 0..E-1 : epilogue (E = 4 or 8); warp w reads TMEM lanes
//              32*(w%4)..+31 (= tile rows); 8 warps split the columns in two
//              runs, chunk by chunk (32 fp32 columns) into the epilogue functor
//   warp E   : TMA producer (A/B tiles, 2:4 metadata atoms) into a ring of
//              STAGES smem slots
//   warp E+1 : MMA issuer (leader CTA, one thread): tcgen05.cp metadata
//              smem->TMEM, tcgen05.mma(.sp), tcgen05.commit
//   warp E+2 : TMEM allocator
// Work distribution: the grid holds one cluster per work unit (tile, or
// tile x K split, of one or two problems). Each cluster runs its own unit,
// then keeps stealing units of clusters that have not started yet through
// Blackwell's cluster launch control (clusterlaunchcontrol.try_cancel), so
// the kernel behaves as a persistent one (one cluster per CTA pair of SMs,
// units taken in launch order) with no device memory behind the scheduler:
// launches are independent of each other, of streams and of graph replays.
// The producer and MMA warps sit at the highest warp ids because the warp
// arbiter prefers higher ids: busy epilogue warps must not delay MMA issue.
// BN = 512 (dense, CTA pairs): each k-step issues two N = 256 MMAs (sub-tiles
//   s = 0, 1: CTA r stages B columns 256s + 128r .. +127 of the tile) into one
//   512-column accumulator. Per CTA a stage moves 16 KB of A and 32 KB of B
//   per 128 x 512 x 64 MACs, a quarter fewer bytes per MAC than BN = 256,
//   for the L2->SM operand feed that bounds these GEMMs. The accumulator is
//   single-buffered: the next tile's MMAs wait for the drain, while the
//   producer keeps filling stages.
// Accumulators: two TMEM slots. Disjoint (2*BN columns) when they fit, else
// overlapping by one 32-column chunk (slot 1 starts at BN-32): the epilogue
// drains the shared chunk first and releases the slot right away, so the next
// tile's MMAs overlap the rest of the drain while the 2:4 metadata keeps its
// own TMEM columns.
//
// Operand smem layouts (SWIZZLE_128B, exactly as TMA writes them):
//   K-major  : rows of 128 bytes (64 bf16 along K), 8-row groups 1024 B apart
//   MN-major : boxes of 64 (M or N) elements x BK rows of K, box stride BK*128 B
// Descriptors: K-major SBO = 1024; MN-major LBO = box stride, SBO = 1024.
#pragma once
#include "meta.cuh"
#include "ptx.cuh"

// Work distribution (see the header): S24_STATIC_SCHED = 1 (default) runs a
// persistent grid of the resident clusters, cluster c taking units c, c + C,
// c + 2C, ...; 0 launches one cluster per unit and lets running clusters
// steal the units of not-yet-started ones through cluster launch control.
// Both need no device memory. Measured (scripts/ab_step.py, c2 step): the
// pending clusters of a CLC launch keep the block scheduler from placing the
// side-stream K4 CTAs next to the running GEMM, which starves K4 and stalls
// the weight gradients that wait for it (1.95 vs 1.92 ms; K4 of act 688 vs
// 254 us while co-running, scripts/timeline.py).
#ifndef S24_STATIC_SCHED
#define S24_STATIC_SCHED 1
#endif
// S24_PROBE (experiments only): 1 = MMA issue without operand loads (stale
// shared memory), 2 = operand loads without MMAs, 3 = as 1 without the 2:4
// metadata copies into TMEM, 5 = the full kernel without those copies.
// Results are garbage.
#ifndef S24_PROBE
#define S24_PROBE 0
#endif
#ifndef S24_CLC_PREFETCH
#define S24_CLC_PREFETCH 1
#endif

namespace s24 {

struct GemmShape {
  int M, N, K;          // logical sizes (K = logical K for sparse A)
  int tiles_m, tiles_n; // in units of (128*CG) x BN
  int group_m;          // raster: group_m M-tiles share one sweep over N
  int k_splits;         // >1: split-K, work unit = (tile, K range); partials go to the epilogue with ks
  int groups;           // 1 or 2 problems of this shape (second: tmA2/tmB2/tmE2, ep2), group-major units
  int a_stream;         // 1: A panels are not re-read after their raster group (L2 evict-first)
  int b_keep;           // 1: B is small enough to pin in L2 (evict-last)
  int tail_split;       // the last tail_split tiles (in unit order) run as two N-halves each
                        // (MN-major B only): a partial last wave of full tiles becomes a
                        // half-length one (see unit_tile)
};

template <bool SPARSE_, bool A_MN_, bool B_MN_, int BN_, int STAGES_, int CG_, int EPI_WARPS_ = 8, bool F8_ = false>
struct GemmCfg {
  static constexpr bool SPARSE = SPARSE_;
  // F8: e4m3 operands (tcgen05 kind::f8f6f4). Every stage and MMA step moves
  // the same BYTES as the bf16 configuration (twice the K elements), so the
  // smem layouts and descriptor strides below are shared; the 2:4 metadata
  // doubles per stage (two atoms, see meta.cuh).
  static constexpr bool F8 = F8_;
  static constexpr int EB = F8 ? 1 : 2;          // bytes per operand element
  static constexpr bool A_MN = A_MN_;
  static constexpr bool B_MN = B_MN_;
  static constexpr int CG = CG_;
  static constexpr int BM = 128;                 // rows per CTA
  static constexpr int TILE_M = BM * CG;         // rows per tile
  static constexpr int BN = BN_;                 // columns per tile (MMA N)
  static constexpr int BN_CTA = BN / CG;         // B columns staged per CTA
  static constexpr int NSUB = BN > 256 ? BN / 256 : 1;  // MMAs per k-step (N = 256 each)
  static constexpr int MMA_N = BN / NSUB;
  static constexpr int SUB_CTA = BN_CTA / NSUB;  // B columns per CTA per sub-tile
  static constexpr int NSLOT = NSUB > 1 ? 1 : 2; // accumulator slots
  static constexpr int STAGES = STAGES_;
  static constexpr int BK = (SPARSE ? 128 : 64) * (2 / EB);  // logical K per stage
  static constexpr int A_COLS = 128 / EB;        // stored A elements per row per stage (128 bytes)
  static constexpr int BOX_K = 128 / EB;         // K elements per 128-byte swizzle row
  static constexpr int KSTEPS = 4;               // MMAs per stage (bf16: K16 dense / K32 sparse; e4m3: K32 / K64)
  static constexpr uint32_t A_BYTES = BM * 128;
  static constexpr uint32_t B_BYTES = BN_CTA * BK * EB;
  static constexpr int E_ATOMS = SPARSE ? (F8 ? 2 : 1) : 0;  // 2 KB metadata atoms per stage
  static constexpr uint32_t E_BYTES = 2048 * E_ATOMS;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES + E_BYTES;
  static constexpr uint32_t E_COLS = STAGES * 4 * E_ATOMS;
  static constexpr bool OVERLAP = NSLOT == 2 && 2 * BN + E_COLS > 512;
  static constexpr uint32_t SLOT1_COL = OVERLAP ? BN - 32 : BN;
  static constexpr uint32_t E_COL = NSLOT == 1 ? BN : SLOT1_COL + BN;
  static constexpr uint32_t TMEM_NEED = E_COL + E_COLS;
  static constexpr uint32_t TMEM_COLS = TMEM_NEED <= 32 ? 32 : TMEM_NEED <= 64 ? 64 : TMEM_NEED <= 128 ? 128
                                       : TMEM_NEED <= 256 ? 256 : 512;
  static_assert(TMEM_NEED <= 512, "TMEM budget");
  static_assert(!(SPARSE && A_MN), "sparse A must be K-major");
  static_assert(!(F8 && (A_MN || B_MN)), "e4m3 operands are K-major");
  static_assert(BN_CTA % 64 == 0 && (BN <= 256 || (BN == 512 && !SPARSE && CG == 2)), "BN");
  static_assert(CG == 1 || CG == 2, "CG");
  static constexpr uint32_t BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int SCHED_SLOTS = 4;  // work-unit ring (cluster launch control responses)
  // barriers: full/empty per stage, tfull/tempty per accumulator slot, the
  // TMEM base word (+pad), sched_full/sched_empty per ring slot, then the
  // 16-byte CLC responses (16-aligned: BAR_OFF is a multiple of 1024)
  static constexpr uint32_t RESP_OFF = BAR_OFF + (2 * STAGES + 4) * 8 + 8 + 2 * SCHED_SLOTS * 8;
  static constexpr uint32_t RESP_OFF16 = (RESP_OFF + 15) / 16 * 16;
  // the dynamic smem base is declared 1024-aligned (SWIZZLE_128B atoms), so no
  // alignment slack is reserved: 7 dense stages fit next to the static smem
  static constexpr uint32_t SMEM_BYTES = RESP_OFF16 + 16 * SCHED_SLOTS;
  static constexpr uint32_t IDESC =
      F8 ? make_idesc_e4m3(TILE_M, MMA_N, SPARSE) : make_idesc_bf16(TILE_M, MMA_N, A_MN, B_MN, SPARSE);
  // half-width units (GemmShape::tail_split): N = BN / 2
  static constexpr bool HALF_OK = B_MN && NSUB == 1 && BN_CTA % 128 == 0;
  static constexpr uint32_t IDESC_HALF =
      F8 ? make_idesc_e4m3(TILE_M, BN / 2, SPARSE) : make_idesc_bf16(TILE_M, BN / 2, A_MN, B_MN, SPARSE);
  static constexpr int NCHUNK = BN / 32;
  static constexpr int EPI_WARPS = EPI_WARPS_;            // 4 or 8 (two warps per TMEM lane quarter)
  static constexpr int EPI_THREADS = 32 * EPI_WARPS;
  static constexpr int THREADS = 128 + EPI_THREADS;
  static constexpr int CPW = NCHUNK / (EPI_WARPS / 4);  // chunks per epilogue warp
  static_assert(EPI_WARPS == 4 || EPI_WARPS == 8, "epilogue warps");
  // 4-epilogue-warp configs cap registers at 128/thread so that an
  // independent kernel (K4 on the side stream) can co-reside on the SM
  static constexpr int MIN_BLOCKS = EPI_WARPS == 4 ? 2 : 1;
  static constexpr int CLUSTER = CG;
  static constexpr int B_KBOX = BK / BOX_K;  // K-major B: 128-byte K boxes per stage
  static constexpr int B_BOX_ROWS = SUB_CTA;
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

template <int CG>
__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                         uint64_t pol) {
  if constexpr (CG == 2)
    tma_load_2d_cg2_hint(dst, map, bar, c0, c1, pol);
  else
    tma_load_2d_hint(dst, map, bar, c0, c1, pol);
}

// L2 policy of the operand loads. B (the weights / the other activation) is
// re-read by every tile row: evict-last when it fits comfortably in L2
// (shape.b_keep; a 64 MiB activation B thrashes instead). When one wave of clusters covers a
// whole raster group (shape.a_stream), the A panel of a tile row is consumed
// by the clusters sweeping that row's N tiles at about the same time and then
// never again: evict-first, so streaming A does not push B out of L2.

// Epilogue contract: each epilogue warp owns one TMEM lane quarter (32 tile
// rows) and a run of CPW consecutive 32-column chunks. Per chunk:
//   Epi::chunk(ep, st, row, row_ok, col0, ci, v[32], lane)   (all lanes call it)
// where ci is the chunk's index within the warp's run (0..CPW-1, columns
// col0..col0+31); Epi::prefetch(ep, st, row, row_ok, col_first, ks) once per
// tile before the accumulator wait (col_first = first column of the run, ks =
// the split-K index of the work unit), and
// Epi::finish(ep, st, lane) once at the end.
template <class Cfg, class Epi>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MIN_BLOCKS)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmE, const __grid_constant__ CUtensorMap tmA2,
                const __grid_constant__ CUtensorMap tmB2, const __grid_constant__ CUtensorMap tmE2,
                const GemmShape shape, const typename Epi::Params ep, const typename Epi::Params ep2) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
  constexpr int CG = Cfg::CG;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if ((smem_u32(smem_raw) & 1023u) != 0u) __trap();  // the layout below relies on it
  uint8_t* smem = smem_raw;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Cfg::BAR_OFF);
  uint64_t* empty_bar = full_bar + Cfg::STAGES;
  uint64_t* tfull_bar = empty_bar + Cfg::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  // work units after the first come from cluster launch control: the leader
  // CTA's producer asks the hardware to cancel a not-yet-started cluster of
  // this launch and takes over its unit. The 16-byte response lands in the
  // same ring slot of both CTAs of the pair (multicast), completing 16 bytes
  // on each CTA's sched_full; every consumer of both CTAs releases the slot on
  // the leader's sched_empty before it is reused.
  constexpr int NS = Cfg::SCHED_SLOTS;
  uint64_t* sched_full = reinterpret_cast<uint64_t*>(tmem_slot + 2);
  uint64_t* sched_empty = sched_full + NS;
  uint8_t* sched_resp = smem + Cfg::RESP_OFF16;

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  // roles: epilogue warps first, the latency-critical producer / MMA warps get
  // the highest ids (the warp arbiter prefers higher ids)
  constexpr int W_PROD = Cfg::EPI_WARPS, W_MMA = W_PROD + 1, W_ALLOC = W_PROD + 2;
  const uint32_t rank = CG > 1 ? cluster_ctarank() : 0u;  // rank within the CTA pair
  const bool leader = rank == 0;
  const int first_unit = static_cast<int>(blockIdx.x) / Cfg::CLUSTER;
  const int mn_tiles = shape.tiles_m * shape.tiles_n;
  const int group_units = mn_tiles * shape.k_splits;
  const int total_tiles = group_units * shape.groups;
  const int tail_split = Cfg::HALF_OK ? shape.tail_split : 0;
  const int total_units = total_tiles + tail_split;
  // scheduler unit u -> tile unit t (and which N-half, or -1 for the whole tile)
  auto unit_tile = [&](int u, int& half) -> int {
    const int full = total_tiles - tail_split;
    if (u < full) {
      half = -1;
      return u;
    }
    half = (u - full) & 1;
    return full + ((u - full) >> 1);
  };
  const int num_kb_all = (shape.K + Cfg::BK - 1) / Cfg::BK;
  // work unit t -> (problem t / group_units; within it: output tile
  // t % mn_tiles, K split t / mn_tiles)
  auto kb_range = [&](int t, int& kb0, int& kb1) {
    const int ks = (t % group_units) / mn_tiles;
    kb0 = static_cast<int>(static_cast<long long>(ks) * num_kb_all / shape.k_splits);
    kb1 = static_cast<int>(static_cast<long long>(ks + 1) * num_kb_all / shape.k_splits);
  };

  if (warp == W_PROD && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if constexpr (Cfg::SPARSE) tma_prefetch(&tmE);
    if (shape.groups > 1) {
      tma_prefetch(&tmA2);
      tma_prefetch(&tmB2);
      if constexpr (Cfg::SPARSE) tma_prefetch(&tmE2);
    }
  }
  if (warp == W_MMA && lane == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full_bar[s], CG);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], CG * (Cfg::OVERLAP ? 128 : Cfg::EPI_THREADS));
    }
    for (int i = 0; i < NS; ++i) {
      mbar_init(&sched_full[i], 1);
      // leader MMA + leader epilogue warps (+ peer producer + peer epilogue warps)
      mbar_init(&sched_empty[i], 1 + Cfg::EPI_WARPS + (CG - 1) * (1 + Cfg::EPI_WARPS));
    }
    fence_barrier_init();
  }
  if (warp == W_ALLOC) {
    if constexpr (CG == 2)
      tmem_alloc_cg2<Cfg::TMEM_COLS>(tmem_slot);
    else
      tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (Cfg::CLUSTER > 1)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // unit of iteration iter >= 1 from ring slot (iter - 1) % NS
  auto resp_unit = [&](int slot) -> int {
    const int x = clc_query(sched_resp + 16 * slot);
    return x < 0 ? total_units : x / Cfg::CLUSTER;
  };
  // consumer side of the ring (all lanes of the calling warp, or a single
  // thread with one_thread): wait, read, release
  auto sched_take = [&](int iter, bool one_thread) -> int {
    if (S24_STATIC_SCHED || iter == 0) return first_unit + iter * static_cast<int>(gridDim.x / Cfg::CLUSTER);
    const int slot = (iter - 1) % NS;
    mbar_wait(&sched_full[slot], static_cast<uint32_t>((iter - 1) / NS) & 1u);
    const int t = resp_unit(slot);
    if (!one_thread) __syncwarp();
    if (one_thread || lane == 0) {
      if (leader)
        mbar_arrive(&sched_empty[slot]);
      else
        mbar_arrive_remote_release(&sched_empty[slot], 0);
    }
    return t;
  };

  if (warp == W_PROD) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t pol_a = shape.a_stream ? l2_policy_evict_first() : l2_policy_evict_normal();
      const uint64_t pol_b = shape.b_keep ? l2_policy_evict_last() : l2_policy_evict_normal();
      // the leader asks for unit iter + 1 as soon as unit iter is known to
      // exist, so the response latency hides under this tile's loads
      auto request = [&](int it) {
        const int slot = (it - 1) % NS;
        mbar_wait(&sched_empty[slot], (static_cast<uint32_t>((it - 1) / NS) & 1u) ^ 1u);
        mbar_arrive_expect_tx(&sched_full[slot], 16);
        if constexpr (CG == 2)
          clc_try_cancel_all(sched_resp + 16 * slot, &sched_full[slot]);
        else
          clc_try_cancel(sched_resp + 16 * slot, &sched_full[slot]);
      };
      for (int iter = 0;; ++iter) {
        int t;
        if (S24_STATIC_SCHED || iter == 0) {
          t = first_unit + iter * static_cast<int>(gridDim.x / Cfg::CLUSTER);
        } else if (leader) {
#if S24_CLC_PREFETCH == 0
          request(iter);
#endif
          const int slot = (iter - 1) % NS;
          mbar_wait(&sched_full[slot], static_cast<uint32_t>((iter - 1) / NS) & 1u);
          t = resp_unit(slot);  // (this thread reuses the slot only after NS more iterations)
        } else {
          mbar_arrive_expect_tx(&sched_full[(iter - 1) % NS], 16);
          t = sched_take(iter, true);
        }
#if S24_CLC_PREFETCH
        if (!S24_STATIC_SCHED && leader && t < total_units) request(iter + 1);
#endif
        if (t >= total_units) break;
        int half;
        t = unit_tile(t, half);
        int mb, nb, kb0, kb1;
        tile_coords(shape, t % mn_tiles, mb, nb);
        kb_range(t, kb0, kb1);
        const bool g2 = t >= group_units;
        const CUtensorMap* mapA = g2 ? &tmA2 : &tmA;
        const CUtensorMap* mapB = g2 ? &tmB2 : &tmB;
        const CUtensorMap* mapE = g2 ? &tmE2 : &tmE;
        const int m0 = mb * Cfg::TILE_M + static_cast<int>(rank) * Cfg::BM;
        // sub-tile s of this CTA: B columns n0 + s * MMA_N .. + SUB_CTA - 1
        const int n0 = nb * Cfg::BN + static_cast<int>(rank) * Cfg::SUB_CTA;
        // half unit: this CTA's B_CTA/2 columns of the half (box 0 .. BN_CTA/128 - 1)
        const int n0h = nb * Cfg::BN + half * (Cfg::BN / 2) + static_cast<int>(rank) * (Cfg::BN_CTA / 2);
        const uint32_t stage_tx = (S24_PROBE == 1 || S24_PROBE == 3) ? 0u : half < 0 ? Cfg::STAGE_BYTES : Cfg::STAGE_BYTES - Cfg::B_BYTES / 2;
        const int atom_row = mb * CG + static_cast<int>(rank);  // 128-row metadata block
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          if (leader)
            mbar_arrive_expect_tx(&full_bar[stage], CG * stage_tx);
          else
            mbar_arrive_remote(&full_bar[stage], 0);
          if (S24_PROBE == 1 || S24_PROBE == 3) {
            if (++stage == Cfg::STAGES) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          if constexpr (Cfg::A_MN) {
            tma_load<CG>(sa, mapA, &full_bar[stage], m0, kb * Cfg::BK, pol_a);
            tma_load<CG>(sa + Cfg::A_BYTES / 2, mapA, &full_bar[stage], m0 + 64, kb * Cfg::BK, pol_a);
          } else {
            tma_load<CG>(sa, mapA, &full_bar[stage], kb * Cfg::A_COLS, m0, pol_a);
          }
          if constexpr (Cfg::B_MN) {
#pragma unroll
            for (int j = 0; j < Cfg::BN_CTA / 64; ++j)
              if (half >= 0) {
                if (j < Cfg::BN_CTA / 128)
                  tma_load<CG>(sb + j * (Cfg::BK * 128), mapB, &full_bar[stage], n0h + 64 * j, kb * Cfg::BK, pol_b);
              } else {
                tma_load<CG>(sb + j * (Cfg::BK * 128), mapB, &full_bar[stage],
                             n0 + (j / (Cfg::SUB_CTA / 64)) * Cfg::MMA_N + 64 * (j % (Cfg::SUB_CTA / 64)),
                             kb * Cfg::BK, pol_b);
              }
          } else {
#pragma unroll
            for (int j = 0; j < Cfg::B_KBOX; ++j)
#pragma unroll
              for (int sub = 0; sub < Cfg::NSUB; ++sub)
                tma_load<CG>(sb + j * (Cfg::BN_CTA * 128) + sub * (Cfg::SUB_CTA * 128), mapB, &full_bar[stage],
                             kb * Cfg::BK + Cfg::BOX_K * j, n0 + sub * Cfg::MMA_N, pol_b);
          }
          if constexpr (Cfg::SPARSE)
            tma_load<CG>(sb + Cfg::B_BYTES, mapE, &full_bar[stage], 0,
                         (atom_row * ((shape.K + 127) / 128) + kb * Cfg::E_ATOMS) * 16, pol_a);
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == W_MMA) {
    // ------------------------------------------------------------ MMA issuer
    if (leader && lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int iter = 0;; ++iter) {
        const int u = sched_take(iter, true);
        if (u >= total_units) break;
        int half;
        const int t = unit_tile(u, half);
        const uint32_t idesc = half < 0 ? Cfg::IDESC : Cfg::IDESC_HALF;
        const int slot = iter % Cfg::NSLOT;
        if constexpr (Cfg::OVERLAP) {
          if (iter > 0) mbar_wait(&tempty_bar[0], (iter - 1) & 1);
        } else {
          mbar_wait(&tempty_bar[slot], ((iter / Cfg::NSLOT) & 1) ^ 1);
        }
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + slot * Cfg::SLOT1_COL;
        int kb0, kb1;
        kb_range(t, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * Cfg::STAGE_BYTES);
          const uint32_t sb = sa + Cfg::A_BYTES;
          uint32_t e_tmem = 0;
          if constexpr (Cfg::SPARSE) {
            e_tmem = tmem_base + Cfg::E_COL + stage * (4 * Cfg::E_ATOMS);
#pragma unroll
            for (int a = 0; a < Cfg::E_ATOMS; ++a) {
              if (S24_PROBE == 2 || S24_PROBE == 3 || S24_PROBE == 5) break;
              const uint64_t edesc = make_sdesc(sb + Cfg::B_BYTES + 2048 * a, 0, 128, kLayoutNone);
              if constexpr (CG == 2)
                tmem_cp_128x128b_cg2(e_tmem + 4 * a, edesc);
              else
                tmem_cp_128x128b(e_tmem + 4 * a, edesc);
            }
          }
#pragma unroll
          for (int j = 0; j < Cfg::KSTEPS; ++j)
#pragma unroll
          for (int sub = 0; sub < Cfg::NSUB; ++sub) {
            // (NSUB > 1: dense only; sub-tile sub's B boxes and accumulator columns)
            const uint32_t sbs = sb + sub * (Cfg::B_MN ? (Cfg::SUB_CTA / 64) * (Cfg::BK * 128) : Cfg::SUB_CTA * 128);
            const uint32_t d_sub = d_tmem + static_cast<uint32_t>(sub * Cfg::MMA_N);
            uint64_t adesc, bdesc;
            if constexpr (Cfg::A_MN) {
              adesc = make_sdesc(sa + j * 2048, Cfg::A_BYTES / 2, 1024, kLayoutSw128);
            } else {
              adesc = make_sdesc(sa + j * 32, 16, 1024, kLayoutSw128);
            }
            if constexpr (Cfg::B_MN) {
              // dense: 16 K rows per step; sparse: 32 K rows per step
              bdesc = make_sdesc(sbs + j * (Cfg::SPARSE ? 4096 : 2048), Cfg::BK * 128, 1024, kLayoutSw128);
            } else if constexpr (Cfg::SPARSE) {
              bdesc = make_sdesc(sb + (j >> 1) * (Cfg::BN_CTA * 128) + (j & 1) * 64, 16, 1024, kLayoutSw128);
            } else {
              bdesc = make_sdesc(sbs + j * 32, 16, 1024, kLayoutSw128);
            }
            const uint32_t accum = (kb > kb0 || j > 0) ? 1u : 0u;
            if (S24_PROBE == 2) continue;
            if constexpr (Cfg::SPARSE && Cfg::F8) {
              // e4m3: one K=64 step reads 64 metadata bits per row = TMEM
              // columns 2j, 2j+1 of the stage
              if constexpr (CG == 2)
                mma_sp_e4m3_cg2(d_tmem, adesc, bdesc, e_tmem + 2 * j, idesc, accum);
              else
                mma_sp_e4m3(d_tmem, adesc, bdesc, e_tmem + 2 * j, idesc, accum);
            } else if constexpr (Cfg::SPARSE) {
              // metadata address must be 2-column aligned; the odd column is
              // selected by the descriptor's sparse-id2 field (bits 0-1)
              const uint32_t id = idesc | static_cast<uint32_t>(j & 1);
              if constexpr (CG == 2)
                mma_sp_bf16_cg2(d_tmem, adesc, bdesc, e_tmem + (j & ~1), id, accum);
              else
                mma_sp_bf16(d_tmem, adesc, bdesc, e_tmem + (j & ~1), id, accum);
            } else if constexpr (Cfg::F8) {
              if constexpr (CG == 2)
                mma_e4m3_cg2(d_sub, adesc, bdesc, idesc, accum);
              else
                mma_e4m3(d_sub, adesc, bdesc, idesc, accum);
            } else {
              if constexpr (CG == 2)
                mma_bf16_cg2(d_sub, adesc, bdesc, idesc, accum);
              else
                mma_bf16(d_sub, adesc, bdesc, idesc, accum);
            }
          }
          uint64_t* tf = &tfull_bar[Cfg::OVERLAP ? 0 : slot];
          if constexpr (CG == 2) {
            mma_commit_cg2(&empty_bar[stage], static_cast<uint16_t>(0x3u));
            if (kb == kb1 - 1) mma_commit_cg2(tf, static_cast<uint16_t>(0x3u));
          } else {
            mma_commit(&empty_bar[stage]);
            if (kb == kb1 - 1) mma_commit(tf);
          }
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp < Cfg::EPI_WARPS) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;                 // TMEM lane quarter
    const int part = warp >> 2;             // which contiguous run of CPW chunks
    const int c_begin = part * Cfg::CPW;
    const bool owns_last = c_begin + Cfg::CPW == Cfg::NCHUNK;
    typename Epi::State st;
    Epi::init(ep, st);
    for (int iter = 0;; ++iter) {
      const int u = sched_take(iter, false);
      if (u >= total_units) break;
      int half;
      const int t = unit_tile(u, half);
      int mb, nb;
      tile_coords(shape, t % mn_tiles, mb, nb);
      // a half unit holds N = BN / 2 columns, starting at BN / 2 * half
      const int col_base = nb * Cfg::BN + (half > 0 ? Cfg::BN / 2 : 0);
      const int nck = half < 0 ? Cfg::NCHUNK : Cfg::NCHUNK / 2;
      const int slot = iter % Cfg::NSLOT;
      const int row = mb * Cfg::TILE_M + static_cast<int>(rank) * Cfg::BM + q * 32 + static_cast<int>(lane);
      const bool row_ok = row < shape.M;
      const typename Epi::Params& epg = t >= group_units ? ep2 : ep;
      Epi::prefetch(epg, st, row, row_ok, col_base + c_begin * 32, (t % group_units) / mn_tiles);
      uint64_t* tempty = &tempty_bar[Cfg::OVERLAP ? 0 : slot];
      // overlapping slots: the chunk shared with the other slot (last chunk of
      // slot 0, first of slot 1) gates the next tile's MMAs. Only the part that
      // owns it releases the accumulator (right after draining it). Ownership
      // alternates with the slot, so the owner of tile t+1 is the other part of
      // tile t: its release of t+1 also certifies it finished reading tile t,
      // whose slot the MMAs of tile t+2 overwrite.
      const bool owner = Cfg::OVERLAP && (slot == 0 ? owns_last : c_begin == 0);
      uint64_t* tfull = &tfull_bar[Cfg::OVERLAP ? 0 : slot];
      const uint32_t tparity = Cfg::OVERLAP ? (iter & 1) : ((iter / Cfg::NSLOT) & 1);
      mbar_wait(tfull, tparity);
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + slot * Cfg::SLOT1_COL;
      const bool rotate = Cfg::OVERLAP && slot == 0 && owns_last;
      // epilogues with per-chunk register state (Epi::kUnroll) get a fully
      // unrolled loop so that state is indexed statically
#pragma unroll(Epi::kUnroll ? Cfg::CPW : 1)
      for (int ci = 0; ci < Cfg::CPW; ++ci) {
        const int c = rotate ? (ci == 0 ? Cfg::NCHUNK - 1 : c_begin + ci - 1) : c_begin + ci;
        const int col0 = col_base + c * 32;
        const bool cvalid = c < nck && col0 < shape.N;  // uniform across the warp
        uint32_t r[32];
        if (cvalid) {
          tmem_ld32(t_row + c * 32, r);
          tmem_ld_wait();
        }
        // release the accumulator as soon as this warp's last load landed
        // (overlapping slots: the shared chunk's owner, after its first load)
        if (Cfg::OVERLAP ? (owner && ci == 0) : ci == Cfg::CPW - 1) {
          tc_fence_before();
          if (leader)
            mbar_arrive(tempty);
          else
            mbar_arrive_remote(tempty, 0);
        }
        if (cvalid) {
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
          Epi::chunk(epg, st, row, row_ok, col0, ci, v, lane);
        }
      }
    }
    Epi::finish(ep, st, lane);
  }

  tc_fence_before();
  if constexpr (Cfg::CLUSTER > 1)
    cluster_sync();
  else
    __syncthreads();
  if (warp == W_ALLOC) {
    tc_fence_after();
    if constexpr (CG == 2)
      tmem_dealloc_cg2<Cfg::TMEM_COLS>(tmem_base);
    else
      tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
  }
#endif
}

}  // namespace s24
