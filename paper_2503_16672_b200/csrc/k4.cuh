// K4 -- feature-wise (transposed) split of a token-wise compressed [n, h]
// matrix, as one warp-sized unit of work (16 features x 128 tokens), run by
// the standalone grid k_feature_split (any layout, optional drop counts; the
// hot path's paired-layout split is the leaner k4x.cuh).
//
// The unit: lane l owns the token group 4l..4l+3 of the 128-token block and
//   1. loads its 4 tokens' compressed 16-feature slices (16 B each) and their
//      metadata halfwords, expanding them with byte permutes into packed bf16
//      pairs X[token][feature pair];
//   2. runs the feature-wise top-2 over the 4 tokens two features at a time in
//      the 16-bit halves of 32-bit registers (native bf16x2 compares, ties to
//      the lower token, NaN ranked last; kept <=> beats two of the other three,
//      a bitwise majority);
//   3. writes sparse features as (v0, v1) pairs + nibbles (coalesced 128 B per
//      warp per feature, metadata halfwords assembled with 2 shuffles) and
//      dense features as their 4 token values (256 B per warp per feature).
// (ref: apply_mask -> column gather -> sparsify_feature_wise, splitgemm.py:72-80,
//  sparse24.py:96-115)
#pragma once
#include <cuda_bf16.h>
#include "meta.cuh"

namespace s24 {

struct K4Args {
  const __nv_bfloat16* vals;  // token-wise compressed [n, h/2]
  const uint8_t* meta;        // its hw metadata
  int n, h;
  const int* feat_pos;        // plan: rank in sparse list, or -(rank in dense)-1
  __nv_bfloat16* vs;          // [pad128(n_sparse), n/2]; nullptr = dense-only
  uint8_t* es;                // hw metadata of vs (rows = sparse rank, K = n)
  __nv_bfloat16* vd;          // [pad128(n_dense), n]
  unsigned long long* stats;  // += nonzeros before/after over sparse features (WITH_STATS)
  int nonneg;                 // 1: values are >= 0 and NaN-free (relu^2): rank raw values
  int pair_rows;              // >= 0: "paired" layout (below); -1: dense features go to vd
};
// Paired layout (pair_rows = 2 * n_dense): vs rows [0, pair_rows) hold each
// dense feature r as two 2:4 rows 2r, 2r+1 -- tokens 4j, 4j+1 (selector
// nibble 0x4) and 4j+2, 4j+3 (0xE) of every group -- and the sparse feature
// of rank s sits at row pair_rows + s. One 2:4 GEMM over all rows then
// computes both parts; its epilogue adds each pair (exact dense dot product,
// summed in two halves), so the split weight gradient needs no dense GEMM.

__device__ __forceinline__ void k4_warp_add(unsigned long long v, unsigned long long* dst) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

// per-warp copy of the nibble -> PRMT selector table (static shared memory)
__device__ __forceinline__ const uint2* k4_lut_init() {
  __shared__ uint2 lut[16][16];
  const uint32_t warp = (threadIdx.x >> 5) & 15u, lane = threadIdx.x & 31u;
  if (lane < 16) {
    const uint32_t i0 = lane & 3u, i1 = lane >> 2;
    uint32_t sel[4];
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q) sel[q] = (q == i0) ? 0x10u : (q == i1) ? 0x32u : 0x44u;
    lut[warp][lane] = make_uint2(sel[0] | (sel[1] << 8), sel[2] | (sel[3] << 8));
  }
  __syncwarp();
  return lut[warp];
}

// bf16x2 magnitude keys, NaN mapped below zero (-1.0); ordered with native
// bf16 compares (HSET2), which keeps the selection at one instruction per pair
__device__ __forceinline__ uint32_t k4_key2(uint32_t x) {
  const uint32_t mag = x & 0x7FFF7FFFu;
  const __nv_bfloat162 m = *reinterpret_cast<const __nv_bfloat162*>(&mag);
  const uint32_t nan = __hneu2_mask(m, m);  // (unordered: true exactly for NaN)
  return (mag & ~nan) | (0xBF80BF80u & nan);
}

__device__ __forceinline__ uint32_t k4_ge(uint32_t a, uint32_t b) {
  return __hge2_mask(*reinterpret_cast<const __nv_bfloat162*>(&a), *reinterpret_cast<const __nv_bfloat162*>(&b));
}

__device__ __forceinline__ uint32_t k4_nz(uint32_t x) {  // 1 per nonzero half, packed
  const uint32_t mag = x & 0x7FFF7FFFu;
  const __nv_bfloat162 z = __floats2bfloat162_rn(0.f, 0.f);
  // (unordered: NaN counts as a nonzero, numpy's count_nonzero)
  return __hneu2_mask(*reinterpret_cast<const __nv_bfloat162*>(&mag), z) & 0x00010001u;
}

__device__ __forceinline__ uint32_t k4_sel(uint32_t m, uint32_t a, uint32_t b) { return (a & m) | (b & ~m); }

// majority of three bitwise masks
__device__ __forceinline__ uint32_t k4_maj(uint32_t a, uint32_t b, uint32_t c) { return (a & b) | (a & c) | (b & c); }

// NONNEG: the operand is relu^2 (>= 0, never NaN), so the raw bf16 values
// order correctly under HSET2 and the magnitude/NaN keys are skipped
template <bool WITH_STATS, bool NONNEG = false>
__device__ __forceinline__ void k4_warp_unit(const K4Args& a, int t0, int fbase, int lane, const uint2* sel_lut) {
  const __nv_bfloat16* __restrict__ vals = a.vals;
  const uint8_t* __restrict__ meta_hw = a.meta;
  const int n = a.n, h = a.h;
  const int* __restrict__ feat_pos = a.feat_pos;
  __nv_bfloat16* __restrict__ vs = a.vs;
  uint8_t* __restrict__ es = a.es;
  __nv_bfloat16* __restrict__ vd = a.vd;
  unsigned long long* stats = a.stats;
  const int t = t0 + 4 * lane;
  // per-feature output bases, computed once by lanes 0..15 (feature fbase+lane)
  // and broadcast with shuffles:
  //   sparse (pos >= 0): ofs = word offset of the feature's vs row at token t0,
  //                      mb  = byte offset of its metadata halfword for q = 0
  //   dense  (pos <  0): ofs = 0x80000000 | uint2 offset of its vd row at t0,
  //                      or (paired) 0x40000000 | word offset of its first vs
  //                      row, mb as for sparse; lanes 16..31 hold the second
  //                      row's mb of feature fbase + lane - 16
  const int paired = a.pair_rows;
  const int my_pos = feat_pos[fbase + (lane & 15)];
  if (vs == nullptr && !__any_sync(0xffffffffu, lane < 16 && my_pos < 0)) return;  // dense-only: no dense here
  uint32_t my_ofs = 0, my_mb = 0;
  if (my_pos >= 0) {
    const uint32_t row = static_cast<uint32_t>(my_pos + (paired > 0 ? paired : 0));
    my_ofs = row * static_cast<uint32_t>(n / 4) + static_cast<uint32_t>(t0 / 4);
    my_mb = static_cast<uint32_t>(meta_hw_halfword_offset(row, t0 / 16, n));
  } else if (paired >= 0) {
    const uint32_t row = 2u * static_cast<uint32_t>(-my_pos - 1) + (lane >= 16 ? 1u : 0u);
    my_ofs = 0x40000000u | ((row & ~1u) * static_cast<uint32_t>(n / 4) + static_cast<uint32_t>(t0 / 4));
    my_mb = static_cast<uint32_t>(meta_hw_halfword_offset(row, t0 / 16, n));
  } else {
    my_ofs = 0x80000000u | (static_cast<uint32_t>(-my_pos - 1) * static_cast<uint32_t>(n / 4) +
                            static_cast<uint32_t>(t0 / 4));
  }
  // this lane's in-atom offset of column chunk q = lane/4 (q = 0 is folded into my_mb)
  const uint32_t qd = static_cast<uint32_t>(lane) >> 2;
  const uint32_t q_off = 4u * (qd >> 1) + 128u * (qd & 1u);

  // 1. load + expand: X[r][k] = bf16 pair of features (2k, 2k+1) for token t+r
  uint32_t X[4][8];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint4 v = *reinterpret_cast<const uint4*>(vals + static_cast<long long>(t + r) * (h / 2) + fbase / 2);
    const uint32_t m16 = *reinterpret_cast<const uint16_t*>(meta_hw + meta_hw_halfword_offset(t + r, fbase / 16, h));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const uint2 sl = sel_lut[(m16 >> (4 * g)) & 0xFu];
      X[r][2 * g] = __byte_perm(w[g], 0u, sl.x);
      X[r][2 * g + 1] = __byte_perm(w[g], 0u, sl.y);
    }
  }
  uint32_t* vs32 = reinterpret_cast<uint32_t*>(vs);
  uint2* vd64 = reinterpret_cast<uint2*>(vd);
  uint32_t cnt_b = 0, cnt_a = 0;  // per-half nonzero counters (sparse features only)

#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t x0 = X[0][k], x1 = X[1][k], x2 = X[2][k], x3 = X[3][k];
    const uint32_t ofs0 = __shfl_sync(0xffffffffu, my_ofs, 2 * k), ofs1 = __shfl_sync(0xffffffffu, my_ofs, 2 * k + 1);
    const bool sp0 = !(ofs0 & 0xC0000000u), sp1 = !(ofs1 & 0xC0000000u);
    if (paired >= 0) {
      // dense features as two fixed-selector 2:4 rows: (x0, x1) | 0x4, (x2, x3) | 0xE
      const uint32_t nw = static_cast<uint32_t>(n / 4);
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const uint32_t ofs = f ? ofs1 : ofs0;
        if (ofs & 0x40000000u) {
          const uint32_t o = ofs & 0x3FFFFFFFu;
          const uint32_t sel_a = f ? 0x7632u : 0x5410u;
          vs32[o + lane] = __byte_perm(x0, x1, sel_a);
          vs32[o + nw + lane] = __byte_perm(x2, x3, sel_a);
        }
      }
      // selector halfwords: every lane takes part in the shuffles, then lanes
      // with lane % 4 == 0 store one halfword per row and token quad
      const uint32_t mba0 = __shfl_sync(0xffffffffu, my_mb, 2 * k), mbb0 = __shfl_sync(0xffffffffu, my_mb, 16 + 2 * k);
      const uint32_t mba1 = __shfl_sync(0xffffffffu, my_mb, 2 * k + 1),
                     mbb1 = __shfl_sync(0xffffffffu, my_mb, 17 + 2 * k);
      if ((lane & 3) == 0) {
        if (ofs0 & 0x40000000u) {
          *reinterpret_cast<uint16_t*>(es + mba0 + q_off) = 0x4444;
          *reinterpret_cast<uint16_t*>(es + mbb0 + q_off) = 0xEEEE;
        }
        if (ofs1 & 0x40000000u) {
          *reinterpret_cast<uint16_t*>(es + mba1 + q_off) = 0x4444;
          *reinterpret_cast<uint16_t*>(es + mbb1 + q_off) = 0xEEEE;
        }
      }
    }
    if (vs != nullptr && (sp0 || sp1)) {
      uint32_t k0 = x0, k1 = x1, k2 = x2, k3 = x3;
      if constexpr (!NONNEG) {
        k0 = k4_key2(x0);
        k1 = k4_key2(x1);
        k2 = k4_key2(x2);
        k3 = k4_key2(x3);
      }
      // token i beats token j (i < j) iff key_i >= key_j: ties go to the lower token
      const uint32_t b01 = k4_ge(k0, k1), b02 = k4_ge(k0, k2), b03 = k4_ge(k0, k3);
      const uint32_t b12 = k4_ge(k1, k2), b13 = k4_ge(k1, k3), b23 = k4_ge(k2, k3);
      // kept <=> beats at least two of the other three
      const uint32_t K0 = k4_maj(b01, b02, b03), K1 = k4_maj(~b01, b12, b13);
      const uint32_t K2 = k4_maj(~b02, ~b12, b23), K3 = k4_maj(~b03, ~b13, ~b23);
      const uint32_t v0 = k4_sel(K0, x0, k4_sel(K1, x1, x2));  // first kept token
      const uint32_t v1 = k4_sel(K3, x3, k4_sel(K2, x2, x1));  // second kept token
      // selector nibble i0 | i1 << 2 of both features (16-bit halves) straight
      // from the keep masks: i0 = first kept (0, 1 or 2), i1 = last kept (1, 2 or 3)
      const uint32_t nib = ((~K0 & K1) & 0x00010001u) | ((~K0 & ~K1) & 0x00020002u) | ((K3 | ~K2) & 0x00040004u) |
                           ((K3 | K2) & 0x00080008u);
      // metadata halfwords of both features at once: 4 lanes (token groups) x 4 bits
      uint32_t hw = nib << (4 * (lane & 3));
      hw |= __shfl_xor_sync(0xffffffffu, hw, 1);
      hw |= __shfl_xor_sync(0xffffffffu, hw, 2);
      const uint32_t mb0 = __shfl_sync(0xffffffffu, my_mb, 2 * k), mb1 = __shfl_sync(0xffffffffu, my_mb, 2 * k + 1);
      if constexpr (WITH_STATS) {
        const uint32_t nzb = k4_nz(x0) + k4_nz(x1) + k4_nz(x2) + k4_nz(x3);
        const uint32_t nza = k4_nz(v0) + k4_nz(v1);
        if (sp0) {
          cnt_b += nzb & 0xFFFFu;
          cnt_a += nza & 0xFFFFu;
        }
        if (sp1) {
          cnt_b += nzb >> 16;
          cnt_a += nza >> 16;
        }
      }
      if (sp0) {
        vs32[ofs0 + lane] = __byte_perm(v0, v1, 0x5410);
        if ((lane & 3) == 0) *reinterpret_cast<uint16_t*>(es + mb0 + q_off) = static_cast<uint16_t>(hw);
      }
      if (sp1) {
        vs32[ofs1 + lane] = __byte_perm(v0, v1, 0x7632);
        if ((lane & 3) == 0) *reinterpret_cast<uint16_t*>(es + mb1 + q_off) = static_cast<uint16_t>(hw >> 16);
      }
    }
    if (ofs0 & 0x80000000u)
      vd64[(ofs0 & 0x7FFFFFFFu) + lane] = make_uint2(__byte_perm(x0, x1, 0x5410), __byte_perm(x2, x3, 0x5410));
    if (ofs1 & 0x80000000u)
      vd64[(ofs1 & 0x7FFFFFFFu) + lane] = make_uint2(__byte_perm(x0, x1, 0x7632), __byte_perm(x2, x3, 0x7632));
  }
  if constexpr (WITH_STATS) {
    k4_warp_add(cnt_b, stats);
    k4_warp_add(cnt_a, stats + 1);
  }
}

}  // namespace s24
