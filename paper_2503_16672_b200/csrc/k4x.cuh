// K4x -- the hot-path feature-wise split (rank order + paired dense rows,
// see k4.cuh) of a token-wise 2:4 operand: the activation (forward) or g_pre
// (backward) of the FFN step. The per-feature output offsets come from a
// small shared-memory table filled once per warp. Grid (h / (16 warps), n/128),
// warps x 16 features x 128 tokens.
#pragma once
#include <cuda_bf16.h>
#include "k4.cuh"
#include "meta.cuh"

namespace s24 {

struct K4xArgs {
  const __nv_bfloat16* vals;     // token-wise compressed [n, h/2]
  const uint8_t* meta;           // its hw metadata (rows = tokens, K = h)
  int n, h;
  const int* feat_pos;           // plan: rank in sparse list, or -(rank in dense)-1
  int pair_rows;                 // 2 * n_dense: rows of the dense pairs in front
  __nv_bfloat16* vs;             // [pad128(pair_rows + n_sparse), n/2]
  uint8_t* es;                   // hw metadata of vs
  // nullable: with NONNEG, a nonzero word here (K1's "a kept value is NaN"
  // flag, written before this launch) switches back to the NaN-aware keys
  const unsigned long long* nan_flag;
};

// NONNEG: the operand is relu^2 (>= 0): raw bf16 values order correctly under
// HSET2 and the magnitude / NaN keys are skipped, unless nan_flag is raised
// K4X_WARPS warps per CTA (16 features each) at <= 64 registers: several CTAs
// fit next to a running GEMM CTA, so the split runs on the side stream
// co-resident with the GEMMs
#ifndef S24_K4X_WARPS
#define S24_K4X_WARPS 4
#endif
constexpr int K4X_WARPS = S24_K4X_WARPS;

// Lane l of a warp unit owns tokens t = t0 + 4l .. +3 and the unit's 16
// features. Per feature the table holds its first operand row's word offset
// at this token block (bit 31: a dense feature, whose second row follows nw
// words later) and its metadata halfword offset for token quad 0 (the second
// row of a pair sits 16 bytes further: rows 2r, 2r + 1 differ only in m0).
// Every lane runs the same instruction stream: per feature pair one table
// read, the selection, a two-shuffle metadata merge and predicated stores.
template <bool NONNEG>
__global__ void __launch_bounds__(32 * K4X_WARPS, 32 / K4X_WARPS) k_feature_split_x(K4xArgs a) {
  __shared__ __align__(16) uint2 slots[K4X_WARPS][16];
  const uint2* lut = k4_lut_init();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = a.h;
  const bool keys = !NONNEG || (a.nan_flag != nullptr && __ldg(a.nan_flag) != 0ull);
  const int fbase = blockIdx.x * (16 * K4X_WARPS) + warp * 16;
  const int t0 = blockIdx.y * 128;
  const uint32_t nw = static_cast<uint32_t>(a.n / 4);
  if (lane < 16) {
    const int pos = __ldg(a.feat_pos + fbase + lane);
    const uint32_t row = pos >= 0 ? static_cast<uint32_t>(a.pair_rows + pos) : 2u * static_cast<uint32_t>(-pos - 1);
    slots[warp][lane] = make_uint2((row * nw + static_cast<uint32_t>(t0 / 4)) | (pos < 0 ? 0x80000000u : 0u),
                                   static_cast<uint32_t>(meta_hw_halfword_offset(row, t0 / 16, a.n)));
  }
  __syncwarp();
  const int t = t0 + 4 * lane;
  const uint32_t qd = static_cast<uint32_t>(lane) >> 2;
  const uint32_t q_off = 4u * (qd >> 1) + 128u * (qd & 1u);

  // load + expand: X[token][feature pair] packed bf16x2. The 4 tokens' metadata
  // halfwords are 16 bytes apart (same atom row group, m0 = t & 7 .. + 3) and
  // their 16-byte value slices h bytes apart.
  uint32_t X[4][8];
  const uint8_t* mp = a.meta + meta_hw_halfword_offset(t, fbase / 16, h);
  const uint4* vp = reinterpret_cast<const uint4*>(a.vals + static_cast<long long>(t) * (h / 2) + fbase / 2);
  const int vstep = h / 16;  // uint4 per token row
  uint32_t m16[4];
  uint4 v[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    m16[r] = __ldg(reinterpret_cast<const uint16_t*>(mp + 16 * r));
    v[r] = __ldg(vp + r * vstep);
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint32_t w[4] = {v[r].x, v[r].y, v[r].z, v[r].w};
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const uint2 sl = lut[(m16[r] >> (4 * g)) & 0xFu];
      X[r][2 * g] = __byte_perm(w[g], 0u, sl.x);
      X[r][2 * g + 1] = __byte_perm(w[g], 0u, sl.y);
    }
  }

  uint32_t* vs32 = reinterpret_cast<uint32_t*>(a.vs);
  uint8_t* es = a.es + q_off;
  const bool quad_lead = (lane & 3) == 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint4 sl = *reinterpret_cast<const uint4*>(&slots[warp][2 * k]);  // features 2k, 2k + 1
    const uint32_t x0 = X[0][k], x1 = X[1][k], x2 = X[2][k], x3 = X[3][k];
    uint32_t k0 = x0, k1 = x1, k2 = x2, k3 = x3;
    if (keys) {
      k0 = k4_key2(x0);
      k1 = k4_key2(x1);
      k2 = k4_key2(x2);
      k3 = k4_key2(x3);
    }
    const uint32_t b01 = k4_ge(k0, k1), b02 = k4_ge(k0, k2), b03 = k4_ge(k0, k3);
    const uint32_t b12 = k4_ge(k1, k2), b13 = k4_ge(k1, k3), b23 = k4_ge(k2, k3);
    const uint32_t K0 = k4_maj(b01, b02, b03), K1 = k4_maj(~b01, b12, b13);
    const uint32_t K2 = k4_maj(~b02, ~b12, b23), K3 = k4_maj(~b03, ~b13, ~b23);
    const uint32_t v0 = k4_sel(K0, x0, k4_sel(K1, x1, x2));
    const uint32_t v1 = k4_sel(K3, x3, k4_sel(K2, x2, x1));
    const uint32_t nib = ((~K0 & K1) & 0x00010001u) | ((~K0 & ~K1) & 0x00020002u) |
                         ((K3 | ~K2) & 0x00040004u) | ((K3 | K2) & 0x00080008u);
    uint32_t hw = nib << (4 * (lane & 3));
    hw |= __shfl_xor_sync(0xffffffffu, hw, 1);
    hw |= __shfl_xor_sync(0xffffffffu, hw, 2);
    // feature 2k (low halves); a dense feature keeps its 4 tokens as the row
    // pair (x0, x1 | x2, x3) with the fixed selectors 0x4 / 0xE
    const bool da = (sl.x >> 31) != 0u, db = (sl.z >> 31) != 0u;
    uint32_t* pa = vs32 + (sl.x & 0x7FFFFFFFu) + lane;
    uint32_t* pb = vs32 + (sl.z & 0x7FFFFFFFu) + lane;
    *pa = da ? __byte_perm(x0, x1, 0x5410) : __byte_perm(v0, v1, 0x5410);
    *pb = db ? __byte_perm(x0, x1, 0x7632) : __byte_perm(v0, v1, 0x7632);
    if (da) pa[nw] = __byte_perm(x2, x3, 0x5410);
    if (db) pb[nw] = __byte_perm(x2, x3, 0x7632);
    if (quad_lead) {
      *reinterpret_cast<uint16_t*>(es + sl.y) = da ? static_cast<uint16_t>(0x4444u) : static_cast<uint16_t>(hw);
      *reinterpret_cast<uint16_t*>(es + sl.w) = db ? static_cast<uint16_t>(0x4444u) : static_cast<uint16_t>(hw >> 16);
      if (da) *reinterpret_cast<uint16_t*>(es + sl.y + 16) = static_cast<uint16_t>(0xEEEEu);
      if (db) *reinterpret_cast<uint16_t*>(es + sl.w + 16) = static_cast<uint16_t>(0xEEEEu);
    }
  }
}

}  // namespace s24
