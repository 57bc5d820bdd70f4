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

// per-feature output slot of one warp unit
struct K4xSlot {
  uint32_t ofs;    // 32-bit word offset of the feature's (first) vs row at this token block
  uint32_t mb;     // byte offset of its metadata halfword for token quad 0
  uint32_t mb2;    // dense: the second row's metadata offset
  uint32_t dense;  // 1: paired dense feature
};

// NONNEG: the operand is relu^2 (>= 0): raw bf16 values order correctly under
// HSET2 and the magnitude / NaN keys are skipped, unless nan_flag is raised
// K4X_WARPS warps per CTA (16 features each) at <= 64 registers: several CTAs
// fit next to a running GEMM CTA, so the split runs on the side stream
// co-resident with the GEMMs
#ifndef S24_K4X_WARPS
#define S24_K4X_WARPS 4
#endif
#ifndef S24_K4X_TB
#define S24_K4X_TB 1
#endif
constexpr int K4X_TB = S24_K4X_TB;
constexpr int K4X_WARPS = S24_K4X_WARPS;
template <bool NONNEG>
__global__ void __launch_bounds__(32 * K4X_WARPS, 32 / K4X_WARPS) k_feature_split_x(K4xArgs a) {
  __shared__ K4xSlot slots[K4X_WARPS][16];
  const uint2* lut = k4_lut_init();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = a.n, h = a.h;
  const bool keys = !NONNEG || (a.nan_flag != nullptr && __ldg(a.nan_flag) != 0ull);
  // CTA = K4X_WARPS x 16 features (blockIdx.x) x K4X_TB consecutive 128-token
  // blocks (blockIdx.y): the per-feature output slots are computed once and
  // advanced by one metadata atom / 32 value words per token block
  const int fbase = blockIdx.x * (16 * K4X_WARPS) + warp * 16;
  const int tblocks = n / 128;
  const uint32_t nw = static_cast<uint32_t>(n / 4);
  if (lane < 16) {
    const int pos = __ldg(a.feat_pos + fbase + lane);
    const uint32_t row = pos >= 0 ? static_cast<uint32_t>(a.pair_rows + pos) : 2u * static_cast<uint32_t>(-pos - 1);
    const int t0 = blockIdx.y * K4X_TB * 128;
    K4xSlot s;
    s.ofs = row * nw + static_cast<uint32_t>(t0 / 4);
    s.mb = static_cast<uint32_t>(meta_hw_halfword_offset(row, t0 / 16, n));
    s.mb2 = static_cast<uint32_t>(meta_hw_halfword_offset(row + 1, t0 / 16, n));
    s.dense = pos < 0 ? 1u : 0u;
    slots[warp][lane] = s;
  }
  __syncwarp();
  for (int bi = 0; bi < K4X_TB; ++bi) {
    const int tb = blockIdx.y * K4X_TB + bi;
    if (tb >= tblocks) break;
    const int t0 = tb * 128;
    const uint32_t dofs = 32u * bi, dmb = 2048u * bi;  // (slot offsets of token block bi)
    const int t = t0 + 4 * lane;
    const uint32_t qd = static_cast<uint32_t>(lane) >> 2;
    const uint32_t q_off = 4u * (qd >> 1) + 128u * (qd & 1u);

    // load + expand: X[token][feature pair] packed bf16x2
    uint32_t X[4][8];
  #pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint32_t m16 = __ldg(reinterpret_cast<const uint16_t*>(a.meta + meta_hw_halfword_offset(t + r, fbase / 16, h)));
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.vals + static_cast<long long>(t + r) * (h / 2) + fbase / 2));
  #pragma unroll
      for (int g = 0; g < 4; ++g) {
        const uint2 sl = lut[(m16 >> (4 * g)) & 0xFu];
        const uint32_t w = g == 0 ? v.x : g == 1 ? v.y : g == 2 ? v.z : v.w;
        X[r][2 * g] = __byte_perm(w, 0u, sl.x);
        X[r][2 * g + 1] = __byte_perm(w, 0u, sl.y);
      }
    }

  #pragma unroll
    for (int k = 0; k < 8; ++k) {
      K4xSlot s0 = slots[warp][2 * k], s1 = slots[warp][2 * k + 1];
      s0.ofs += dofs;
      s1.ofs += dofs;
      s0.mb += dmb;
      s1.mb += dmb;
      s0.mb2 += dmb;
      s1.mb2 += dmb;
      const uint32_t x0 = X[0][k], x1 = X[1][k], x2 = X[2][k], x3 = X[3][k];
      uint32_t* vs32 = reinterpret_cast<uint32_t*>(a.vs);
      uint8_t* es = a.es;
      if (!(s0.dense & s1.dense)) {
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
        if (!s0.dense) {
          vs32[s0.ofs + lane] = __byte_perm(v0, v1, 0x5410);
          if ((lane & 3) == 0) *reinterpret_cast<uint16_t*>(es + s0.mb + q_off) = static_cast<uint16_t>(hw);
        }
        if (!s1.dense) {
          vs32[s1.ofs + lane] = __byte_perm(v0, v1, 0x7632);
          if ((lane & 3) == 0) *reinterpret_cast<uint16_t*>(es + s1.mb + q_off) = static_cast<uint16_t>(hw >> 16);
        }
      }
      // paired dense features: (x0, x1) | selector 0x4, (x2, x3) | 0xE
      if (s0.dense) {
        vs32[s0.ofs + lane] = __byte_perm(x0, x1, 0x5410);
        vs32[s0.ofs + nw + lane] = __byte_perm(x2, x3, 0x5410);
        if ((lane & 3) == 0) {
          *reinterpret_cast<uint16_t*>(es + s0.mb + q_off) = 0x4444;
          *reinterpret_cast<uint16_t*>(es + s0.mb2 + q_off) = 0xEEEE;
        }
      }
      if (s1.dense) {
        vs32[s1.ofs + lane] = __byte_perm(x0, x1, 0x7632);
        vs32[s1.ofs + nw + lane] = __byte_perm(x2, x3, 0x7632);
        if ((lane & 3) == 0) {
          *reinterpret_cast<uint16_t*>(es + s1.mb + q_off) = 0x4444;
          *reinterpret_cast<uint16_t*>(es + s1.mb2 + q_off) = 0xEEEE;
        }
      }
    }

  }
}

}  // namespace s24
