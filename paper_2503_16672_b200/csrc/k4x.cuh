// K4x -- the hot-path feature-wise split (rank order + paired dense rows,
// see k4.cuh) for one or two token-wise 2:4 operands that share their
// metadata: the activation and g_pre of the same FFN step (g_pre lives on
// the forward keep pattern, ffn.py:415-417). Everything that depends only on
// the metadata and the plan -- metadata loads, the nibble -> byte-permute
// selectors, output row offsets -- is done once for both operands, and the
// per-feature offsets come from a small shared-memory table instead of warp
// shuffles. Grid (h/128, n/128), 8 warps x 16 features x 128 tokens.
#pragma once
#include <cuda_bf16.h>
#include "k4.cuh"
#include "meta.cuh"

namespace s24 {

struct K4xArgs {
  const __nv_bfloat16* vals[2];  // token-wise compressed [n, h/2]
  const uint8_t* meta;           // shared hw metadata (rows = tokens, K = h)
  int n, h;
  const int* feat_pos;           // plan: rank in sparse list, or -(rank in dense)-1
  int pair_rows;                 // 2 * n_dense: rows of the dense pairs in front
  __nv_bfloat16* vs[2];          // [pad128(pair_rows + n_sparse), n/2]
  uint8_t* es[2];                // hw metadata of vs
  const int* row_map;            // nullable [n]: token j of the split is row row_map[j] of vals / meta
};

// per-feature output slot of one warp unit
struct K4xSlot {
  uint32_t ofs;    // 32-bit word offset of the feature's (first) vs row at this token block
  uint32_t mb;     // byte offset of its metadata halfword for token quad 0
  uint32_t mb2;    // dense: the second row's metadata offset
  uint32_t dense;  // 1: paired dense feature
};

#ifndef S24_K4X_SWIZZLE
#define S24_K4X_SWIZZLE 1
#endif
template <int NOPS, bool NONNEG0>
__global__ void __launch_bounds__(256) k_feature_split_x(K4xArgs a) {
  __shared__ K4xSlot slots[8][16];
  const uint2* lut = k4_lut_init();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = a.n, h = a.h;
  // CTA order: square super-tiles of SW x SW blocks (feature-block fastest
  // inside), so that consecutive CTAs read adjacent 128-byte pieces of the
  // same token rows AND write adjacent pieces of the same feature rows
  int fb = blockIdx.x, tb = blockIdx.y;
  if constexpr (S24_K4X_SWIZZLE > 1) {
    constexpr int SW = S24_K4X_SWIZZLE;
    const int nfb = gridDim.x, ntb = gridDim.y;
    const int id = blockIdx.y * nfb + blockIdx.x;
    const int per_row = SW * nfb;  // CTAs per super-row (SW token blocks x all feature blocks)
    const int sr = id / per_row, rem = id - sr * per_row;
    const int rows_here = min(SW, ntb - sr * SW);
    const int sc = rem / (SW * rows_here), in = rem - sc * SW * rows_here;
    const int cols_here = min(SW, nfb - sc * SW);
    fb = sc * SW + in % cols_here;
    tb = sr * SW + in / cols_here;
  }
  const int t0 = tb * 128, fbase = fb * 128 + warp * 16;
  const uint32_t nw = static_cast<uint32_t>(n / 4);
  if (lane < 16) {
    const int pos = __ldg(a.feat_pos + fbase + lane);
    const uint32_t row = pos >= 0 ? static_cast<uint32_t>(a.pair_rows + pos) : 2u * static_cast<uint32_t>(-pos - 1);
    K4xSlot s;
    s.ofs = row * nw + static_cast<uint32_t>(t0 / 4);
    s.mb = static_cast<uint32_t>(meta_hw_halfword_offset(row, t0 / 16, n));
    s.mb2 = static_cast<uint32_t>(meta_hw_halfword_offset(row + 1, t0 / 16, n));
    s.dense = pos < 0 ? 1u : 0u;
    slots[warp][lane] = s;
  }
  __syncwarp();
  const int t = t0 + 4 * lane;
  const uint32_t qd = static_cast<uint32_t>(lane) >> 2;
  const uint32_t q_off = 4u * (qd >> 1) + 128u * (qd & 1u);

  // load + expand both operands with one set of selectors
  uint32_t X[NOPS][4][8];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    // (row_map: the split's token order is a permutation of the rows of vals)
    const int src = a.row_map ? __ldg(a.row_map + t + r) : t + r;
    const uint32_t m16 = __ldg(reinterpret_cast<const uint16_t*>(a.meta + meta_hw_halfword_offset(src, fbase / 16, h)));
    uint4 v[NOPS];
#pragma unroll
    for (int o = 0; o < NOPS; ++o)
      v[o] = __ldg(reinterpret_cast<const uint4*>(a.vals[o] + static_cast<long long>(src) * (h / 2) + fbase / 2));
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const uint2 sl = lut[(m16 >> (4 * g)) & 0xFu];
#pragma unroll
      for (int o = 0; o < NOPS; ++o) {
        const uint32_t w = g == 0 ? v[o].x : g == 1 ? v[o].y : g == 2 ? v[o].z : v[o].w;
        X[o][r][2 * g] = __byte_perm(w, 0u, sl.x);
        X[o][r][2 * g + 1] = __byte_perm(w, 0u, sl.y);
      }
    }
  }

#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const K4xSlot s0 = slots[warp][2 * k], s1 = slots[warp][2 * k + 1];
#pragma unroll
    for (int o = 0; o < NOPS; ++o) {
      const uint32_t x0 = X[o][0][k], x1 = X[o][1][k], x2 = X[o][2][k], x3 = X[o][3][k];
      uint32_t* vs32 = reinterpret_cast<uint32_t*>(a.vs[o]);
      uint8_t* es = a.es[o];
      if (!(s0.dense & s1.dense)) {
        uint32_t k0 = x0, k1 = x1, k2 = x2, k3 = x3;
        if (!(NONNEG0 && o == 0)) {
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
