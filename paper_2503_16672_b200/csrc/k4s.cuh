// K4s -- the feature-wise split (K4x, k4x.cuh) computed inside the 2:4 GEMM
// whose A operand is the token-wise compressed tensor it splits (fwd.out
// reads act, bwd.d_x reads g_pre): dedicated warps of the GEMM CTA take the
// A tile (128 tokens x 128 features, 64 kept values per row, SWIZZLE_128B)
// and its metadata atom straight from the pipeline stage the TMA producer
// filled for the MMA, so the split reads nothing from global memory.
//
// Work split: the stage of k-block kb holds 8 units of 16 features; every
// N tile of the same token rows loads the same stage, so N tile nb takes the
// units j == nb (mod min(tiles_n, 8)) and each unit is done exactly once.
// A unit is copied to registers, the stage is released (one extra arrival on
// its empty barrier), and the selection / stores run from registers.
// Same rank rule, layout (paired dense rows, rank order) and output as K4x.
#pragma once
#include <cuda_bf16.h>
#include "k4.cuh"
#include "meta.cuh"

namespace s24 {

struct K4sSlot {
  uint32_t ofs;    // 32-bit word offset of the feature's (first) vs row at this token block
  uint32_t mb;     // byte offset of its metadata halfword for token quad 0
  uint32_t mb2;    // dense: the second row's metadata offset
  uint32_t dense;  // 1: paired dense feature
};

// registers of one unit: 4 token rows x 16 features of one lane
struct K4sRegs {
  uint4 v[4];
  uint32_t m16[4];
};

// copy unit j (16 features) of the stage: lane holds tokens 4*lane .. +3
__device__ __forceinline__ void k4s_load(const uint8_t* sa, const uint8_t* se, int j, int lane, K4sRegs& u) {
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint32_t row = static_cast<uint32_t>(4 * lane + r);
    // SWIZZLE_128B: 16-byte chunk c of row r sits at chunk c ^ (r % 8)
    u.v[r] = *reinterpret_cast<const uint4*>(sa + row * 128u + ((static_cast<uint32_t>(j) ^ (row & 7u)) << 4));
    u.m16[r] = *reinterpret_cast<const uint16_t*>(se + meta_atom_halfword_byte(row, static_cast<uint32_t>(j)));
  }
}

// OR of every loaded word (an always-nonzero dependency for the stage release)
__device__ __forceinline__ uint32_t k4s_fold(const K4sRegs& u) {
  uint32_t x = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r) x |= u.v[r].x | u.v[r].y | u.v[r].z | u.v[r].w | u.m16[r];
  return x;
}

// selection + stores of one unit (features f0 .. f0+15, tokens t0 .. t0+127)
__device__ __forceinline__ void k4s_compute(const K4Args& a, const K4sRegs& u, int f0, int t0, int lane,
                                            const uint2* lut, K4sSlot* slots) {
  const uint32_t nw = static_cast<uint32_t>(a.n / 4);
  if (lane < 16) {
    const int pos = __ldg(a.feat_pos + f0 + lane);
    const uint32_t row = pos >= 0 ? static_cast<uint32_t>(a.pair_rows + pos) : 2u * static_cast<uint32_t>(-pos - 1);
    K4sSlot s;
    s.ofs = row * nw + static_cast<uint32_t>(t0 / 4);
    s.mb = static_cast<uint32_t>(meta_hw_halfword_offset(row, t0 / 16, a.n));
    s.mb2 = static_cast<uint32_t>(meta_hw_halfword_offset(row + 1, t0 / 16, a.n));
    s.dense = pos < 0 ? 1u : 0u;
    slots[lane] = s;
  }
  __syncwarp();
  uint32_t X[4][8];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const uint2 sl = lut[(u.m16[r] >> (4 * g)) & 0xFu];
      const uint32_t w = g == 0 ? u.v[r].x : g == 1 ? u.v[r].y : g == 2 ? u.v[r].z : u.v[r].w;
      X[r][2 * g] = __byte_perm(w, 0u, sl.x);
      X[r][2 * g + 1] = __byte_perm(w, 0u, sl.y);
    }
  }
  const uint32_t qd = static_cast<uint32_t>(lane) >> 2;
  const uint32_t q_off = 4u * (qd >> 1) + 128u * (qd & 1u);
  uint32_t* vs32 = reinterpret_cast<uint32_t*>(a.vs);
  uint8_t* es = a.es;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const K4sSlot s0 = slots[2 * k], s1 = slots[2 * k + 1];
    const uint32_t x0 = X[0][k], x1 = X[1][k], x2 = X[2][k], x3 = X[3][k];
    if (!(s0.dense & s1.dense)) {
      uint32_t k0 = x0, k1 = x1, k2 = x2, k3 = x3;
      if (!a.nonneg) {
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
  __syncwarp();  // slots are rewritten by the next unit
}

}  // namespace s24
