// Feature-wise (transposed) 2:4 selection fused into a GEMM epilogue.
//
// In the K1/K3 epilogues lane l of a warp holds token row (tile row) l and one
// 32-feature chunk of that row, already token-wise compressed: 8 kept pairs
// (bf16x2) + 8 nibbles. The feature-wise groups of the reference's split GEMM
// (ref sparsify_feature_wise, sparse24.py:96-115) are 4 CONSECUTIVE TOKENS of
// one feature = the 4 lanes of a lane quad. This routine
//   1. exchanges within each quad so lane r owns features 8r..8r+7 of the
//      chunk for all 4 tokens (3 xor-shuffle rounds of 2 words + nibbles),
//   2. expands them to bf16 pairs (PRMT with a nibble -> selector LUT),
//   3. runs the top-2 over the 4 tokens two features at a time (native bf16x2
//      compares + bitwise majority: the rule of meta.cuh, on the stored bf16
//      values), and
//   4. writes the transposed operand the weight-gradient sparse GEMM reads:
//      vals [features, tokens/2] (K-major along tokens) + hw metadata
//      (rows = features, K = tokens), plus per-feature nonzero counts
//      (before | after << 32) for the drop statistics.
// It runs for every feature, independent of the split plan (only known after
// K1's counts): the sparse weight-gradient GEMM later skips dense features.
#pragma once
#include <cuda_bf16.h>
#include "meta.cuh"

namespace s24 {

struct FwTarget {
  __nv_bfloat16* vals;         // [features_pad128, kdim/2]; nullptr disables the fused selection
  uint8_t* meta;               // hw layout: rows = features, K = kdim tokens
  unsigned long long* counts;  // [features] += before | after << 32 (nullable)
  int kdim;                    // padded token count (multiple of 128)
};

// nibble -> PRMT selectors expanding a kept pair (lo, hi) into the group's 4
// halfwords (x: halfwords 0,1; y: halfwords 2,3)
__device__ __forceinline__ uint2 fw_sel_for(uint32_t nib) {
  const uint32_t i0 = nib & 3u, i1 = nib >> 2;
  uint32_t s[4];
#pragma unroll
  for (uint32_t q = 0; q < 4; ++q) s[q] = (q == i0) ? 0x10u : (q == i1) ? 0x32u : 0x44u;
  return make_uint2(s[0] | (s[1] << 8), s[2] | (s[3] << 8));
}

// per-warp copy of the 16-entry selector table in static shared memory
// (lanes 0..15 fill it; every warp writes the same values)
__device__ __forceinline__ const uint2* fw_lut_init() {
  __shared__ uint2 lut[16][16];
  const uint32_t warp = (threadIdx.x >> 5) & 15u, lane = threadIdx.x & 31u;
  if (lane < 16) lut[warp][lane] = fw_sel_for(lane);
  __syncwarp();
  return lut[warp];
}

__device__ __forceinline__ uint32_t fw_key2(uint32_t x) {
  const uint32_t mag = x & 0x7FFF7FFFu;
  const __nv_bfloat162 m = *reinterpret_cast<const __nv_bfloat162*>(&mag);
  const uint32_t nan = __hne2_mask(m, m);
  return (mag & ~nan) | (0xBF80BF80u & nan);
}

__device__ __forceinline__ uint32_t fw_ge(uint32_t a, uint32_t b) {
  return __hge2_mask(*reinterpret_cast<const __nv_bfloat162*>(&a), *reinterpret_cast<const __nv_bfloat162*>(&b));
}

__device__ __forceinline__ uint32_t fw_nz(uint32_t x) {
  const uint32_t mag = x & 0x7FFF7FFFu;
  const __nv_bfloat162 z = __floats2bfloat162_rn(0.f, 0.f);
  return __hne2_mask(*reinterpret_cast<const __nv_bfloat162*>(&mag), z) & 0x00010001u;
}

__device__ __forceinline__ uint32_t fw_pick4(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t i) {
  return i == 0 ? a0 : i == 1 ? a1 : i == 2 ? a2 : a3;
}

// packed[g]: kept pair of group g (features col0+4g..+3) of this lane's token;
// nib8: the 8 group nibbles (group g at bits 4g). token: global token index of
// this lane's row (quads of lanes are 4-aligned token groups).
__device__ __forceinline__ void fw_select_chunk(const FwTarget& o, const uint32_t (&packed)[8], uint32_t nib8,
                                                int token, int col0, uint32_t lane, const uint2* lut) {
  // tile rows past the padded token count (last CTA of a pair) have nowhere to
  // go; kdim is a multiple of 128 so this is uniform across the warp
  if (token >= o.kdim) return;
  const uint32_t r = lane & 3u;  // my token position within the group
  // 1. quad exchange: slot x receives token r^x's pairs of groups 2r, 2r+1
  uint32_t Wx[4][2], Nx[4];
#pragma unroll
  for (uint32_t x = 0; x < 4; ++x) {
    const uint32_t p = r ^ x;  // the receiver's quad position: send it its groups 2p, 2p+1
    const uint32_t s0 = fw_pick4(packed[0], packed[2], packed[4], packed[6], p);
    const uint32_t s1 = fw_pick4(packed[1], packed[3], packed[5], packed[7], p);
    const uint32_t sn = (nib8 >> (8 * p)) & 0xFFu;
    if (x == 0) {
      Wx[0][0] = s0;
      Wx[0][1] = s1;
      Nx[0] = sn;
    } else {
      Wx[x][0] = __shfl_xor_sync(0xffffffffu, s0, x);
      Wx[x][1] = __shfl_xor_sync(0xffffffffu, s1, x);
      Nx[x] = __shfl_xor_sync(0xffffffffu, sn, x);
    }
  }
  // back to token order: token t sits in slot r^t; expand to bf16 pairs
  // X[t][k] = features (8r + 2k, 8r + 2k + 1) of token t
  uint32_t X[4][4];
#pragma unroll
  for (uint32_t t = 0; t < 4; ++t) {
    const uint32_t sx = r ^ t;
    const uint32_t w0 = fw_pick4(Wx[0][0], Wx[1][0], Wx[2][0], Wx[3][0], sx);
    const uint32_t w1 = fw_pick4(Wx[0][1], Wx[1][1], Wx[2][1], Wx[3][1], sx);
    const uint32_t nn = fw_pick4(Nx[0], Nx[1], Nx[2], Nx[3], sx);
    const uint2 l0 = lut[nn & 0xFu], l1 = lut[(nn >> 4) & 0xFu];
    X[t][0] = __byte_perm(w0, 0u, l0.x);
    X[t][1] = __byte_perm(w0, 0u, l0.y);
    X[t][2] = __byte_perm(w1, 0u, l1.x);
    X[t][3] = __byte_perm(w1, 0u, l1.y);
  }
  // 2. per-lane output bases: features f0 .. f0+7 share one metadata atom row
  // (f0 % 8 == 0) so feature j's halfword is 16*j bytes after feature f0's
  const int f0 = col0 + 8 * static_cast<int>(r);
  const int tg = token >> 2;
  const uint32_t qd = (lane >> 2) & 3u;  // quad within the 16-token run of one metadata halfword
  uint32_t* vrow0 = reinterpret_cast<uint32_t*>(o.vals + static_cast<long long>(f0) * (o.kdim / 2)) + tg;
  uint8_t* mrow0 = o.meta + meta_hw_halfword_offset(f0, token >> 4, o.kdim);
  // 3. top-2 over the 4 tokens, two features per register
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t x0 = X[0][k], x1 = X[1][k], x2 = X[2][k], x3 = X[3][k];
    const uint32_t k0 = fw_key2(x0), k1 = fw_key2(x1), k2 = fw_key2(x2), k3 = fw_key2(x3);
    // token i beats token j (i < j) iff key_i >= key_j: ties go to the lower token
    const uint32_t b01 = fw_ge(k0, k1), b02 = fw_ge(k0, k2), b03 = fw_ge(k0, k3);
    const uint32_t b12 = fw_ge(k1, k2), b13 = fw_ge(k1, k3), b23 = fw_ge(k2, k3);
    // kept <=> beats at least two of the other three
    const uint32_t K0 = (b01 & b02) | (b01 & b03) | (b02 & b03);
    const uint32_t K1 = (~b01 & b12) | (~b01 & b13) | (b12 & b13);
    const uint32_t K2 = (~b02 & ~b12) | (~b02 & b23) | (~b12 & b23);
    const uint32_t K3 = (~b03 & ~b13) | (~b03 & ~b23) | (~b13 & ~b23);
    const uint32_t v0 = (x0 & K0) | (((x1 & K1) | (x2 & ~K1)) & ~K0);  // first kept token
    const uint32_t v1 = (x3 & K3) | (((x2 & K2) | (x1 & ~K2)) & ~K3);  // second kept token
    const uint32_t kb = (K0 & 0x00010001u) | (K1 & 0x00020002u) | (K2 & 0x00040004u) | (K3 & 0x00080008u);
    uint32_t nzb = 0, nza = 0;
    if (o.counts) {
      nzb = fw_nz(x0) + fw_nz(x1) + fw_nz(x2) + fw_nz(x3);
      nza = fw_nz(v0) + fw_nz(v1);
    }
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int j = 2 * k + half;
      const uint32_t sh = 16u * half;
      vrow0[static_cast<long long>(j) * (o.kdim / 4)] = ((v0 >> sh) & 0xFFFFu) | (((v1 >> sh) & 0xFFFFu) << 16);
      // metadata halfword of (feature, 16 tokens) = nibbles of 4 consecutive quads
      uint32_t hw = keep_nibble((kb >> sh) & 0xFu) << (4u * qd);
      hw |= __shfl_xor_sync(0xffffffffu, hw, 4);
      hw |= __shfl_xor_sync(0xffffffffu, hw, 8);
      if (qd == 0) *reinterpret_cast<uint16_t*>(mrow0 + 16 * j) = static_cast<uint16_t>(hw);
      if (o.counts) {
        unsigned long long c = static_cast<unsigned long long>((nzb >> sh) & 0xFFFFu) |
                               (static_cast<unsigned long long>((nza >> sh) & 0xFFFFu) << 32);
        c += __shfl_xor_sync(0xffffffffu, c, 4);
        c += __shfl_xor_sync(0xffffffffu, c, 8);
        c += __shfl_xor_sync(0xffffffffu, c, 16);
        if ((lane >> 2) == 0 && c) atomicAdd(o.counts + f0 + j, c);
      }
    }
  }
}

}  // namespace s24
