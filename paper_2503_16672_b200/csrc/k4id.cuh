// K4, identity layout: the feature-wise (transposed) split of a token-wise
// 2:4-compressed [n, h] matrix with every memory access coalesced.
//
// Output operand (rows of one 2:4 GEMM over K = tokens):
//   rows [0, 2*n_dense)          dense feature of rank r as two fixed-selector
//                                2:4 rows: 2r = tokens 4j, 4j+1 (selector 0x4),
//                                2r+1 = tokens 4j+2, 4j+3 (0xE)
//   rows [2*n_dense, pair_pad)   zero padding (pair_pad = pad128(2*n_dense))
//   rows [pair_pad, pair_pad+h)  feature f at row pair_pad + f: the
//                                feature-wise top-2 of every group of 4 tokens
//                                (ref sparsify_feature_wise, sparse24.py:96-115)
//                                -- for all features; the GEMM's row_valid
//                                skips the dense ones
// Because output rows follow the input feature order, one CTA (128 tokens x
// 128 features) reads one 16 KiB value tile + one 2 KiB metadata atom and
// writes 128 full 128-byte value rows + one whole 2 KiB metadata atom: no
// partial-sector traffic (the rank-ordered layout of k4.cuh scatters 2-byte
// metadata writes and 16-byte reads).
#pragma once
#include <cuda_bf16.h>
#include "k4.cuh"
#include "meta.cuh"

namespace s24 {

struct K4IdArgs {
  const __nv_bfloat16* vals;  // token-wise compressed [n, h/2]
  const uint8_t* meta;        // its hw metadata (rows = tokens, K = h)
  int n, h;
  const int* feat_pos;        // plan: rank in sparse list, or -(rank in dense)-1
  int n_dense;
  int pair_pad;               // pad128(2 * n_dense)
  __nv_bfloat16* vs;          // [pair_pad + h, n/2]
  uint8_t* es;                // hw metadata of vs (rows pair_pad + h, K = n)
  unsigned long long* stats;  // += nonzeros before/after over sparse features (WITH_STATS)
};

template <bool WITH_STATS, bool NONNEG>
__global__ void __launch_bounds__(256) k_feature_split_id(K4IdArgs a) {
  __shared__ __align__(16) uint8_t s_vals[128 * 128];  // 128 token rows x 64 kept values
  __shared__ __align__(16) uint8_t s_meta[2048];        // input atom (tokens x features)
  __shared__ __align__(16) uint8_t s_out[2048];         // output atom (features x tokens)
  const uint2* lut = k4_lut_init();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int fb = blockIdx.x, tb = blockIdx.y;  // feature block, token block
  const int n = a.n, h = a.h;

  // 1. coalesced loads: 128 rows x 128 B values (8 threads per row), 2 KiB meta
  {
    const uint8_t* src = reinterpret_cast<const uint8_t*>(a.vals) + static_cast<long long>(tb) * 128 * h +
                         static_cast<long long>(fb) * 128;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = tid + 256 * i, row = idx >> 3, c = idx & 7;
      *reinterpret_cast<uint4*>(s_vals + row * 128 + c * 16) =
          __ldg(reinterpret_cast<const uint4*>(src + static_cast<long long>(row) * h + c * 16));
    }
    if (tid < 128) {
      const uint8_t* m = a.meta + (static_cast<long long>(tb) * (h / 128) + fb) * 2048;
      *reinterpret_cast<uint4*>(s_meta + tid * 16) = __ldg(reinterpret_cast<const uint4*>(m + tid * 16));
    }
  }
  __syncthreads();

  // 2. warp w: features 16w..16w+15 of the block; lane: tokens 4*lane..+3
  const int f0 = fb * 128 + warp * 16;
  const int my_pos = __ldg(a.feat_pos + f0 + (lane & 15));
  uint32_t X[4][8];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int row = 4 * lane + r;
    const uint4 v = *reinterpret_cast<const uint4*>(s_vals + row * 128 + warp * 16);
    const uint32_t m16 = *reinterpret_cast<const uint16_t*>(s_meta + meta_atom_halfword_byte(row, warp));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const uint2 sl = lut[(m16 >> (4 * g)) & 0xFu];
      X[r][2 * g] = __byte_perm(w[g], 0u, sl.x);
      X[r][2 * g + 1] = __byte_perm(w[g], 0u, sl.y);
    }
  }
  const uint32_t nw = static_cast<uint32_t>(n / 4);  // 32-bit words per output row
  uint32_t* vs32 = reinterpret_cast<uint32_t*>(a.vs);
  const uint32_t col = static_cast<uint32_t>(tb) * 32u + static_cast<uint32_t>(lane);  // this lane's word
  uint32_t cnt_b = 0, cnt_a = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t x0 = X[0][k], x1 = X[1][k], x2 = X[2][k], x3 = X[3][k];
    uint32_t k0 = x0, k1 = x1, k2 = x2, k3 = x3;
    if constexpr (!NONNEG) {
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
    const uint32_t nib = ((~K0 & K1) & 0x00010001u) | ((~K0 & ~K1) & 0x00020002u) | ((K3 | ~K2) & 0x00040004u) |
                         ((K3 | K2) & 0x00080008u);
    uint32_t hw = nib << (4 * (lane & 3));
    hw |= __shfl_xor_sync(0xffffffffu, hw, 1);
    hw |= __shfl_xor_sync(0xffffffffu, hw, 2);
    const int pos0 = __shfl_sync(0xffffffffu, my_pos, 2 * k), pos1 = __shfl_sync(0xffffffffu, my_pos, 2 * k + 1);
    // feature-wise rows (identity order), 128 B per feature per block: coalesced
    const uint32_t r0 = static_cast<uint32_t>(a.pair_pad + f0 + 2 * k);
    vs32[static_cast<unsigned long long>(r0) * nw + col] = __byte_perm(v0, v1, 0x5410);
    vs32[static_cast<unsigned long long>(r0 + 1) * nw + col] = __byte_perm(v0, v1, 0x7632);
    if ((lane & 3) == 0) {
      const uint32_t q = static_cast<uint32_t>(lane) >> 2;
      *reinterpret_cast<uint16_t*>(s_out + meta_atom_halfword_byte(warp * 16 + 2 * k, q)) = static_cast<uint16_t>(hw);
      *reinterpret_cast<uint16_t*>(s_out + meta_atom_halfword_byte(warp * 16 + 2 * k + 1, q)) =
          static_cast<uint16_t>(hw >> 16);
    }
    // dense features also go out exactly, as two fixed-selector rows
    if (pos0 < 0) {
      const unsigned long long rr = 2ull * static_cast<unsigned long long>(-pos0 - 1);
      vs32[rr * nw + col] = __byte_perm(x0, x1, 0x5410);
      vs32[(rr + 1) * nw + col] = __byte_perm(x2, x3, 0x5410);
    }
    if (pos1 < 0) {
      const unsigned long long rr = 2ull * static_cast<unsigned long long>(-pos1 - 1);
      vs32[rr * nw + col] = __byte_perm(x0, x1, 0x7632);
      vs32[(rr + 1) * nw + col] = __byte_perm(x2, x3, 0x7632);
    }
    if constexpr (WITH_STATS) {
      const uint32_t nzb = k4_nz(x0) + k4_nz(x1) + k4_nz(x2) + k4_nz(x3);
      const uint32_t nza = k4_nz(v0) + k4_nz(v1);
      if (pos0 >= 0) {
        cnt_b += nzb & 0xFFFFu;
        cnt_a += nza & 0xFFFFu;
      }
      if (pos1 >= 0) {
        cnt_b += nzb >> 16;
        cnt_a += nza >> 16;
      }
    }
  }
  if constexpr (WITH_STATS) {
    k4_warp_add(cnt_b, a.stats);
    k4_warp_add(cnt_a, a.stats + 1);
  }
  __syncthreads();
  // 3. the output metadata atom (rows pair_pad + 128 fb .., tokens 128 tb ..): 2 KiB, coalesced
  if (tid < 128) {
    uint8_t* e = a.es + (static_cast<long long>(a.pair_pad / 128 + fb) * (n / 128) + tb) * 2048;
    *reinterpret_cast<uint4*>(e + tid * 16) = *reinterpret_cast<const uint4*>(s_out + tid * 16);
  }
  // 4. feature block 0 also writes this token block of the pair region:
  // selector atoms (rows 2r: 0x4444, 2r+1: 0xEEEE; a 16-byte unit of the
  // atom holds rows of one parity) and zero values for the padding rows
  if (fb == 0) {
    const int atoms = a.pair_pad / 128;
    for (int i = tid; i < atoms * 128; i += 256) {
      const int ab = i >> 7, u = i & 127;  // atom, 16-byte unit (m0 = (u >> 0) & 7 of offset 16*m0 + ...)
      const uint32_t m0 = static_cast<uint32_t>(u) & 7u;
      const uint32_t pat = (m0 & 1u) ? 0xEEEEEEEEu : 0x44444444u;
      uint8_t* e = a.es + (static_cast<long long>(ab) * (n / 128) + tb) * 2048;
      *reinterpret_cast<uint4*>(e + u * 16) = make_uint4(pat, pat, pat, pat);
    }
    for (int i = tid; i < (a.pair_pad - 2 * a.n_dense) * 32; i += 256) {
      const int row = 2 * a.n_dense + (i >> 5), w = i & 31;
      vs32[static_cast<unsigned long long>(row) * nw + static_cast<uint32_t>(tb) * 32u + w] = 0u;
    }
  }
}

}  // namespace s24
