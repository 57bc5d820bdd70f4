// HBM-bound 2:4 kernels and their C-ABI entry points:
//   token-wise / feature-wise sparsify, mask compression, decompress,
//   metadata converters, row gather (token permutation), the split plan (K7)
//   and the feature-wise transposed split (K4).
#include <cuda_bf16.h>

#include <type_traits>

#include "host_util.h"
#include "meta.cuh"
#include "ptx.cuh"
#include "k4.cuh"
#include "k4x.cuh"

namespace s24 {

template <typename T>
__device__ __forceinline__ float ldf(const T* p) {
  if constexpr (std::is_same_v<T, float>)
    return *p;
  else
    return __bfloat162float(*p);
}

template <typename T>
__device__ __forceinline__ void stf(T* p, float v) {
  if constexpr (std::is_same_v<T, float>)
    *p = v;
  else
    *p = __float2bfloat16_rn(v);
}

__device__ __forceinline__ unsigned long long block_sum_u64_to(unsigned long long v, unsigned long long* dst) {
  // warp reduce then one atomic per warp
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
  return v;
}

// ---------------------------------------------------------------------------
// token-wise sparsify: each thread owns GPT consecutive groups of one row.
template <typename T, int GPT>
__global__ void k_sparsify_token(const T* __restrict__ a, long long rows, long long cols, long long lda,
                                 __nv_bfloat16* __restrict__ vals, uint8_t* __restrict__ meta_ref,
                                 uint8_t* __restrict__ meta_hw, uint8_t* __restrict__ mask,
                                 unsigned long long* stats) {
  const long long chunks_per_row = cols / (4 * GPT);
  const long long total = rows * chunks_per_row;
  unsigned long long nb = 0, na = 0;
  for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < total;
       w += (long long)gridDim.x * blockDim.x) {
    const long long r = w / chunks_per_row;
    const long long c0 = (w - r * chunks_per_row) * 4 * GPT;
    const T* src = a + r * lda + c0;
    uint32_t m16 = 0;
#pragma unroll
    for (int g = 0; g < GPT; ++g) {
      const float x0 = ldf(src + 4 * g), x1 = ldf(src + 4 * g + 1), x2 = ldf(src + 4 * g + 2),
                  x3 = ldf(src + 4 * g + 3);
      nb += (x0 != 0.f) + (x1 != 0.f) + (x2 != 0.f) + (x3 != 0.f);
      const uint32_t keep = top2_keep_mask(x0, x1, x2, x3);
      const uint32_t nib = keep_to_nibble(keep);
      const float v0 = sel4(x0, x1, x2, x3, nib & 3u), v1 = sel4(x0, x1, x2, x3, nib >> 2);
      na += (v0 != 0.f) + (v1 != 0.f);
      const long long gi = c0 / 4 + g;
      reinterpret_cast<__nv_bfloat162*>(vals + r * (cols / 2))[gi] = __floats2bfloat162_rn(v0, v1);
      if (meta_ref) {
        meta_ref[(r * (cols / 4) + gi) * 2] = static_cast<uint8_t>(nib & 3u);
        meta_ref[(r * (cols / 4) + gi) * 2 + 1] = static_cast<uint8_t>(nib >> 2);
      }
      if (mask) {
#pragma unroll
        for (int i = 0; i < 4; ++i) mask[r * cols + c0 + 4 * g + i] = (keep >> i) & 1u;
      }
      m16 |= nib << (4 * g);
    }
    if constexpr (GPT == 4) {
      if (meta_hw)
        *reinterpret_cast<uint16_t*>(meta_hw + meta_hw_halfword_offset(r, c0 / 16, cols)) = (uint16_t)m16;
    }
  }
  if (stats) {
    block_sum_u64_to(nb, stats);
    block_sum_u64_to(na, stats + 1);
  }
}

// Fast path of the above for the operand the GEMMs consume (values + hw
// metadata only; cols % 128 == 0). A warp unit is 4 rows x 128 columns: rows
// {2j, 2j+1, 2j+8, 2j+9} of a 16-row group, lane = (k1, row, k2) owning the
// 16-column chunk q = k1 + 2 k2 of the atom column. That is exactly the
// rows x chunks that share the hw layout's 32-byte metadata sectors (meta.cuh:
// rows m0 = 2j, 2j+1 and m1 = 0, 1; chunks k2 = 0..3 at fixed k1), so each
// half-warp's halfword stores fill one whole sector instead of scattering
// halfwords that other warps complete much later. Per row the warp reads 256
// contiguous input bytes and writes 128 contiguous value bytes.
#ifndef S24_TOK_U
#define S24_TOK_U 2
#endif
template <typename T, bool STATS>
__global__ void __launch_bounds__(256) k_sparsify_token_hw(const T* __restrict__ a, long long rows, long long cols,
                                                           long long lda, __nv_bfloat16* __restrict__ vals,
                                                           uint8_t* __restrict__ meta_hw,
                                                           unsigned long long* stats) {
  constexpr int VEC = 16 / sizeof(T);  // elements per 16-byte load
  constexpr int NV = 16 / VEC;         // 16-byte loads per chunk
  constexpr int U = S24_TOK_U;         // warp units per iteration (their loads in flight together)
  const int lane = threadIdx.x & 31;
  const int k1 = lane >> 4, rho = (lane >> 2) & 3, k2 = lane & 3;
  const long long kbs = cols / 128;                       // atom columns
  const long long units = (rows + 15) / 16 * 4 * kbs;     // row quartets (4 per 16-row group) x atom columns
  const long long wstride = (long long)gridDim.x * (blockDim.x >> 5);
  unsigned long long nb = 0, na = 0;
  for (long long u0 = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); u0 < units; u0 += U * wstride) {
    uint4 ld[U][NV];
    long long rr[U], qq[U];
#pragma unroll
    for (int c = 0; c < U; ++c) {
      const long long u = u0 + c * wstride;
      const long long quartet = u / kbs, kb = u - quartet * kbs;
      rr[c] = (quartet >> 2) * 16 + (quartet & 3) * 2 + (rho & 1) + 8 * (rho >> 1);
      qq[c] = kb * 8 + k1 + 2 * k2;
      if (u < units && rr[c] < rows) {
        const uint4* src = reinterpret_cast<const uint4*>(a + rr[c] * lda + qq[c] * 16);
#pragma unroll
        for (int v = 0; v < NV; ++v) ld[c][v] = __ldcs(src + v);  // (streamed: read once)
      }
    }
#pragma unroll
    for (int c = 0; c < U; ++c) {
      const long long u = u0 + c * wstride;
      if (u >= units || rr[c] >= rows) continue;
      const long long r = rr[c], q = qq[c];
      if constexpr (sizeof(T) == 2) {
        // bf16 in: two groups per bf16x2 word (the same in-group position of
        // groups g and g + 1), ranked with K4x's packed compares (k4.cuh)
        const uint32_t w[8] = {ld[c][0].x, ld[c][0].y, ld[c][0].z, ld[c][0].w,
                               ld[c][1].x, ld[c][1].y, ld[c][1].z, ld[c][1].w};
        uint32_t packed[4];
        uint32_t m16 = 0;
#pragma unroll
        for (int g = 0; g < 4; g += 2) {
          const uint32_t x0 = __byte_perm(w[2 * g], w[2 * g + 2], 0x5410);
          const uint32_t x1 = __byte_perm(w[2 * g], w[2 * g + 2], 0x7632);
          const uint32_t x2 = __byte_perm(w[2 * g + 1], w[2 * g + 3], 0x5410);
          const uint32_t x3 = __byte_perm(w[2 * g + 1], w[2 * g + 3], 0x7632);
          const uint32_t k0 = k4_key2(x0), k1 = k4_key2(x1), k2 = k4_key2(x2), k3 = k4_key2(x3);
          const uint32_t b01 = k4_ge(k0, k1), b02 = k4_ge(k0, k2), b03 = k4_ge(k0, k3);
          const uint32_t b12 = k4_ge(k1, k2), b13 = k4_ge(k1, k3), b23 = k4_ge(k2, k3);
          const uint32_t K0 = k4_maj(b01, b02, b03), K1 = k4_maj(~b01, b12, b13);
          const uint32_t K2 = k4_maj(~b02, ~b12, b23), K3 = k4_maj(~b03, ~b13, ~b23);
          const uint32_t v0 = k4_sel(K0, x0, k4_sel(K1, x1, x2));
          const uint32_t v1 = k4_sel(K3, x3, k4_sel(K2, x2, x1));
          const uint32_t nib = ((~K0 & K1) & 0x00010001u) | ((~K0 & ~K1) & 0x00020002u) |
                               ((K3 | ~K2) & 0x00040004u) | ((K3 | K2) & 0x00080008u);
          packed[g] = __byte_perm(v0, v1, 0x5410);
          packed[g + 1] = __byte_perm(v0, v1, 0x7632);
          m16 |= ((nib & 0xFu) | ((nib >> 12) & 0xF0u)) << (4 * g);
          if constexpr (STATS) {
            nb += __popc(k4_nz(x0) | (k4_nz(x1) << 1) | (k4_nz(x2) << 2) | (k4_nz(x3) << 3));
            na += __popc(k4_nz(v0) | (k4_nz(v1) << 1));
          }
        }
        *reinterpret_cast<uint4*>(vals + r * (cols / 2) + q * 8) =
            make_uint4(packed[0], packed[1], packed[2], packed[3]);
        *reinterpret_cast<uint16_t*>(meta_hw + meta_hw_halfword_offset(r, q, cols)) = static_cast<uint16_t>(m16);
        continue;
      }
      float x[16];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const uint32_t wv[4] = {ld[c][v].x, ld[c][v].y, ld[c][v].z, ld[c][v].w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if constexpr (sizeof(T) == 4) {
            x[v * 4 + i] = __uint_as_float(wv[i]);
          } else {
            x[v * 8 + 2 * i] = __uint_as_float(wv[i] << 16);
            x[v * 8 + 2 * i + 1] = __uint_as_float(wv[i] & 0xFFFF0000u);
          }
        }
      }
      uint32_t packed[4];
      uint32_t m16 = 0;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const float x0 = x[4 * g], x1 = x[4 * g + 1], x2 = x[4 * g + 2], x3 = x[4 * g + 3];
        // magnitude keys, NaN -> -1 (ranked below every number: max(NaN, -1) = -1)
        const float k0 = fmaxf(fabsf(x0), -1.f), k1 = fmaxf(fabsf(x1), -1.f);
        const float k2 = fmaxf(fabsf(x2), -1.f), k3 = fmaxf(fabsf(x3), -1.f);
        const uint32_t b01 = fge_mask(k0, k1), b02 = fge_mask(k0, k2), b03 = fge_mask(k0, k3);
        const uint32_t b12 = fge_mask(k1, k2), b13 = fge_mask(k1, k3), b23 = fge_mask(k2, k3);
        const uint32_t K0 = maj3(b01, b02, b03), K1 = maj3(~b01, b12, b13);
        const uint32_t K2 = maj3(~b02, ~b12, b23), K3 = maj3(~b03, ~b13, ~b23);
        const uint32_t u0 = __float_as_uint(x0), u1 = __float_as_uint(x1), u2 = __float_as_uint(x2),
                       u3 = __float_as_uint(x3);
        const float v0 = __uint_as_float(bsel(K0, u0, bsel(K1, u1, u2)));  // first kept
        const float v1 = __uint_as_float(bsel(K3, u3, bsel(K2, u2, u1)));  // second kept
        if constexpr (STATS) {
          nb += (x0 != 0.f) + (x1 != 0.f) + (x2 != 0.f) + (x3 != 0.f);
          na += (v0 != 0.f) + (v1 != 0.f);
        }
        packed[g] = pack_bf16x2(v0, v1);
        m16 |= keep_nibble((K0 & 1u) | (K1 & 2u) | (K2 & 4u) | (K3 & 8u)) << (4 * g);
      }
      *reinterpret_cast<uint4*>(vals + r * (cols / 2) + q * 8) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
      *reinterpret_cast<uint16_t*>(meta_hw + meta_hw_halfword_offset(r, q, cols)) = static_cast<uint16_t>(m16);
    }
  }
  if constexpr (STATS) {
    block_sum_u64_to(nb, stats);
    block_sum_u64_to(na, stats + 1);
  }
}

// ---------------------------------------------------------------------------
// feature-wise sparsify: thread owns GPT consecutive row-groups of column j.
// fwd_mask (nullable, uint8 [rows, cols]): entries outside it read as zero
// before the selection and the counts (sparsify_feature_wise_masked,
// ref sparse24.py:118-129: masked-out values are not "dropped").
template <typename T, int GPT>
__global__ void k_sparsify_feature(const T* __restrict__ a, long long rows, long long cols, long long lda,
                                   __nv_bfloat16* __restrict__ vals_t, uint8_t* __restrict__ meta_ref,
                                   uint8_t* __restrict__ meta_hw, uint8_t* __restrict__ mask,
                                   unsigned long long* stats, const uint8_t* __restrict__ fwd_mask) {
  const long long chunks = rows / (4 * GPT);
  const long long total = chunks * cols;
  unsigned long long nb = 0, na = 0;
  for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < total;
       w += (long long)gridDim.x * blockDim.x) {
    const long long ch = w / cols;
    const long long j = w - ch * cols;
    uint32_t m16 = 0;
#pragma unroll
    for (int g = 0; g < GPT; ++g) {
      const long long gi = ch * GPT + g;  // row group index
      const long long r0 = gi * 4;
      float x0 = ldf(a + r0 * lda + j), x1 = ldf(a + (r0 + 1) * lda + j), x2 = ldf(a + (r0 + 2) * lda + j),
            x3 = ldf(a + (r0 + 3) * lda + j);
      if (fwd_mask) {
        x0 = fwd_mask[r0 * cols + j] ? x0 : 0.f;
        x1 = fwd_mask[(r0 + 1) * cols + j] ? x1 : 0.f;
        x2 = fwd_mask[(r0 + 2) * cols + j] ? x2 : 0.f;
        x3 = fwd_mask[(r0 + 3) * cols + j] ? x3 : 0.f;
      }
      nb += (x0 != 0.f) + (x1 != 0.f) + (x2 != 0.f) + (x3 != 0.f);
      const uint32_t keep = top2_keep_mask(x0, x1, x2, x3);
      const uint32_t nib = keep_to_nibble(keep);
      const float v0 = sel4(x0, x1, x2, x3, nib & 3u), v1 = sel4(x0, x1, x2, x3, nib >> 2);
      na += (v0 != 0.f) + (v1 != 0.f);
      reinterpret_cast<__nv_bfloat162*>(vals_t + j * (rows / 2))[gi] = __floats2bfloat162_rn(v0, v1);
      if (meta_ref) {
        meta_ref[(gi * cols + j) * 2] = static_cast<uint8_t>(nib & 3u);
        meta_ref[(gi * cols + j) * 2 + 1] = static_cast<uint8_t>(nib >> 2);
      }
      if (mask) {
#pragma unroll
        for (int i = 0; i < 4; ++i) mask[(r0 + i) * cols + j] = (keep >> i) & 1u;
      }
      m16 |= nib << (4 * g);
    }
    if constexpr (GPT == 4) {
      if (meta_hw)
        *reinterpret_cast<uint16_t*>(meta_hw + meta_hw_halfword_offset(j, ch, rows)) = (uint16_t)m16;
    }
  }
  if (stats) {
    block_sum_u64_to(nb, stats);
    block_sum_u64_to(na, stats + 1);
  }
}

// ---------------------------------------------------------------------------
// compress with a given mask (exact when supp(a) is inside the mask)
template <typename T>
__global__ void k_compress_mask(const T* __restrict__ a, long long rows, long long cols, long long lda,
                                const uint8_t* __restrict__ mask, __nv_bfloat16* __restrict__ vals,
                                uint8_t* __restrict__ meta_ref, uint8_t* __restrict__ meta_hw, int* bad) {
  const long long groups = rows * (cols / 4);
  int my_bad = 0;
  for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < groups;
       w += (long long)gridDim.x * blockDim.x) {
    const long long r = w / (cols / 4);
    const long long gi = w - r * (cols / 4);
    const long long c0 = gi * 4;
    uint32_t keep = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) keep |= (mask[r * cols + c0 + i] ? 1u : 0u) << i;
    if (__popc(keep) != 2) {
      ++my_bad;
      keep = 3u;
    }
    const uint32_t nib = keep_to_nibble(keep);
    const T* src = a + r * lda + c0;
    const float v0 = ldf(src + (nib & 3u)), v1 = ldf(src + (nib >> 2));
    reinterpret_cast<__nv_bfloat162*>(vals + r * (cols / 2))[gi] = __floats2bfloat162_rn(v0, v1);
    if (meta_ref) {
      meta_ref[w * 2] = static_cast<uint8_t>(nib & 3u);
      meta_ref[w * 2 + 1] = static_cast<uint8_t>(nib >> 2);
    }
    if (meta_hw) {
      // nibble-granular write: 4 groups share a halfword -> atomic OR on the
      // containing 32-bit word (caller zeroes meta_hw)
      const uint64_t off = meta_hw_halfword_offset(r, c0 / 16, cols);
      const uint32_t shift = 4u * (gi & 3) + 8u * (off & 2);
      atomicOr(reinterpret_cast<unsigned int*>(meta_hw + (off & ~3ull)), nib << shift);
    }
  }
  if (bad && my_bad) atomicAdd(bad, my_bad);
}

// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t read_nibble_token(const uint8_t* meta_ref, const uint8_t* meta_hw,
                                                      long long r, long long gi, long long cols) {
  if (meta_ref) {
    const long long o = (r * (cols / 4) + gi) * 2;
    return meta_ref[o] | (meta_ref[o + 1] << 2);
  }
  const uint16_t h = *reinterpret_cast<const uint16_t*>(meta_hw + meta_hw_halfword_offset(r, gi / 4, cols));
  return (h >> (4 * (gi & 3))) & 0xFu;
}

template <typename OutT>
__global__ void k_decompress_token(const __nv_bfloat16* __restrict__ vals, const uint8_t* __restrict__ meta_ref,
                                   const uint8_t* __restrict__ meta_hw, long long rows, long long cols,
                                   OutT* __restrict__ out, long long ldo) {
  const long long groups = rows * (cols / 4);
  for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < groups;
       w += (long long)gridDim.x * blockDim.x) {
    const long long r = w / (cols / 4);
    const long long gi = w - r * (cols / 4);
    const uint32_t nib = read_nibble_token(meta_ref, meta_hw, r, gi, cols);
    const __nv_bfloat162 v = reinterpret_cast<const __nv_bfloat162*>(vals + r * (cols / 2))[gi];
    float o[4] = {0.f, 0.f, 0.f, 0.f};
    o[nib & 3u] = __bfloat162float(v.x);
    o[nib >> 2] = __bfloat162float(v.y);
#pragma unroll
    for (int i = 0; i < 4; ++i) stf(out + r * ldo + gi * 4 + i, o[i]);
  }
}

template <typename OutT>
__global__ void k_decompress_feature(const __nv_bfloat16* __restrict__ vals_t, const uint8_t* __restrict__ meta_ref,
                                     const uint8_t* __restrict__ meta_hw, long long rows, long long cols,
                                     OutT* __restrict__ out, long long ldo) {
  const long long groups = (rows / 4) * cols;
  for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < groups;
       w += (long long)gridDim.x * blockDim.x) {
    const long long gi = w / cols;
    const long long j = w - gi * cols;
    uint32_t nib;
    if (meta_ref) {
      nib = meta_ref[(gi * cols + j) * 2] | (meta_ref[(gi * cols + j) * 2 + 1] << 2);
    } else {
      const uint16_t h = *reinterpret_cast<const uint16_t*>(meta_hw + meta_hw_halfword_offset(j, gi / 4, rows));
      nib = (h >> (4 * (gi & 3))) & 0xFu;
    }
    const __nv_bfloat162 v = reinterpret_cast<const __nv_bfloat162*>(vals_t + j * (rows / 2))[gi];
    float o[4] = {0.f, 0.f, 0.f, 0.f};
    o[nib & 3u] = __bfloat162float(v.x);
    o[nib >> 2] = __bfloat162float(v.y);
#pragma unroll
    for (int i = 0; i < 4; ++i) stf(out + (gi * 4 + i) * ldo + j, o[i]);
  }
}

__global__ void k_meta_hw_to_ref(const uint8_t* __restrict__ hw, long long rows, long long cols,
                                 uint8_t* __restrict__ ref) {
  const long long groups = rows * (cols / 4);
  for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < groups;
       w += (long long)gridDim.x * blockDim.x) {
    const long long r = w / (cols / 4);
    const long long gi = w - r * (cols / 4);
    const uint32_t nib = read_nibble_token(nullptr, hw, r, gi, cols);
    ref[w * 2] = nib & 3u;
    ref[w * 2 + 1] = nib >> 2;
  }
}

__global__ void k_meta_ref_to_hw(const uint8_t* __restrict__ ref, long long rows, long long cols,
                                 uint8_t* __restrict__ hw) {
  const long long halves = rows * (cols / 16);
  for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < halves;
       w += (long long)gridDim.x * blockDim.x) {
    const long long r = w / (cols / 16);
    const long long q = w - r * (cols / 16);
    uint32_t h = 0;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const long long o = (r * (cols / 4) + q * 4 + g) * 2;
      h |= (ref[o] | (ref[o + 1] << 2)) << (4 * g);
    }
    *reinterpret_cast<uint16_t*>(hw + meta_hw_halfword_offset(r, q, cols)) = (uint16_t)h;
  }
}

// ---------------------------------------------------------------------------
// K6: row gather, one warp per row, 16-byte vectors (eight in flight per lane;
// the source is streamed once, so its loads are evict-first)
__global__ void k_gather_rows(const uint8_t* __restrict__ in, long long rows, long long row_bytes,
                              long long ld_in, const int* __restrict__ src, uint8_t* __restrict__ out,
                              long long ld_out) {
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  const long long vecs = row_bytes >> 4;
  for (long long r = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    const uint4* s = reinterpret_cast<const uint4*>(in + (long long)src[r] * ld_in);
    uint4* d = reinterpret_cast<uint4*>(out + r * ld_out);
    long long v = lane;
    for (; v + 32 * 7 < vecs; v += 256) {  // eight 16-byte loads in flight per lane, then the stores
      uint4 t[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) t[j] = __ldcs(s + v + 32 * j);
#pragma unroll
      for (int j = 0; j < 8; ++j) d[v + 32 * j] = t[j];
    }
    for (; v < vecs; v += 32) d[v] = s[v];
  }
}

// ---------------------------------------------------------------------------
// K7: partition_features (ref splitgemm.py:41-52) on the device. Stable
// ascending order of (count, index): the n_sparse smallest keys are sparse.
// Radix select on the count value (11-bit digits over the significant bits,
// warp-aggregated shared-memory histograms), then the tie-break among the
// threshold count's features by index (a block scan), then one block scan
// that writes both ascending index lists and feat_pos. One CTA.
__device__ __forceinline__ int block_excl_scan_1024(int v, int* warp_tot, int lane, int wid, int& total) {
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  __syncthreads();  // (warp_tot may still be read by a previous scan)
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const int w = warp_tot[lane];
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    warp_tot[lane] = wi - w;
    if (lane == 31) warp_tot[32] = wi;
  }
  __syncthreads();
  total = warp_tot[32];
  return warp_tot[wid] + inc - v;
}

// Each thread owns PER consecutive features (j0 = tid * PER) and keeps their
// counts in registers, so the counts are read from memory once: the passes
// below (max, two radix digits, tie-break, lists) only touch registers and the
// 8 KB of shared memory (histogram, scan totals).
template <int PER>
__global__ void __launch_bounds__(1024, 2) k_plan(const int* __restrict__ counts_g, int h, int n_sparse,
                                               int* __restrict__ sparse_idx, int* __restrict__ dense_idx,
                                               int* __restrict__ feat_pos) {
  constexpr int DIGIT = 11, BINS = 1 << DIGIT;
  __shared__ unsigned hist[BINS];
  __shared__ int warp_tot[33];
  __shared__ unsigned sh_max, sh_prefix;
  __shared__ int sh_rank, sh_jstar;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int j0 = tid * PER;
  unsigned c[PER];
  if (j0 + PER <= h && (h & 3) == 0 && PER % 4 == 0) {
#pragma unroll
    for (int i = 0; i < PER; i += 4) {
      const int4 v = __ldg(reinterpret_cast<const int4*>(counts_g + j0 + i));
      c[i] = v.x, c[i + 1] = v.y, c[i + 2] = v.z, c[i + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < PER; ++i) c[i] = j0 + i < h ? static_cast<unsigned>(__ldg(counts_g + j0 + i)) : 0u;
  }
  auto valid = [&](int i) { return j0 + i < h; };

  unsigned cstar = 0xFFFFFFFFu;  // threshold count; features with count < cstar are sparse
  int jstar = -1;                // ... and those with count == cstar up to index jstar
  if (n_sparse > 0) {
    if (tid == 0) {
      sh_max = 0;
      sh_prefix = 0;
      sh_rank = n_sparse - 1;
    }
    unsigned mx = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) mx = max(mx, valid(i) ? c[i] : 0u);
    mx = __reduce_max_sync(0xffffffffu, mx);
    __syncthreads();
    if (lane == 0) atomicMax(&sh_max, mx);
    __syncthreads();
    const int bits = 32 - __clz(static_cast<int>(sh_max | 1u));
    // digits from the most significant one down
    for (int hi = bits; hi > 0; hi -= DIGIT) {
      const int shift = max(hi - DIGIT, 0), width = hi - shift;
      for (int b = tid; b < BINS; b += 1024) hist[b] = 0;
      __syncthreads();
      const unsigned prefix = sh_prefix;  // the bits above `hi` of the threshold
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        unsigned bin = 0xFFFFFFFFu;
        if (valid(i) && (hi >= 32 ? 0u : (c[i] >> hi)) == prefix) bin = (c[i] >> shift) & ((1u << width) - 1u);
        const unsigned peers = __match_any_sync(0xffffffffu, bin);
        if (bin != 0xFFFFFFFFu && lane == __ffs(peers) - 1) atomicAdd(&hist[bin], __popc(peers));
      }
      __syncthreads();
      // locate the digit holding rank sh_rank: each thread scans 2 bins
      const unsigned h0 = hist[2 * tid], h1 = hist[2 * tid + 1];
      int total;
      const int exc = block_excl_scan_1024(static_cast<int>(h0 + h1), warp_tot, lane, wid, total);
      const int rank = sh_rank;
      __syncthreads();
      if (rank >= exc && rank < exc + static_cast<int>(h0 + h1)) {
        const bool first = rank < exc + static_cast<int>(h0);
        const unsigned digit = 2u * tid + (first ? 0u : 1u);
        sh_rank = rank - exc - (first ? 0 : static_cast<int>(h0));
        sh_prefix = (prefix << width) | digit;
      }
      __syncthreads();
    }
    cstar = sh_prefix;
    // tie-break: the (sh_rank)-th feature (by index) with count == cstar
    int my_eq = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) my_eq += valid(i) && c[i] == cstar ? 1 : 0;
    int total;
    const int exc = block_excl_scan_1024(my_eq, warp_tot, lane, wid, total);
    const int r = sh_rank;
    if (r >= exc && r < exc + my_eq) {
      int seen = exc;
#pragma unroll
      for (int i = 0; i < PER; ++i)
        if (valid(i) && c[i] == cstar && seen++ == r) sh_jstar = j0 + i;
    }
    __syncthreads();
    jstar = sh_jstar;
  }

  // flags and block-wide exclusive scan of sparse counts in index order
  unsigned long long sparse_bits = 0;
#pragma unroll
  for (int i = 0; i < PER; ++i)
    if (valid(i) && n_sparse > 0 && (c[i] < cstar || (c[i] == cstar && j0 + i <= jstar))) sparse_bits |= 1ull << i;
  int total;
  int s_off = block_excl_scan_1024(__popcll(sparse_bits), warp_tot, lane, wid, total);
  int d_off = min(j0, h) - s_off;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    if (!valid(i)) break;
    const int j = j0 + i;
    if (sparse_bits >> i & 1ull) {
      sparse_idx[s_off] = j;
      feat_pos[j] = s_off;
      ++s_off;
    } else {
      dense_idx[d_off] = j;
      feat_pos[j] = -d_off - 1;
      ++d_off;
    }
  }
}

// ---------------------------------------------------------------------------
// K4 standalone grid: CTA = 128 tokens x 128 features = 8 warp units.
template <bool WITH_STATS, bool NONNEG>
__global__ void __launch_bounds__(256) k_feature_split(K4Args a) {
  const uint2* lut = k4_lut_init();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grid (h/128, n/128), or fewer CTAs striding over the blocks (a light
  // footprint that leaves room for a co-running GEMM's CTAs)
  const int fblocks = a.h / 128, blocks = fblocks * (a.n / 128);
  for (int b = blockIdx.y * gridDim.x + blockIdx.x; b < blocks; b += gridDim.x * gridDim.y) {
    const int fb = b % fblocks, tb = b / fblocks;
    k4_warp_unit<WITH_STATS, NONNEG>(a, tb * 128, fb * 128 + warp * 16, lane, lut);
  }
}

static int grid_for(long long work, int block) {
  long long g = (work + block - 1) / block;
  const long long cap = static_cast<long long>(num_sms()) * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

// validates a K4 job and writes the padding rows of its outputs (zero values,
// valid (0,1) selectors); shared by the standalone grid and the GEMM
// background mode
int k4_prepare(const void* vals, const uint8_t* meta_hw, int64_t n, int64_t h, const int* feat_pos,
               int64_t n_sparse, int64_t n_dense, void* vs, uint8_t* es, void* vd, cudaStream_t st, K4Args* out,
               int64_t pair_rows) {
  if (n % 128 != 0 || h % 128 != 0) return fail(S24_ERR_DIMENSION, "feature split needs n, h multiples of 128");
  if (n_sparse + n_dense != h) return fail(S24_ERR_STATE, "plan sizes do not add up to h");
  if ((vs == nullptr) != (es == nullptr)) return fail(S24_ERR_DIMENSION, "vs and es go together");
  const bool paired = pair_rows >= 0;
  if (paired && (pair_rows != 2 * n_dense || vs == nullptr))
    return fail(S24_ERR_DIMENSION, "paired layout needs pair_rows == 2 * n_dense and the sparse operand");
  const int64_t vs_rows = (paired ? pair_rows : 0) + n_sparse;  // rows of the 2:4 operand
  const int64_t sp_pad = (vs_rows + 127) / 128 * 128, d_pad = (n_dense + 127) / 128 * 128;
  if (vs != nullptr && sp_pad > vs_rows) {
    cudaMemsetAsync(static_cast<__nv_bfloat16*>(vs) + vs_rows * (n / 2), 0, (sp_pad - vs_rows) * (n / 2) * 2, st);
    cudaMemsetAsync(es + (vs_rows / 128) * (n / 128) * 2048, 0x44, (n / 128) * 2048, st);
  }
  if (!paired && d_pad > n_dense && vd)
    cudaMemsetAsync(static_cast<__nv_bfloat16*>(vd) + n_dense * n, 0, (d_pad - n_dense) * n * 2, st);
  *out = K4Args{static_cast<const __nv_bfloat16*>(vals), meta_hw, static_cast<int>(n), static_cast<int>(h), feat_pos,
                static_cast<__nv_bfloat16*>(vs), es, static_cast<__nv_bfloat16*>(vd), nullptr, 0,
                static_cast<int>(paired ? pair_rows : -1)};
  return S24_OK;
}

__global__ void k_timestamp(unsigned long long* out) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *out = t;
}

// diagnostics: SM clock over a busy-wait of `ns` nanoseconds, one record
// (clock64 delta, globaltimer delta) per CTA
__global__ void k_clock_probe(unsigned long long* out, unsigned long long ns) {
  unsigned long long c0, g0, c1, g1;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c0));
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  } while (g1 - g0 < ns);
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c1));
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = c1 - c0;
    out[2 * blockIdx.x + 1] = g1 - g0;
  }
}

}  // namespace s24

using namespace s24;

extern "C" {

int s24_sparsify_token(const void* a, int dtype, int64_t rows, int64_t cols, int64_t lda, void* vals,
                       uint8_t* meta_ref, uint8_t* meta_hw, uint8_t* mask, unsigned long long* stats,
                       void* stream) {
  if (rows < 0 || cols < 0) return fail(S24_ERR_DIMENSION, "negative shape");
  if (cols % 4 != 0) return fail(S24_ERR_DIMENSION, "token-wise groups need cols %% 4 == 0, got %lld", (long long)cols);
  if (lda < cols) return fail(S24_ERR_DIMENSION, "lda < cols");
  if (meta_hw && cols % 128 != 0) return fail(S24_ERR_DIMENSION, "hw metadata needs cols %% 128 == 0");
  if (dtype != S24_F32 && dtype != S24_BF16) return fail(S24_ERR_PRECISION, "unsupported dtype");
  if (rows == 0 || cols == 0) return S24_OK;
  auto st = static_cast<cudaStream_t>(stream);
  const bool q = cols % 16 == 0;
  const long long work = rows * cols / (q ? 16 : 4);
  const int g = grid_for(work, 256);
  const int esz = dtype == S24_F32 ? 4 : 2;
  if (meta_hw && !meta_ref && !mask && aligned16(a) && aligned16(vals) && (lda * esz) % 16 == 0) {
    auto run = [&](auto stats_tag) {
      constexpr bool ST = decltype(stats_tag)::value;
      if (dtype == S24_F32)
        k_sparsify_token_hw<float, ST><<<g, 256, 0, st>>>(static_cast<const float*>(a), rows, cols, lda,
                                                          static_cast<__nv_bfloat16*>(vals), meta_hw, stats);
      else
        k_sparsify_token_hw<__nv_bfloat16, ST><<<g, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(a), rows, cols,
                                                                  lda, static_cast<__nv_bfloat16*>(vals), meta_hw,
                                                                  stats);
    };
    if (stats)
      run(std::true_type{});
    else
      run(std::false_type{});
    return check_launch("k_sparsify_token_hw");
  }
  if (dtype == S24_F32) {
    if (q)
      k_sparsify_token<float, 4><<<g, 256, 0, st>>>(static_cast<const float*>(a), rows, cols, lda,
                                                     static_cast<__nv_bfloat16*>(vals), meta_ref, meta_hw, mask, stats);
    else
      k_sparsify_token<float, 1><<<g, 256, 0, st>>>(static_cast<const float*>(a), rows, cols, lda,
                                                     static_cast<__nv_bfloat16*>(vals), meta_ref, nullptr, mask, stats);
  } else {
    if (q)
      k_sparsify_token<__nv_bfloat16, 4><<<g, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(a), rows, cols, lda,
                                                             static_cast<__nv_bfloat16*>(vals), meta_ref, meta_hw,
                                                             mask, stats);
    else
      k_sparsify_token<__nv_bfloat16, 1><<<g, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(a), rows, cols, lda,
                                                             static_cast<__nv_bfloat16*>(vals), meta_ref, nullptr,
                                                             mask, stats);
  }
  return check_launch("k_sparsify_token");
}

int s24_sparsify_feature_masked(const void* a, int dtype, int64_t rows, int64_t cols, int64_t lda,
                                const uint8_t* fwd_mask, void* vals_t, uint8_t* meta_ref, uint8_t* meta_hw,
                                uint8_t* mask, unsigned long long* stats, void* stream) {
  if (rows < 0 || cols < 0) return fail(S24_ERR_DIMENSION, "negative shape");
  if (rows % 4 != 0) return fail(S24_ERR_DIMENSION, "feature-wise groups need rows %% 4 == 0, got %lld", (long long)rows);
  if (lda < cols) return fail(S24_ERR_DIMENSION, "lda < cols");
  if (meta_hw && rows % 128 != 0) return fail(S24_ERR_DIMENSION, "hw metadata needs rows %% 128 == 0");
  if (dtype != S24_F32 && dtype != S24_BF16) return fail(S24_ERR_PRECISION, "unsupported dtype");
  if (rows == 0 || cols == 0) return S24_OK;
  auto st = static_cast<cudaStream_t>(stream);
  const bool q = rows % 16 == 0;
  const long long work = rows * cols / (q ? 16 : 4);
  const int g = grid_for(work, 256);
  auto vt = static_cast<__nv_bfloat16*>(vals_t);
  if (dtype == S24_F32) {
    auto ap = static_cast<const float*>(a);
    if (q)
      k_sparsify_feature<float, 4><<<g, 256, 0, st>>>(ap, rows, cols, lda, vt, meta_ref, meta_hw, mask, stats, fwd_mask);
    else
      k_sparsify_feature<float, 1><<<g, 256, 0, st>>>(ap, rows, cols, lda, vt, meta_ref, nullptr, mask, stats, fwd_mask);
  } else {
    auto ap = static_cast<const __nv_bfloat16*>(a);
    if (q)
      k_sparsify_feature<__nv_bfloat16, 4><<<g, 256, 0, st>>>(ap, rows, cols, lda, vt, meta_ref, meta_hw, mask, stats,
                                                               fwd_mask);
    else
      k_sparsify_feature<__nv_bfloat16, 1><<<g, 256, 0, st>>>(ap, rows, cols, lda, vt, meta_ref, nullptr, mask, stats,
                                                               fwd_mask);
  }
  return check_launch("k_sparsify_feature");
}

int s24_sparsify_feature(const void* a, int dtype, int64_t rows, int64_t cols, int64_t lda, void* vals_t,
                         uint8_t* meta_ref, uint8_t* meta_hw, uint8_t* mask, unsigned long long* stats,
                         void* stream) {
  return s24_sparsify_feature_masked(a, dtype, rows, cols, lda, nullptr, vals_t, meta_ref, meta_hw, mask, stats,
                                     stream);
}

int s24_compress_token_with_mask(const void* a, int dtype, int64_t rows, int64_t cols, int64_t lda,
                                 const uint8_t* mask, void* vals, uint8_t* meta_ref, uint8_t* meta_hw,
                                 int* bad_groups, void* stream) {
  if (rows < 0 || cols < 0 || cols % 4 != 0) return fail(S24_ERR_DIMENSION, "mask/matrix shapes unusable");
  if (meta_hw && cols % 128 != 0) return fail(S24_ERR_DIMENSION, "hw metadata needs cols %% 128 == 0");
  if (rows == 0 || cols == 0) return S24_OK;
  auto st = static_cast<cudaStream_t>(stream);
  if (meta_hw) {
    const int64_t bytes = s24_meta_hw_bytes(rows, cols);
    cudaMemsetAsync(meta_hw, 0, bytes, st);
  }
  const int g = grid_for(rows * cols / 4, 256);
  if (dtype == S24_F32)
    k_compress_mask<float><<<g, 256, 0, st>>>(static_cast<const float*>(a), rows, cols, lda, mask,
                                              static_cast<__nv_bfloat16*>(vals), meta_ref, meta_hw, bad_groups);
  else if (dtype == S24_BF16)
    k_compress_mask<__nv_bfloat16><<<g, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(a), rows, cols, lda, mask,
                                                      static_cast<__nv_bfloat16*>(vals), meta_ref, meta_hw, bad_groups);
  else
    return fail(S24_ERR_PRECISION, "unsupported dtype");
  return check_launch("k_compress_mask");
}

int s24_decompress_token(const void* vals, const uint8_t* meta_ref, const uint8_t* meta_hw, int64_t rows,
                         int64_t cols, void* out, int out_dtype, int64_t ldo, void* stream) {
  if (rows < 0 || cols < 0 || cols % 4 != 0) return fail(S24_ERR_DIMENSION, "bad shape for decompress");
  if ((meta_ref == nullptr) == (meta_hw == nullptr)) return fail(S24_ERR_DIMENSION, "exactly one metadata form");
  if (meta_hw && cols % 128 != 0) return fail(S24_ERR_DIMENSION, "hw metadata needs cols %% 128 == 0");
  if (rows == 0 || cols == 0) return S24_OK;
  auto st = static_cast<cudaStream_t>(stream);
  const int g = grid_for(rows * cols / 4, 256);
  auto v = static_cast<const __nv_bfloat16*>(vals);
  if (out_dtype == S24_F32)
    k_decompress_token<float><<<g, 256, 0, st>>>(v, meta_ref, meta_hw, rows, cols, static_cast<float*>(out), ldo);
  else if (out_dtype == S24_BF16)
    k_decompress_token<__nv_bfloat16><<<g, 256, 0, st>>>(v, meta_ref, meta_hw, rows, cols,
                                                         static_cast<__nv_bfloat16*>(out), ldo);
  else
    return fail(S24_ERR_PRECISION, "unsupported dtype");
  return check_launch("k_decompress_token");
}

int s24_decompress_feature(const void* vals_t, const uint8_t* meta_ref, const uint8_t* meta_hw, int64_t rows,
                           int64_t cols, void* out, int out_dtype, int64_t ldo, void* stream) {
  if (rows < 0 || cols < 0 || rows % 4 != 0) return fail(S24_ERR_DIMENSION, "bad shape for decompress");
  if ((meta_ref == nullptr) == (meta_hw == nullptr)) return fail(S24_ERR_DIMENSION, "exactly one metadata form");
  if (meta_hw && rows % 128 != 0) return fail(S24_ERR_DIMENSION, "hw metadata needs rows %% 128 == 0");
  if (rows == 0 || cols == 0) return S24_OK;
  auto st = static_cast<cudaStream_t>(stream);
  const int g = grid_for(rows * cols / 4, 256);
  auto v = static_cast<const __nv_bfloat16*>(vals_t);
  if (out_dtype == S24_F32)
    k_decompress_feature<float><<<g, 256, 0, st>>>(v, meta_ref, meta_hw, rows, cols, static_cast<float*>(out), ldo);
  else if (out_dtype == S24_BF16)
    k_decompress_feature<__nv_bfloat16><<<g, 256, 0, st>>>(v, meta_ref, meta_hw, rows, cols,
                                                           static_cast<__nv_bfloat16*>(out), ldo);
  else
    return fail(S24_ERR_PRECISION, "unsupported dtype");
  return check_launch("k_decompress_feature");
}

int s24_meta_hw_to_ref(const uint8_t* meta_hw, int64_t rows, int64_t cols, uint8_t* meta_ref, void* stream) {
  if (rows < 0 || cols % 128 != 0) return fail(S24_ERR_DIMENSION, "hw metadata needs cols %% 128 == 0");
  if (rows == 0 || cols == 0) return S24_OK;
  k_meta_hw_to_ref<<<grid_for(rows * cols / 4, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(meta_hw, rows, cols,
                                                                                                 meta_ref);
  return check_launch("k_meta_hw_to_ref");
}

int s24_meta_ref_to_hw(const uint8_t* meta_ref, int64_t rows, int64_t cols, uint8_t* meta_hw, void* stream) {
  if (rows < 0 || cols % 128 != 0) return fail(S24_ERR_DIMENSION, "hw metadata needs cols %% 128 == 0");
  if (rows == 0 || cols == 0) return S24_OK;
  k_meta_ref_to_hw<<<grid_for(rows * cols / 16, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(meta_ref, rows,
                                                                                                  cols, meta_hw);
  return check_launch("k_meta_ref_to_hw");
}

int s24_gather_rows(const void* in, int64_t rows, int64_t row_bytes, int64_t ld_in_bytes, const int* src,
                    void* out, int64_t ld_out_bytes, void* stream) {
  if (rows < 0 || row_bytes < 0) return fail(S24_ERR_DIMENSION, "negative shape");
  if (row_bytes % 16 != 0 || ld_in_bytes % 16 != 0 || ld_out_bytes % 16 != 0 || !aligned16(in) || !aligned16(out))
    return fail(S24_ERR_DIMENSION, "row gather needs 16-byte aligned rows");
  if (rows == 0 || row_bytes == 0) return S24_OK;
  const int g = grid_for(rows * 32, 256);
  launch_high(k_gather_rows, dim3(g), dim3(256), static_cast<cudaStream_t>(stream), 0, static_cast<const uint8_t*>(in),
              static_cast<long long>(rows), static_cast<long long>(row_bytes), static_cast<long long>(ld_in_bytes), src,
              static_cast<uint8_t*>(out), static_cast<long long>(ld_out_bytes));
  return check_launch("k_gather_rows");
}

int s24_timestamp(unsigned long long* out, void* stream) {
  if (!out) return fail(S24_ERR_DIMENSION, "null output");
  k_timestamp<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(out);
  return check_launch("k_timestamp");
}

int s24_clock_probe(unsigned long long* out, int ctas, int64_t ns, void* stream) {
  if (!out || ctas < 1) return fail(S24_ERR_DIMENSION, "bad probe arguments");
  k_clock_probe<<<ctas, 32, 0, static_cast<cudaStream_t>(stream)>>>(out, static_cast<unsigned long long>(ns));
  return check_launch("k_clock_probe");
}

int s24_plan(const int* counts, int64_t h, int64_t n_sparse, int* sparse_idx, int* dense_idx, int* feat_pos,
             void* stream) {
  if (h < 0 || h > 65536) return fail(S24_ERR_DIMENSION, "plan supports 0 <= h <= 65536");
  if (n_sparse < 0 || n_sparse > h) return fail(S24_ERR_CONFIG, "n_sparse out of range");
  if (h == 0) return S24_OK;
  // (32 registers x 1024 threads and 8 KB of shared memory: the one CTA fits
  // next to a running 2:4 GEMM CTA, so the plan can overlap fwd.out)
  const int per = static_cast<int>((h + 1023) / 1024);
  const auto st = static_cast<cudaStream_t>(stream);
  const int hh = static_cast<int>(h), ns = static_cast<int>(n_sparse);
  if (per <= 4)
    k_plan<4><<<1, 1024, 0, st>>>(counts, hh, ns, sparse_idx, dense_idx, feat_pos);
  else if (per <= 8)
    k_plan<8><<<1, 1024, 0, st>>>(counts, hh, ns, sparse_idx, dense_idx, feat_pos);
  else if (per <= 16)
    k_plan<16><<<1, 1024, 0, st>>>(counts, hh, ns, sparse_idx, dense_idx, feat_pos);
  else if (per <= 32)
    k_plan<32><<<1, 1024, 0, st>>>(counts, hh, ns, sparse_idx, dense_idx, feat_pos);
  else
    k_plan<64><<<1, 1024, 0, st>>>(counts, hh, ns, sparse_idx, dense_idx, feat_pos);
  return check_launch("k_plan");
}

int s24_feature_split_x(const void* vals, const uint8_t* meta_hw, int64_t n, int64_t h, const int* feat_pos,
                        int64_t n_sparse, int64_t n_dense, void* vs, uint8_t* es, int operand_nonneg,
                        const unsigned long long* nan_flag, void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  K4Args pa;
  int rc = k4_prepare(vals, meta_hw, n, h, feat_pos, n_sparse, n_dense, vs, es, nullptr, st, &pa, 2 * n_dense);
  if (rc) return rc;
  if (!vals || !meta_hw || !feat_pos) return fail(S24_ERR_DIMENSION, "null operand");
  if (!aligned16(vals) || !aligned16(vs) || !aligned16(meta_hw))
    return fail(S24_ERR_DIMENSION, "operands must be 16-byte aligned");
  if (n == 0 || h == 0) return S24_OK;
  K4xArgs a{static_cast<const __nv_bfloat16*>(vals), meta_hw, static_cast<int>(n), static_cast<int>(h), feat_pos,
            static_cast<int>(2 * n_dense), static_cast<__nv_bfloat16*>(vs), es, nan_flag};
  const dim3 grid(static_cast<unsigned>(h / (16 * K4X_WARPS)), static_cast<unsigned>(n / 128));
  (operand_nonneg ? k_feature_split_x<true> : k_feature_split_x<false>)<<<grid, 32 * K4X_WARPS, 0, st>>>(a);
  return check_launch("k_feature_split_x");
}

int s24_feature_split(const void* vals, const uint8_t* meta_hw, int64_t n, int64_t h, const int* feat_pos,
                      int64_t n_sparse, int64_t n_dense, void* vs, uint8_t* es, void* vd,
                      unsigned long long* stats, int operand_nonneg, int64_t pair_rows, void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  K4Args a;
  int rc = k4_prepare(vals, meta_hw, n, h, feat_pos, n_sparse, n_dense, vs, es, vd, st, &a, pair_rows);
  if (rc) return rc;
  if (n == 0 || h == 0) return S24_OK;
  a.stats = stats;
  a.nonneg = operand_nonneg ? 1 : 0;
  dim3 grid(static_cast<unsigned>(h / 128), static_cast<unsigned>(n / 128));
  if (stats)
    (a.nonneg ? k_feature_split<true, true> : k_feature_split<true, false>)<<<grid, 256, 0, st>>>(a);
  else
    (a.nonneg ? k_feature_split<false, true> : k_feature_split<false, false>)<<<grid, 256, 0, st>>>(a);
  return check_launch("k_feature_split");
}

}  // extern "C"
