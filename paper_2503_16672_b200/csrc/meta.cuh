// 2:4 selection rule and the two metadata layouts.
//
// Selection (ref: pkg/src/srelu24/sparse24.py:72-77, `_top2_stable`): in every
// aligned group of 4 keep the 2 largest |x|; ties go to the lower in-group
// index; zeros rank last, so a group with < 2 nonzeros is padded with its
// lowest-index zero positions. Kept positions are stored ascending (i0 < i1).
// We restate it as a rank test: element i is kept iff fewer than two elements
// beat it, where j beats i when |x_j| > |x_i| or (|x_j| == |x_i| and j < i).
// NaN is ranked below everything (numpy's argsort puts NaN keys last).
//
// Reference layout ("ref"): uint8 [rows, cols/4, 2] holding (i0, i1) per group
// (token orientation, ref: sparse24.py:30-47).
//
// Hardware layout ("hw"): the operand-E format tcgen05.mma.sp.kind::f16 reads
// from TMEM. Per group one nibble i0 | i1 << 2 (the same packing as the
// reference's S24C files, sparse24.py:240). Nibbles are arranged in atoms of
// 128 rows x 128 logical K (2048 bytes): atom (rb, kb) starts at byte
// (rb * (K/128) + kb) * 2048. Inside an atom, the 16-bit halfword that holds
// the 4 nibbles of row r, logical columns [16q, 16q+16) sits at byte
//     2*m1 + 4*k2 + 16*m0 + 128*k1 + 256*m2
// with m0 = r&7, m1 = (r>>3)&1, m2 = r>>4, k1 = q&1, k2 = q>>1 (nibble j of the
// halfword = group j of those 16 columns). Each atom is 128 contiguous rows of
// 16 bytes, which tcgen05.cp.128x128b copies one-to-one onto 128 TMEM lanes x
// 4 columns; TMEM column c then feeds the K=32 MMA step c of that atom.
#pragma once
#include <cstdint>

namespace s24 {

__host__ __device__ __forceinline__ uint32_t meta_atom_halfword_byte(uint32_t r, uint32_t q) {
  const uint32_t m0 = r & 7u, m1 = (r >> 3) & 1u, m2 = r >> 4;
  const uint32_t k1 = q & 1u, k2 = q >> 1;
  return 2u * m1 + 4u * k2 + 16u * m0 + 128u * k1 + 256u * m2;
}

// byte offset of the halfword for (row, 16-column chunk `col16`) in a
// hw-layout buffer whose logical K extent is `kdim` (multiple of 128)
__host__ __device__ __forceinline__ uint64_t meta_hw_halfword_offset(uint64_t row, uint64_t col16, uint64_t kdim) {
  const uint64_t rb = row >> 7, kb = col16 >> 3;
  return (rb * (kdim >> 7) + kb) * 2048u +
         meta_atom_halfword_byte(static_cast<uint32_t>(row & 127u), static_cast<uint32_t>(col16 & 7u));
}

__host__ __device__ __forceinline__ uint64_t meta_hw_bytes(uint64_t rows_padded, uint64_t kdim) {
  return rows_padded * kdim / 8u;
}

// rank-based top-2 over one group; returns the 4-bit keep mask
__device__ __forceinline__ uint32_t top2_keep_mask(float x0, float x1, float x2, float x3) {
  const float k0 = (x0 != x0) ? -1.f : fabsf(x0);
  const float k1 = (x1 != x1) ? -1.f : fabsf(x1);
  const float k2 = (x2 != x2) ? -1.f : fabsf(x2);
  const float k3 = (x3 != x3) ? -1.f : fabsf(x3);
  const uint32_t b01 = k0 >= k1, b02 = k0 >= k2, b03 = k0 >= k3;
  const uint32_t b12 = k1 >= k2, b13 = k1 >= k3, b23 = k2 >= k3;
  const uint32_t r0 = 3u - b01 - b02 - b03;
  const uint32_t r1 = b01 + 2u - b12 - b13;
  const uint32_t r2 = b02 + b12 + 1u - b23;
  const uint32_t r3 = b03 + b13 + b23;
  return (r0 < 2u ? 1u : 0u) | (r1 < 2u ? 2u : 0u) | (r2 < 2u ? 4u : 0u) | (r3 < 2u ? 8u : 0u);
}

// keep mask -> (i0, i1) nibble
__device__ __forceinline__ uint32_t keep_to_nibble(uint32_t keep) {
  const uint32_t i0 = __ffs(keep) - 1u;
  const uint32_t i1 = 31u - __clz(keep);
  return i0 | (i1 << 2);
}

// The same rule on 0 / 0xffffffff masks (the fused epilogues' form): i beats
// j (i < j) iff key_i >= key_j; kept iff it beats two of the other three
// (a bitwise majority); the kept values are picked with bitwise selects.
// fge_mask compiles to one compare (+ select) per pair.
__device__ __forceinline__ uint32_t fge_mask(float a, float b) {
  uint32_t r;
  asm("set.ge.u32.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b));
  return r;
}

__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) { return (a & b) | (a & c) | (b & c); }
__device__ __forceinline__ uint32_t bsel(uint32_t m, uint32_t a, uint32_t b) { return (a & m) | (b & ~m); }

// keep bits (4-bit mask with two bits set) -> nibble i0 | i1 << 2
constexpr unsigned long long kKeepNibbleLut = 0x000E0DC009804000ull;

__device__ __forceinline__ uint32_t keep_nibble(uint32_t kb) {
  return static_cast<uint32_t>(kKeepNibbleLut >> (4u * kb)) & 0xFu;
}

__device__ __forceinline__ float sel4(float x0, float x1, float x2, float x3, uint32_t i) {
  float r = x0;
  r = (i == 1u) ? x1 : r;
  r = (i == 2u) ? x2 : r;
  r = (i == 3u) ? x3 : r;
  return r;
}

}  // namespace s24
