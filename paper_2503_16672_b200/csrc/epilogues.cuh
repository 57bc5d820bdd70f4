// Epilogue functors for gemm_kernel. Each call sees one 32-column chunk of one
// accumulator row (fp32, straight out of TMEM); all 32 lanes of the warp call
// in lock-step (lane == row within the warp's 32-row slab).
#pragma once
#include <cuda_bf16.h>
#include "meta.cuh"
#include "ptx.cuh"

namespace s24 {

struct NoState {};

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}


// e4m3 GEMMs: v = (sr * col_scale[j]) * acc (the reference's order), the 32
// column scales of the chunk read as 8 broadcast 16-byte loads
__device__ __forceinline__ void scale_chunk(const float* cs, float sr, const float (&acc)[32], float (&v)[32]) {
#pragma unroll
  for (int i = 0; i < 32; i += 4) {
    const float4 c = __ldg(reinterpret_cast<const float4*>(cs + i));
    v[i] = __fmul_rn(__fmul_rn(sr, c.x), acc[i]);
    v[i + 1] = __fmul_rn(__fmul_rn(sr, c.y), acc[i + 1]);
    v[i + 2] = __fmul_rn(__fmul_rn(sr, c.z), acc[i + 2]);
    v[i + 3] = __fmul_rn(__fmul_rn(sr, c.w), acc[i + 3]);
  }
}

__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}


// relu that keeps NaN (numpy's maximum(y, 0), ref ffn.py:167-169)
__device__ __forceinline__ float relu_nan(float x) {
  float r;
  asm("max.NaN.f32 %0, %1, 0f00000000;" : "=f"(r) : "f"(x));
  return r;
}

// any NaN among the 16 bf16 halves of 8 packed words (bf16 NaN: |bits| > 0x7F80)
__device__ __forceinline__ bool any_nan_bf16x2(const uint32_t (&w)[8]) {
  uint32_t t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) t |= (w[i] & 0x7FFF7FFFu) + 0x007F007Fu;
  return (t & 0x80008000u) != 0u;
}

// 32x32 bit-matrix transpose across the warp: on return, bit l of lane i's
// word is bit i of lane l's input word.
__device__ __forceinline__ uint32_t warp_bit_transpose(uint32_t x, uint32_t lane) {
  const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int j = 16 >> s;
    const uint32_t m = masks[s];
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
    x = (lane & j) ? (((y >> j) & m) | (x & ~m)) : ((x & m) | ((y << j) & ~m));
  }
  return x;
}

// ---------------------------------------------------------------------------
// Plain store: D[row_map(row), col] (or transposed D[col, row_map(row)]),
// bf16 or fp32. Used for fwd.out / bwd.d_x (row_map = inverse permutation),
// the dense twins, and the split weight-gradient GEMMs (row_map = feature
// index list of the partition, transposed for dW1).
// SCALED: e4m3 GEMMs, D = (row_scale[row] * col_scale[col]) * acc (the
// reference's order, ref matcore.py:257-258), applied before any pair sum.
template <typename OutT, bool SCALED = false>
struct EpiStore {
  struct Params {
    OutT* out;
    long long ldo;
    const int* row_map;  // nullable
    int transposed;      // 1: out[col * ldo + r]
    int n_rows_valid;    // rows >= this are padding (skip)
    const int* row_valid;  // nullable: skip rows with row_valid[row] < 0
    long long split_stride;  // split-K: partial of split ks goes to out + ks * split_stride
    int pair_rows;           // rows < pair_rows come in (even, odd) pairs: their sum is the even row's
                             // output (a dense feature stored as two 2:4 rows, see k4.cuh)
    const float* row_scale;  // SCALED only: [M] per GEMM row
    const float* col_scale;  // SCALED only: [N]
  };
  struct State {
    long long split_off;
  };
  static constexpr bool kUnroll = false;
  __device__ static void init(const Params&, State& s) { s.split_off = 0; }
  __device__ static void prefetch(const Params& p, State& s, int, bool, int, int ks) {
    s.split_off = ks * p.split_stride;
  }
  __device__ static void finish(const Params&, State&, uint32_t) {}
  __device__ static void chunk(const Params& p, State& s, int row, bool row_ok, int col0, int,
                               const float (&v_in)[32], uint32_t lane) {
    float v[32];
    if constexpr (SCALED) {
      const float sr = row_ok ? __ldg(p.row_scale + row) : 0.f;
      scale_chunk(p.col_scale + col0, sr, v_in, v);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = v_in[i];
    }
    // (warp-uniform test: every lane of the warp calls chunk)
    if (__any_sync(0xffffffffu, row < p.pair_rows)) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float o = __shfl_down_sync(0xffffffffu, v[i], 1);
        if (row < p.pair_rows) v[i] += o;
      }
      if (row < p.pair_rows && (row & 1)) return;  // added into the even row
    }
    (void)lane;
    if (!row_ok || row >= p.n_rows_valid) return;
    if (p.row_valid && p.row_valid[row] < 0) return;
    const long long r = (p.row_map ? p.row_map[row] : row);
    OutT* const out = p.out + s.split_off;
    if (p.transposed) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        if constexpr (sizeof(OutT) == 4)
          out[static_cast<long long>(col0 + i) * p.ldo + r] = v[i];
        else
          out[static_cast<long long>(col0 + i) * p.ldo + r] = __float2bfloat16_rn(v[i]);
      }
    } else {
      OutT* dst = out + r * p.ldo + col0;
      // whole 32-byte sectors per store (st_global_32b)
      if constexpr (sizeof(OutT) == 4) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          const uint32_t w[8] = {__float_as_uint(v[i]),     __float_as_uint(v[i + 1]), __float_as_uint(v[i + 2]),
                                 __float_as_uint(v[i + 3]), __float_as_uint(v[i + 4]), __float_as_uint(v[i + 5]),
                                 __float_as_uint(v[i + 6]), __float_as_uint(v[i + 7])};
          st_global_32b(dst + i, w);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; i += 16) {
          const uint32_t w[8] = {pack_bf16x2(v[i], v[i + 1]),         pack_bf16x2(v[i + 2], v[i + 3]),
                                 pack_bf16x2(v[i + 4], v[i + 5]),     pack_bf16x2(v[i + 6], v[i + 7]),
                                 pack_bf16x2(v[i + 8], v[i + 9]),     pack_bf16x2(v[i + 10], v[i + 11]),
                                 pack_bf16x2(v[i + 12], v[i + 13]), pack_bf16x2(v[i + 14], v[i + 15])};
          st_global_32b(dst + i, w);
        }
      }
    }
  }
};

// ---------------------------------------------------------------------------
// K1: fwd.pre_act epilogue. y = acc; a = relu(y)^2 (fp32, ref ffn.py:167-169);
// token-wise top-2 per group of 4 features (ref sparse24.py:80-93) on the fp32
// a; emits bf16 kept values [M, N/2], hw metadata, per-feature nonzero counts
// of the pre-sparsify a (ref splitgemm.py:28-30, ffn.py:320-322) and the
// nonzeros before/after totals (ref sparse24.py:60-69). The dense activation
// never leaves registers. Optional debug dump of y (fp32) for parity tests.
// Selection: pairwise FSET masks b_ij (i < j: i beats j iff k_i >= k_j, ties
// to the lower index); "kept iff it beats two of the other three" is a
// bitwise majority; values are picked with bitwise selects.
// Non-finite values follow the reference's numpy semantics: relu keeps NaN
// (np.maximum), NaN counts as a nonzero (np.count_nonzero) and ranks below
// every number including zero (np.argsort puts NaN keys last): the selection
// key is max(a, -1), which maps NaN to -1 and leaves a >= 0 unchanged. A kept
// NaN raises stats[2] so that the feature-wise split ranks NaN-aware.
// F8 (e4m3 K1, ref ffn.py:305 + :330-341): y = (row_scale[r] * col_scale[c]) * acc;
// the kept values go out as fp32 (vals32) with a per-row running max of the
// kept |a| (row_amax, float bits, atomicMax) for the per-token quantization
// that follows (fp8.cu); the bf16 vals are not written.
template <bool F8>
struct EpiFwd1T {
  struct Params {
    __nv_bfloat16* vals;  // [Mpad, N/2]
    uint8_t* meta;        // hw layout, K = N
    int* counts;          // [N], accumulated (nullable)
    unsigned long long* stats;  // [3] nnz before / after, accumulated; [2] != 0: a kept value is NaN
    float* y_dbg;         // nullable [M, N]
    int N;
    const float* row_scale;  // F8 only
    const float* col_scale;
    float* vals32;           // F8 only: [Mpad, N/2]
    unsigned* row_amax;      // F8 only: [Mpad], zeroed before the launch
  };
  struct State {
    unsigned long long before, after;
    uint32_t nan_kept;
    uint32_t mq[4];       // metadata halfwords (k1 = 0 | k1 = 1 << 16) of the atom's chunks k2 = 0..3
  };
  static constexpr bool kUnroll = true;  // (mq is indexed by the chunk)
  // The warp's run of chunks covers whole 128-column metadata atoms (a
  // multiple of 4 chunks starting at a multiple of 4): the 8 halfwords a row
  // has in an atom are gathered across lane pairs (rows r, r ^ 8 interleave
  // per 4-byte word) and written as one 16-byte store per lane, whole
  // sectors, instead of two 2-byte stores per chunk.
  __device__ static void meta_flush(const Params& p, const State& s, int row, bool any_ok, int col0, uint32_t lane) {
    const bool hi = (lane & 8u) != 0u;  // m1 = 1: this lane writes the k1 = 1 half of the pair
    uint32_t w[4];
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) {
      const uint32_t lo16 = s.mq[k2] & 0xFFFFu, hi16 = s.mq[k2] >> 16;
      const uint32_t recv = __shfl_xor_sync(0xffffffffu, hi ? lo16 : hi16, 8);
      w[k2] = hi ? (recv | (hi16 << 16)) : (lo16 | (recv << 16));
    }
    if (!any_ok) return;  // (warp-uniform) every row of the warp is padding beyond the buffer's rows
    const uint64_t off = meta_hw_halfword_offset(static_cast<uint64_t>(row) & ~8ull,
                                                 static_cast<uint64_t>(col0 / 16) + (hi ? 1u : 0u), p.N);
    st_global_v4(p.meta + off, w[0], w[1], w[2], w[3]);
  }
  __device__ static void init(const Params&, State& s) {
    s.before = s.after = 0;
    s.nan_kept = 0;
  }
  __device__ static void prefetch(const Params&, State&, int, bool, int, int) {}
  __device__ static void finish(const Params& p, State& s, uint32_t lane) {
    const unsigned long long b = warp_sum_u64(s.before), a = warp_sum_u64(s.after);
    const bool nan_kept = __any_sync(0xffffffffu, s.nan_kept != 0u);
    if (lane == 0 && p.stats) {
      atomicAdd(p.stats, b);
      atomicAdd(p.stats + 1, a);
      if (nan_kept) atomicOr(p.stats + 2, 1ull);
    }
  }
  __device__ static void chunk(const Params& p, State& s, int row, bool row_ok, int col0, int ci,
                               const float (&v_in)[32], uint32_t lane) {
    float v[32];
    if constexpr (F8) {
      const float sr = row_ok ? __ldg(p.row_scale + row) : 0.f;
      scale_chunk(p.col_scale + col0, sr, v_in, v);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = v_in[i];
    }
    float a[32], k[32];
    uint32_t nz = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float r = relu_nan(v[i]);
      a[i] = __fmul_rn(r, r);
      k[i] = fmaxf(a[i], -1.f);
      nz |= (a[i] != 0.f ? 1u : 0u) << i;
    }
    // rows >= M read TMA zero fill, so y = 0 there -- unless B holds NaN / Inf
    // (0 * Inf = NaN): they never count
    if (!row_ok) nz = 0u;
    // per-feature counts over the warp's 32 rows: transpose the nonzero bit
    // matrix so lane i holds column i, then popcount
    if (p.counts) {
      const uint32_t col_bits = warp_bit_transpose(nz, lane);
      if (col_bits) atomicAdd(p.counts + col0 + lane, __popc(col_bits));
    }
    uint32_t packed[8];
    float kept[16];
    uint32_t m16[2] = {0u, 0u};
    uint32_t keep32 = 0;
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const float k0 = k[4 * g], k1 = k[4 * g + 1], k2 = k[4 * g + 2], k3 = k[4 * g + 3];
      const uint32_t b01 = fge_mask(k0, k1), b02 = fge_mask(k0, k2), b03 = fge_mask(k0, k3);
      const uint32_t b12 = fge_mask(k1, k2), b13 = fge_mask(k1, k3), b23 = fge_mask(k2, k3);
      const uint32_t K0 = maj3(b01, b02, b03), K1 = maj3(~b01, b12, b13);
      const uint32_t K2 = maj3(~b02, ~b12, b23), K3 = maj3(~b03, ~b13, ~b23);
      const uint32_t kb = (K0 & 1u) | (K1 & 2u) | (K2 & 4u) | (K3 & 8u);
      const uint32_t u0 = __float_as_uint(a[4 * g]), u1 = __float_as_uint(a[4 * g + 1]),
                     u2 = __float_as_uint(a[4 * g + 2]), u3 = __float_as_uint(a[4 * g + 3]);
      const float v0 = __uint_as_float(bsel(K0, u0, bsel(K1, u1, u2)));  // first kept
      const float v1 = __uint_as_float(bsel(K3, u3, bsel(K2, u2, u1)));  // second kept
      if constexpr (F8) {
        kept[2 * g] = v0;
        kept[2 * g + 1] = v1;
      } else {
        packed[g] = pack_bf16x2(v0, v1);
      }
      m16[g >> 2] |= keep_nibble(kb) << (4 * (g & 3));
      keep32 |= kb << (4 * g);
    }
    // padding rows inside the buffer (row >= M) get the (0, 1) selectors of
    // an all-zero group, 0x4444: the value the host pre-fills them with
    s.mq[ci & 3] = m16[0] | (m16[1] << 16);
    if ((ci & 3) == 3) meta_flush(p, s, row, __any_sync(0xffffffffu, row_ok), col0 - 96, lane);
    if (!row_ok) return;
    s.before += __popc(nz);
    s.after += __popc(nz & keep32);
    if constexpr (F8) {
      float* dst = p.vals32 + static_cast<long long>(row) * (p.N / 2) + col0 / 2;
      float mx = 0.f;
#pragma unroll
      for (int i = 0; i < 16; i += 8) {
        const uint32_t w[8] = {__float_as_uint(kept[i]),     __float_as_uint(kept[i + 1]), __float_as_uint(kept[i + 2]),
                               __float_as_uint(kept[i + 3]), __float_as_uint(kept[i + 4]), __float_as_uint(kept[i + 5]),
                               __float_as_uint(kept[i + 6]), __float_as_uint(kept[i + 7])};
        st_global_32b(dst + i, w);
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) mx = fmaxf(mx, kept[i]);
      if (mx > 0.f) atomicMax(p.row_amax + row, __float_as_uint(mx));  // a >= 0: uint order = float order
    } else {
      s.nan_kept |= any_nan_bf16x2(packed) ? 1u : 0u;
      __nv_bfloat16* dst = p.vals + static_cast<long long>(row) * (p.N / 2) + col0 / 2;
      st_global_32b(dst, packed);
    }
    if (p.y_dbg) {
      float* y = p.y_dbg + static_cast<long long>(row) * p.N + col0;
#pragma unroll
      for (int i = 0; i < 32; i += 4)
        st_global_v4(y + i, __float_as_uint(v[i]), __float_as_uint(v[i + 1]), __float_as_uint(v[i + 2]),
                     __float_as_uint(v[i + 3]));
    }
  }
};

using EpiFwd1 = EpiFwd1T<false>;

// ---------------------------------------------------------------------------
// K3: bwd.d_act epilogue. G = acc (= dY_c . W2^T). On the forward keep pattern
// only (ref ffn.py:415-417 + sparse24.py:138-154, exact by construction):
//   g_pre = G * 2 * relu(y1),  relu(y1) recovered as sqrt(a) from the cached
// compressed activation a = relu(y1)^2. Output: compressed g_pre [M, N/2] on
// the forward metadata (which is reused as-is for the dX sparse GEMM).
// The warp's act values (CPW chunks x 32 B / row) and metadata rows are
// prefetched into registers before the accumulator wait, so their latency
// hides under the MMA.
// F8 (fp8_backward, ref ffn.py:395): G = (row_scale[r] * col_scale[c]) * acc.
template <bool F8>
struct EpiBwd1T {
  struct Params {
    const __nv_bfloat16* act_vals;  // [Mpad, N/2]
    const uint8_t* meta;            // hw layout, K = N
    __nv_bfloat16* gvals;           // [Mpad, N/2] out
    int N;
    const float* row_scale;         // F8 only
    const float* col_scale;
  };
  static constexpr int CPW = 4;  // chunks per epilogue warp (BN = 256, 8 epilogue warps)
  static constexpr bool kUnroll = true;
  struct State {
    uint4 act[2 * CPW];  // 8 kept values per uint4 = 16 logical columns
    uint4 meta[2];       // the row's two 16-byte metadata rows (k1 = 0, 1) of its atom
  };
  __device__ static void init(const Params&, State&) {}
  __device__ static void finish(const Params&, State&, uint32_t) {}
  __device__ static void prefetch(const Params& p, State& s, int row, bool row_ok, int col_first, int) {
    if (!row_ok || col_first >= p.N) return;
    const uint4* a =
        reinterpret_cast<const uint4*>(p.act_vals + static_cast<long long>(row) * (p.N / 2) + col_first / 2);
#pragma unroll
    for (int i = 0; i < 2 * CPW; ++i) s.act[i] = a[i];
    const uint32_t r = static_cast<uint32_t>(row) & 127u;
    const uint8_t* base =
        p.meta + meta_hw_halfword_offset(row, col_first / 16, p.N) - meta_atom_halfword_byte(r, 0);
    const uint32_t row16 = 16u * (r & 7u) + 256u * (r >> 4);
    s.meta[0] = *reinterpret_cast<const uint4*>(base + row16);
    s.meta[1] = *reinterpret_cast<const uint4*>(base + row16 + 128);
  }
  __device__ static uint32_t word(const uint4& v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }
  __device__ static void chunk(const Params& p, State& s, int row, bool row_ok, int col0, int ci,
                               const float (&v_in)[32], uint32_t) {
    if (!row_ok) return;
    float v[32];
    if constexpr (F8) {
      const float sr = __ldg(p.row_scale + row);
      scale_chunk(p.col_scale + col0, sr, v_in, v);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = v_in[i];
    }
    const uint32_t m1 = (static_cast<uint32_t>(row) >> 3) & 1u;
    // the chunk's two 16-column quads (k1 = 0, 1) sit in word k2 = ci of the atom rows
    const uint32_t w0 = word(s.meta[0], ci & 3), w1 = word(s.meta[1], ci & 3);
    const uint32_t m16[2] = {(w0 >> (16 * m1)) & 0xFFFFu, (w1 >> (16 * m1)) & 0xFFFFu};
    const uint32_t aw[8] = {s.act[2 * ci].x,     s.act[2 * ci].y,     s.act[2 * ci].z,     s.act[2 * ci].w,
                            s.act[2 * ci + 1].x, s.act[2 * ci + 1].y, s.act[2 * ci + 1].z, s.act[2 * ci + 1].w};
    uint32_t packed[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const uint32_t nib = (m16[g >> 2] >> (4 * (g & 3))) & 0xFu;
      const float g0 = sel4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3], nib & 3u);
      const float g1 = sel4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3], nib >> 2);
      const float a0 = __uint_as_float(aw[g] << 16), a1 = __uint_as_float(aw[g] & 0xFFFF0000u);
      packed[g] = pack_bf16x2(g0 * (2.f * sqrt_approx(a0)), g1 * (2.f * sqrt_approx(a1)));
    }
    __nv_bfloat16* dst = p.gvals + static_cast<long long>(row) * (p.N / 2) + col0 / 2;
    st_global_32b(dst, packed);
  }
};

using EpiBwd1 = EpiBwd1T<false>;

// ---------------------------------------------------------------------------
// Dense-mode twins. fwd: act = relu(y)^2 stored dense bf16 (ref ffn.py:314).
struct EpiRelu2 {
  struct Params {
    __nv_bfloat16* act;
    long long ld;
  };
  using State = NoState;
  static constexpr bool kUnroll = false;
  __device__ static void init(const Params&, State&) {}
  __device__ static void prefetch(const Params&, State&, int, bool, int, int) {}
  __device__ static void finish(const Params&, State&, uint32_t) {}
  __device__ static void chunk(const Params& p, State&, int row, bool row_ok, int col0, int,
                               const float (&v)[32], uint32_t) {
    if (!row_ok) return;
    float a[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float r = relu_nan(v[i]);
      a[i] = __fmul_rn(r, r);
    }
    __nv_bfloat16* dst = p.act + static_cast<long long>(row) * p.ld + col0;
#pragma unroll
    for (int i = 0; i < 32; i += 16) {
      const uint32_t w[8] = {pack_bf16x2(a[i], a[i + 1]),         pack_bf16x2(a[i + 2], a[i + 3]),
                             pack_bf16x2(a[i + 4], a[i + 5]),     pack_bf16x2(a[i + 6], a[i + 7]),
                             pack_bf16x2(a[i + 8], a[i + 9]),     pack_bf16x2(a[i + 10], a[i + 11]),
                             pack_bf16x2(a[i + 12], a[i + 13]), pack_bf16x2(a[i + 14], a[i + 15])};
      st_global_32b(dst + i, w);
    }
  }
};

// bwd: g_pre = G * 2 * sqrt(act), dense (ref ffn.py:415 with act_squared_relu_grad
// :172-173). The warp's act run (CPW chunks x 64 B / row) is prefetched into
// registers before the accumulator wait.
struct EpiDact {
  struct Params {
    const __nv_bfloat16* act;
    long long ld_act;
    __nv_bfloat16* gpre;
    long long ld_g;
    int N;
  };
  static constexpr int CPW = 4;
  static constexpr bool kUnroll = true;
  struct State {
    uint4 buf[CPW][4];
  };
  __device__ static void init(const Params&, State&) {}
  __device__ static void finish(const Params&, State&, uint32_t) {}
  __device__ static void prefetch(const Params& p, State& s, int row, bool row_ok, int col_first, int) {
    if (!row_ok) return;
#pragma unroll
    for (int c = 0; c < CPW; ++c) {
      if (col_first + 32 * c < p.N) {
        const uint4* src =
            reinterpret_cast<const uint4*>(p.act + static_cast<long long>(row) * p.ld_act + col_first + 32 * c);
#pragma unroll
        for (int i = 0; i < 4; ++i) s.buf[c][i] = src[i];
      }
    }
  }
  __device__ static void chunk(const Params& p, State& s, int row, bool row_ok, int col0, int ci,
                               const float (&v)[32], uint32_t) {
    if (!row_ok) return;
    __nv_bfloat16* dst = p.gpre + static_cast<long long>(row) * p.ld_g + col0;
    uint32_t o[16];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t ww[4] = {s.buf[ci][i].x, s.buf[ci][i].y, s.buf[ci][i].z, s.buf[ci][i].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float a0 = __uint_as_float(ww[j] << 16), a1 = __uint_as_float(ww[j] & 0xFFFF0000u);
        o[4 * i + j] = pack_bf16x2(v[8 * i + 2 * j] * (2.f * sqrt_approx(a0)),
                                   v[8 * i + 2 * j + 1] * (2.f * sqrt_approx(a1)));
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t w[8] = {o[8 * h], o[8 * h + 1], o[8 * h + 2], o[8 * h + 3],
                             o[8 * h + 4], o[8 * h + 5], o[8 * h + 6], o[8 * h + 7]};
      st_global_32b(dst + 16 * h, w);
    }
  }
};

}  // namespace s24
