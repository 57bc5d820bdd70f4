// Epilogue functors for gemm_kernel. Each sees one 32-column chunk of one
// accumulator row (fp32, straight out of TMEM) per call; all 32 lanes of the
// warp call in lock-step (lane == row within the warp's 32-row slab).
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

// ---------------------------------------------------------------------------
// Plain store: D[row_map(row), col] (or transposed D[col, row_map(row)]),
// bf16 or fp32. Used for fwd.out / bwd.d_x (row_map = inverse permutation),
// the dense twins, and the split weight-gradient GEMMs (row_map = feature
// index list of the partition, transposed for dW1).
template <typename OutT>
struct EpiStore {
  struct Params {
    OutT* out;
    long long ldo;
    const int* row_map;  // nullable
    int transposed;      // 1: out[col * ldo + r]
    int n_rows_valid;    // rows >= this are padding (skip)
  };
  using State = NoState;
  static constexpr bool kUnroll = false;
  __device__ static void init(const Params&, State&) {}
  __device__ static void prefetch(const Params&, State&, int, bool, int) {}
  __device__ static void finish(const Params&, State&, uint32_t) {}
  __device__ static void chunk(const Params& p, State&, int row, bool row_ok, int col0, int c,
                               const float (&v)[32], uint32_t) {
    if (!row_ok || row >= p.n_rows_valid) return;
    const long long r = p.row_map ? p.row_map[row] : row;
    if (p.transposed) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        if constexpr (sizeof(OutT) == 4)
          p.out[static_cast<long long>(col0 + i) * p.ldo + r] = v[i];
        else
          p.out[static_cast<long long>(col0 + i) * p.ldo + r] = __float2bfloat16_rn(v[i]);
      }
    } else {
      OutT* dst = p.out + r * p.ldo + col0;
      if constexpr (sizeof(OutT) == 4) {
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          st_global_v4(dst + i, __float_as_uint(v[i]), __float_as_uint(v[i + 1]), __float_as_uint(v[i + 2]),
                       __float_as_uint(v[i + 3]));
      } else {
#pragma unroll
        for (int i = 0; i < 32; i += 8)
          st_global_v4(dst + i, pack_bf16x2(v[i], v[i + 1]), pack_bf16x2(v[i + 2], v[i + 3]),
                       pack_bf16x2(v[i + 4], v[i + 5]), pack_bf16x2(v[i + 6], v[i + 7]));
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
struct EpiFwd1 {
  struct Params {
    __nv_bfloat16* vals;  // [Mpad, N/2]
    uint8_t* meta;        // hw layout, K = N
    int* counts;          // [N], accumulated (nullable)
    unsigned long long* stats;  // [2] nnz before / after, accumulated
    float* y_dbg;         // nullable [M, N]
    int N;
  };
  struct State {
    unsigned long long before, after;
  };
  static constexpr bool kUnroll = false;
  __device__ static void init(const Params&, State& s) { s.before = s.after = 0; }
  __device__ static void prefetch(const Params&, State&, int, bool, int) {}
  __device__ static void finish(const Params& p, State& s, uint32_t lane) {
    const unsigned long long b = warp_sum_u64(s.before), a = warp_sum_u64(s.after);
    if (lane == 0 && p.stats) {
      atomicAdd(p.stats, b);
      atomicAdd(p.stats + 1, a);
    }
  }
  __device__ static void chunk(const Params& p, State& s, int row, bool row_ok, int col0, int c,
                               const float (&v)[32], uint32_t lane) {
    float a[32];
    uint32_t nz = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float r = fmaxf(v[i], 0.f);
      a[i] = row_ok ? __fmul_rn(r, r) : 0.f;
      nz |= (a[i] != 0.f ? 1u : 0u) << i;
    }
    // per-feature counts: column i of this chunk over the warp's 32 rows
    if (p.counts) {
      uint32_t my = 0;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const uint32_t b = __ballot_sync(0xffffffffu, (nz >> i) & 1u);
        my = (lane == static_cast<uint32_t>(i)) ? static_cast<uint32_t>(__popc(b)) : my;
      }
      if (my) atomicAdd(p.counts + col0 + lane, static_cast<int>(my));
    }
    if (!row_ok) return;
    s.before += __popc(nz);
    uint32_t packed[8];
    uint32_t m16[2] = {0u, 0u};
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const uint32_t keep = top2_keep_mask(a[4 * g], a[4 * g + 1], a[4 * g + 2], a[4 * g + 3]);
      const uint32_t nib = keep_to_nibble(keep);
      const float v0 = sel4(a[4 * g], a[4 * g + 1], a[4 * g + 2], a[4 * g + 3], nib & 3u);
      const float v1 = sel4(a[4 * g], a[4 * g + 1], a[4 * g + 2], a[4 * g + 3], nib >> 2);
      s.after += (v0 != 0.f) + (v1 != 0.f);
      packed[g] = pack_bf16x2(v0, v1);
      m16[g >> 2] |= nib << (4 * (g & 3));
    }
    __nv_bfloat16* dst = p.vals + static_cast<long long>(row) * (p.N / 2) + col0 / 2;
    st_global_v4(dst, packed[0], packed[1], packed[2], packed[3]);
    st_global_v4(dst + 8, packed[4], packed[5], packed[6], packed[7]);
    uint16_t* mh = reinterpret_cast<uint16_t*>(p.meta);
    mh[meta_hw_halfword_offset(row, col0 / 16, p.N) / 2] = static_cast<uint16_t>(m16[0]);
    mh[meta_hw_halfword_offset(row, col0 / 16 + 1, p.N) / 2] = static_cast<uint16_t>(m16[1]);
    if (p.y_dbg) {
      float* y = p.y_dbg + static_cast<long long>(row) * p.N + col0;
#pragma unroll
      for (int i = 0; i < 32; i += 4)
        st_global_v4(y + i, __float_as_uint(v[i]), __float_as_uint(v[i + 1]), __float_as_uint(v[i + 2]),
                     __float_as_uint(v[i + 3]));
    }
  }
};

// ---------------------------------------------------------------------------
// K3: bwd.d_act epilogue. G = acc (= dY_c . W2^T). On the forward keep pattern
// only (ref ffn.py:415-417 + sparse24.py:138-154, exact by construction):
//   g_pre = G * 2 * relu(y1),  relu(y1) recovered as sqrt(a) from the cached
// compressed activation a = relu(y1)^2. Output: compressed g_pre [M, N/2] on
// the forward metadata (which is reused as-is for the dX sparse GEMM).
// The tile's act values (256 B / row) and metadata rows are prefetched into
// registers before the accumulator wait, so their latency hides under the MMA.
struct EpiBwd1 {
  struct Params {
    const __nv_bfloat16* act_vals;  // [Mpad, N/2]
    const uint8_t* meta;            // hw layout, K = N
    __nv_bfloat16* gvals;           // [Mpad, N/2] out
    int N;
  };
  static constexpr int TILE_N = 256;
  static constexpr bool kUnroll = true;
  struct State {
    uint4 act[TILE_N / 16];  // 8 bf16 kept values per uint4 = 16 logical columns
    uint4 meta[TILE_N / 128][2];
  };
  __device__ static void init(const Params&, State&) {}
  __device__ static void finish(const Params&, State&, uint32_t) {}
  __device__ static void prefetch(const Params& p, State& s, int row, bool row_ok, int col_base) {
    if (!row_ok) return;
    const uint4* a = reinterpret_cast<const uint4*>(p.act_vals + static_cast<long long>(row) * (p.N / 2) + col_base / 2);
#pragma unroll
    for (int i = 0; i < TILE_N / 16; ++i)
      if (col_base + 16 * i < p.N) s.act[i] = a[i];
    const uint32_t r = static_cast<uint32_t>(row) & 127u;
#pragma unroll
    for (int at = 0; at < TILE_N / 128; ++at) {
      if (col_base + 128 * at >= p.N) break;
      const uint8_t* base = p.meta + meta_hw_halfword_offset(row, (col_base + 128 * at) / 16, p.N) -
                            meta_atom_halfword_byte(r, 0);
      const uint32_t row16 = 16u * (r & 7u) + 256u * (r >> 4);
      s.meta[at][0] = *reinterpret_cast<const uint4*>(base + row16);
      s.meta[at][1] = *reinterpret_cast<const uint4*>(base + row16 + 128);
    }
  }
  __device__ static uint32_t word(const uint4& v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
  }
  __device__ static void chunk(const Params& p, State& s, int row, bool row_ok, int col0, int c,
                               const float (&v)[32], uint32_t) {
    if (!row_ok) return;
    const uint32_t m1 = (static_cast<uint32_t>(row) >> 3) & 1u;
    // chunk c covers the 16-column quads 2c (k1 = 0) and 2c+1 (k1 = 1) of atom c/4, word k2 = c%4
    const uint32_t w0 = word(s.meta[c >> 2][0], c & 3), w1 = word(s.meta[c >> 2][1], c & 3);
    const uint32_t m16[2] = {(w0 >> (16 * m1)) & 0xFFFFu, (w1 >> (16 * m1)) & 0xFFFFu};
    const uint32_t aw[8] = {s.act[2 * c].x, s.act[2 * c].y, s.act[2 * c].z, s.act[2 * c].w,
                            s.act[2 * c + 1].x, s.act[2 * c + 1].y, s.act[2 * c + 1].z, s.act[2 * c + 1].w};
    uint32_t packed[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const uint32_t nib = (m16[g >> 2] >> (4 * (g & 3))) & 0xFu;
      const float g0 = sel4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3], nib & 3u);
      const float g1 = sel4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3], nib >> 2);
      const __nv_bfloat162 a2 = *reinterpret_cast<const __nv_bfloat162*>(&aw[g]);
      const float a0 = __bfloat162float(a2.x), a1 = __bfloat162float(a2.y);
      packed[g] = pack_bf16x2(g0 * (2.f * sqrtf(a0)), g1 * (2.f * sqrtf(a1)));
    }
    __nv_bfloat16* dst = p.gvals + static_cast<long long>(row) * (p.N / 2) + col0 / 2;
    st_global_v4(dst, packed[0], packed[1], packed[2], packed[3]);
    st_global_v4(dst + 8, packed[4], packed[5], packed[6], packed[7]);
  }
};

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
  __device__ static void prefetch(const Params&, State&, int, bool, int) {}
  __device__ static void finish(const Params&, State&, uint32_t) {}
  __device__ static void chunk(const Params& p, State&, int row, bool row_ok, int col0, int c,
                               const float (&v)[32], uint32_t) {
    if (!row_ok) return;
    float a[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float r = fmaxf(v[i], 0.f);
      a[i] = __fmul_rn(r, r);
    }
    __nv_bfloat16* dst = p.act + static_cast<long long>(row) * p.ld + col0;
#pragma unroll
    for (int i = 0; i < 32; i += 8)
      st_global_v4(dst + i, pack_bf16x2(a[i], a[i + 1]), pack_bf16x2(a[i + 2], a[i + 3]),
                   pack_bf16x2(a[i + 4], a[i + 5]), pack_bf16x2(a[i + 6], a[i + 7]));
  }
};

// bwd: g_pre = G * 2 * sqrt(act), dense (ref ffn.py:415 with act_squared_relu_grad :172-173).
// act chunks are software-pipelined 4 chunks ahead through registers.
struct EpiDact {
  struct Params {
    const __nv_bfloat16* act;
    long long ld_act;
    __nv_bfloat16* gpre;
    long long ld_g;
    int N;
  };
  static constexpr int AHEAD = 4;
  static constexpr bool kUnroll = true;
  struct State {
    uint4 buf[AHEAD][4];
    int col_base;
  };
  __device__ static void init(const Params&, State&) {}
  __device__ static void finish(const Params&, State&, uint32_t) {}
  __device__ static void load(const Params& p, State& s, int row, int c, int slot) {
    const int col = s.col_base + 32 * c;
    if (col >= p.N) return;
    const uint4* src = reinterpret_cast<const uint4*>(p.act + static_cast<long long>(row) * p.ld_act + col);
#pragma unroll
    for (int i = 0; i < 4; ++i) s.buf[slot][i] = src[i];
  }
  __device__ static void prefetch(const Params& p, State& s, int row, bool row_ok, int col_base) {
    s.col_base = col_base;
    if (!row_ok) return;
#pragma unroll
    for (int c = 0; c < AHEAD; ++c) load(p, s, row, c, c);
  }
  __device__ static void chunk(const Params& p, State& s, int row, bool row_ok, int col0, int c,
                               const float (&v)[32], uint32_t) {
    if (!row_ok) return;
    const int slot = c % AHEAD;
    uint32_t ww[16];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      ww[4 * i] = s.buf[slot][i].x;
      ww[4 * i + 1] = s.buf[slot][i].y;
      ww[4 * i + 2] = s.buf[slot][i].z;
      ww[4 * i + 3] = s.buf[slot][i].w;
    }
    load(p, s, row, c + AHEAD, slot);
    __nv_bfloat16* dst = p.gpre + static_cast<long long>(row) * p.ld_g + col0;
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
      uint32_t o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const __nv_bfloat162 a2 = *reinterpret_cast<const __nv_bfloat162*>(&ww[i / 2 + j]);
        o[j] = pack_bf16x2(v[i + 2 * j] * (2.f * sqrtf(__bfloat162float(a2.x))),
                           v[i + 2 * j + 1] * (2.f * sqrtf(__bfloat162float(a2.y))));
      }
      st_global_v4(dst + i, o[0], o[1], o[2], o[3]);
    }
  }
};

}  // namespace s24
