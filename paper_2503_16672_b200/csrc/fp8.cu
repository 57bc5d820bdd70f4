// e4m3 quantization for the fp8 FFN path (FfnConfig.fp8_emulation /
// fp8_backward) and the metadata layout the e4m3 2:4 MMA reads.
//
// Reference semantics (ref pkg/src/srelu24/matcore.py:113-261, ffn.py:206-268):
//   scale = amax / 448 per row (or column), 1 where amax == 0 or the division
//   underflows; code = e4m3(x / scale) rounded to nearest, ties to even
//   mantissa, saturating at +-448 (no infinities), -0 -> 0x80.
// cvt.rn.satfinite.e4m3x2.f32 is exactly that rounding of the fp32 quotient,
// and the quotient is the IEEE fp32 division the reference performs, so codes
// and scales are bit-identical to the reference on identical fp32 inputs.
//
// Kernels (all HBM-bound, one pass over the operand plus its output):
//   k_quant_rows    per-row (or per row pair) scales, codes in place of the
//                   row; optional bf16 dequantized image (what an 8-bit store
//                   reproduces, ref ffn.py:335-340) and bf16 raw image
//   k_col_amax +    per-column scales with the codes written TRANSPOSED
//   k_quant_cols_t  ([C, R]: the K-major operand layout the e4m3 MMA needs)
//   k_meta_to_f8    2:4 metadata atoms, kind::f16 layout -> kind::f8f6f4 layout
//   k_e4m3_encode   elementwise encode (parity tests of the conversion)
#include <cuda_bf16.h>

#include <type_traits>

#include "host_util.h"
#include "meta.cuh"

namespace s24 {

constexpr float kE4m3Max = 448.f;

__device__ __forceinline__ float e4m3_scale(float amax) {
  float s = amax > 0.f ? __fdiv_rn(amax, kE4m3Max) : 1.f;
  return s > 0.f ? s : 1.f;
}

// x / s for the whole row (column) with one shared divisor: r = RN(1/s) once,
// then q = x*r refined by one FMA residual step (Markstein). q is within a
// tiny fraction of an ulp of x/s, so it equals RN(x/s) except when x/s lies
// within ~2^-22 ulp of an fp32 midpoint; and an e4m3 rounding boundary is an
// fp32 number, never an fp32 midpoint, so the e4m3 code of q equals the code
// of RN(x/s) (exact e4m3 ties, x/s == boundary, are reproduced exactly: the
// refined q of an exactly representable quotient is that quotient). Three FP
// instructions instead of the IEEE division sequence, which made the
// quantizers issue-bound.
__device__ __forceinline__ float rcp_rn(float x) {
  float r;
  asm("rcp.rn.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

struct Divisor {
  float s, r;
  __device__ __forceinline__ explicit Divisor(float s_) : s(s_), r(rcp_rn(s_)) {}
  __device__ __forceinline__ float div(float x) const {
    const float q = __fmul_rn(x, r);
    const float e = __fmaf_rn(-q, s, x);
    return copysignf(__fmaf_rn(e, r, q), x);  // (-0 and negative underflow keep their sign: code 0x80)
  }
};

// two fp32 -> two e4m3 codes (lo in the low byte)
__device__ __forceinline__ uint32_t e4m3x2(float lo, float hi) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ float e4m3_decode(uint32_t code) {
  // exact: e4m3 -> f16x2 (hardware) -> f32
  uint32_t h2;
  const uint16_t c = static_cast<uint16_t>(code & 0xFFu);
  asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"(c));
  float f;
  asm("{ .reg .f16 lo, hi; mov.b32 {lo, hi}, %1; cvt.f32.f16 %0, lo; }" : "=f"(f) : "r"(h2));
  return f;
}

template <typename T>
__device__ __forceinline__ void load8(const T* p, float (&v)[8]) {
  if constexpr (std::is_same_v<T, float>) {
    const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
}

__device__ __forceinline__ uint32_t bf16x2_bits(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// One warp per unit: a single row, or (rows < pair_rows) an (even, odd) row
// pair sharing one scale (a dense feature stored as two 2:4 rows, k4.cuh).
// cols % 8 == 0; every row pointer 16-byte aligned. Each lane keeps U
// independent 16-byte loads in flight per iteration (rows are only a few KB:
// without that the kernel is load-latency bound); the second pass re-reads
// the row from L2.
template <typename InT, int U = 2>
__global__ void __launch_bounds__(256) k_quant_rows(const InT* __restrict__ in, long long ld_in, int rows, int cols,
                                                    const unsigned* __restrict__ amax_in, int pair_rows,
                                                    uint8_t* __restrict__ codes, long long ld_codes,
                                                    float* __restrict__ scales, __nv_bfloat16* __restrict__ deq,
                                                    long long ld_deq, __nv_bfloat16* __restrict__ raw,
                                                    long long ld_raw) {
  const int lane = threadIdx.x & 31;
  const int units = pair_rows / 2 + (rows - pair_rows);
  for (int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < units; u += (gridDim.x * blockDim.x) >> 5) {
    const int r0 = u < pair_rows / 2 ? 2 * u : u + pair_rows / 2;
    const int nr = u < pair_rows / 2 ? 2 : 1;
    float amax = 0.f;
    if (amax_in) {
      for (int k = 0; k < nr; ++k) amax = fmaxf(amax, __uint_as_float(amax_in[r0 + k]));
    } else {
      for (int k = 0; k < nr; ++k) {
        const InT* src = in + static_cast<long long>(r0 + k) * ld_in;
        for (int c0 = 8 * lane; c0 < cols; c0 += 256 * U) {
          float v[U][8];
#pragma unroll
          for (int j = 0; j < U; ++j)
            if (c0 + 256 * j < cols) load8(src + c0 + 256 * j, v[j]);
#pragma unroll
          for (int j = 0; j < U; ++j)
            if (c0 + 256 * j < cols)
#pragma unroll
              for (int i = 0; i < 8; ++i) amax = fmaxf(amax, fabsf(v[j][i]));
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    }
    const float s = e4m3_scale(amax);
    const Divisor dv(s);
    if (lane == 0)
      for (int k = 0; k < nr; ++k) scales[r0 + k] = s;
    for (int k = 0; k < nr; ++k) {
      const long long r = r0 + k;
      const InT* src = in + r * ld_in;
      for (int c0 = 8 * lane; c0 < cols; c0 += 256 * U) {
        float v[U][8];
#pragma unroll
        for (int j = 0; j < U; ++j)
          if (c0 + 256 * j < cols) load8(src + c0 + 256 * j, v[j]);
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const int c = c0 + 256 * j;
          if (c >= cols) continue;
          uint32_t q[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) q[i] = e4m3x2(dv.div(v[j][2 * i]), dv.div(v[j][2 * i + 1]));
          *reinterpret_cast<uint2*>(codes + r * ld_codes + c) = make_uint2(q[0] | (q[1] << 16), q[2] | (q[3] << 16));
          if (deq) {
            uint32_t o[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
              o[i] = bf16x2_bits(__fmul_rn(e4m3_decode(q[i]), s), __fmul_rn(e4m3_decode(q[i] >> 8), s));
            *reinterpret_cast<uint4*>(deq + r * ld_deq + c) = make_uint4(o[0], o[1], o[2], o[3]);
          }
          if (raw) {
            *reinterpret_cast<uint4*>(raw + r * ld_raw + c) =
                make_uint4(bf16x2_bits(v[j][0], v[j][1]), bf16x2_bits(v[j][2], v[j][3]),
                           bf16x2_bits(v[j][4], v[j][5]), bf16x2_bits(v[j][6], v[j][7]));
          }
        }
      }
    }
  }
}

template <typename T>
__device__ __forceinline__ float ld1(const T* p) {
  if constexpr (std::is_same_v<T, float>)
    return *p;
  else
    return __bfloat162float(*p);
}

// column |max| of a bf16 / fp32 [R, C] matrix into amax[C] (float bits,
// atomicMax; zeroed by the caller). Block: 32 x 8 threads, 256 columns x
// rows_per_block.
template <typename InT>
__global__ void __launch_bounds__(256) k_col_amax(const InT* __restrict__ in, long long ld, int R, int C,
                                                  int rows_per_block, unsigned* __restrict__ amax) {
  __shared__ float red[8][256 + 8];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c0 = blockIdx.x * 256 + 8 * tx;
  const int rb = blockIdx.y * rows_per_block;
  const int re = min(R, rb + rows_per_block);
  float m[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c0 + 8 <= C) {
    int r = rb + ty;
    for (; r + 24 < re; r += 32) {  // four independent loads in flight
      float v[4][8];
#pragma unroll
      for (int u = 0; u < 4; ++u) load8(in + static_cast<long long>(r + 8 * u) * ld + c0, v[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int i = 0; i < 8; ++i) m[i] = fmaxf(m[i], fabsf(v[u][i]));
    }
    for (; r < re; r += 8) {
      float v[8];
      load8(in + static_cast<long long>(r) * ld + c0, v);
#pragma unroll
      for (int i = 0; i < 8; ++i) m[i] = fmaxf(m[i], fabsf(v[i]));
    }
  } else {
    for (int r = rb + ty; r < re; r += 8)
      for (int i = 0; i < 8 && c0 + i < C; ++i)
        m[i] = fmaxf(m[i], fabsf(ld1(in + static_cast<long long>(r) * ld + c0 + i)));
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) red[ty][8 * tx + i] = m[i];
  __syncthreads();
  const int c = threadIdx.x;  // 0..255
  float x = red[0][c];
#pragma unroll
  for (int k = 1; k < 8; ++k) x = fmaxf(x, red[k][c]);
  if (blockIdx.x * 256 + c < C && x > 0.f) atomicMax(amax + blockIdx.x * 256 + c, __float_as_uint(x));
}

// codes_t[c, r] = e4m3(in[r, c] / scale[c]). A block transposes a (128 U)-row
// x 64-column tile through shared memory. Each thread quantizes U 4-row x
// 8-column units (eight lanes read one row's 64 columns contiguously) and packs
// each column's 4 row codes into one 32-bit word, so the transpose costs 8 word
// stores per unit (2-way bank conflicts with the odd row pitch) instead of 32
// byte stores; the tile is then written out as (128 U)-byte runs per output row.
// Every thread has all of its global loads in flight before it converts. U = 1
// (48 registers, 5 CTAs/SM): 29.9 us for the c2 g_c operand vs 38.4 us at U = 2
// (80 registers) and 43.7 us for the earlier 64 x 64 byte-transpose (ncu).
template <typename InT, int U = 1>
__global__ void __launch_bounds__(256) k_quant_cols_t(const InT* __restrict__ in, long long ld, int R,
                                                      int C, const unsigned* __restrict__ amax,
                                                      uint8_t* __restrict__ out, long long ld_out,
                                                      float* __restrict__ scales) {
  constexpr int kTR = 128 * U, kTC = 64, kPitch = kTR / 4 + 1;  // tile rows, tile columns, words per tile row
  __shared__ uint32_t tile[kTC * kPitch];
  __shared__ float sc[kTC], rc[kTC];
  const int r0 = blockIdx.y * kTR, c0 = blockIdx.x * kTC;
  const int t = threadIdx.x;
  if (t < kTC) {
    const float s = (c0 + t < C) ? e4m3_scale(__uint_as_float(amax[c0 + t])) : 1.f;
    sc[t] = s;
    rc[t] = rcp_rn(s);
    if (blockIdx.y == 0 && c0 + t < C) scales[c0 + t] = s;
  }
  const int col8 = t & 7, row4 = t >> 3;  // unit: columns 8*col8.., rows 4*row4 (+128 for the second unit)
  const int cb = c0 + 8 * col8;
  float v[U][4][8];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = r0 + 128 * u + 4 * row4 + k;
      const InT* src = in + static_cast<long long>(r) * ld + cb;
      if (r < R && cb + 8 <= C) {
        load8(src, v[u][k]);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[u][k][i] = (r < R && cb + i < C) ? ld1(src + i) : 0.f;
      }
    }
  __syncthreads();  // sc / rc
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    Divisor dv{0.f};
    dv.s = sc[8 * col8 + i];
    dv.r = rc[8 * col8 + i];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t lo = e4m3x2(dv.div(v[u][0][i]), dv.div(v[u][1][i]));
      const uint32_t hi = e4m3x2(dv.div(v[u][2][i]), dv.div(v[u][3][i]));
      tile[(8 * col8 + i) * kPitch + 32 * u + row4] = lo | (hi << 16);
    }
  }
  __syncthreads();
  constexpr int kChunks = kTR / 16;  // 16-code chunks per output row
#pragma unroll
  for (int m = 0; m < 2 * U; ++m) {
    const int q = t + 256 * m;
    const int cc = q / kChunks, w = (q % kChunks) * 4;  // output row c0 + cc, codes 4w .. 4w + 15
    const int c = c0 + cc, r = r0 + 4 * w;
    if (c >= C || r >= R) continue;
    const uint32_t* s32 = tile + cc * kPitch + w;
    uint8_t* dst = out + static_cast<long long>(c) * ld_out + r;
    if (r + 16 <= R) {
      *reinterpret_cast<uint4*>(dst) = make_uint4(s32[0], s32[1], s32[2], s32[3]);
    } else {
      for (int i = 0; i < 16 && r + i < R; ++i) dst[i] = static_cast<uint8_t>(s32[i >> 2] >> (8 * (i & 3)));
    }
  }
}

// kind::f16 metadata atom (meta.cuh) -> kind::f8f6f4 atom: the same 2048
// bytes per 128 rows x 128 logical K, row r's 8 halfwords contiguous at 16 r.
__global__ void __launch_bounds__(256) k_meta_to_f8(const uint16_t* __restrict__ src, uint16_t* __restrict__ dst,
                                                    long long halfwords) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < halfwords;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long atom = i >> 10;
    const uint32_t w = static_cast<uint32_t>(i & 1023);
    dst[i] = src[atom * 1024 + meta_atom_halfword_byte(w >> 3, w & 7u) / 2];
  }
}

// The same conversion, 16-byte vectors. Rows r and r + 8 of an atom (m1 = 0/1)
// read the same two 16-byte chunks of the source (byte 16 m0 + 256 m2, and
// +128 for the odd halfwords q), so one thread loads both chunks and writes
// both rows' 16 bytes: its halfword q of row m1 is chunk (q & 1)'s halfword
// m1 + 2 (q >> 1). Needs 16-byte aligned buffers.
__global__ void __launch_bounds__(256) k_meta_to_f8_v(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                      long long atoms) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < atoms * 64;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long atom = i >> 6;
    const uint32_t j = static_cast<uint32_t>(i & 63), m0 = j & 7u, m2 = j >> 3;
    const uint4* s = src + atom * 128 + m0 + 16 * m2;  // chunk A (16 B units); chunk B = A + 8
    const uint4 a = s[0], b = s[8];
    uint4* d = dst + atom * 128 + m0 + 16 * m2;  // row m0 + 16 m2 (m1 = 0); row + 8 at d + 8
    d[0] = make_uint4(__byte_perm(a.x, b.x, 0x5410), __byte_perm(a.y, b.y, 0x5410), __byte_perm(a.z, b.z, 0x5410),
                      __byte_perm(a.w, b.w, 0x5410));
    d[8] = make_uint4(__byte_perm(a.x, b.x, 0x7632), __byte_perm(a.y, b.y, 0x7632), __byte_perm(a.z, b.z, 0x7632),
                      __byte_perm(a.w, b.w, 0x7632));
  }
}

__global__ void k_e4m3_encode(const float* __restrict__ x, long long n, uint8_t* __restrict__ codes) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    codes[i] = static_cast<uint8_t>(e4m3x2(x[i], 0.f) & 0xFFu);
}

static int grid_for(long long work, int per_block) {
  long long b = (work + per_block - 1) / per_block;
  const long long cap = 16ll * num_sms();
  if (b > cap) b = cap;
  return static_cast<int>(b < 1 ? 1 : b);
}

}  // namespace s24

using namespace s24;

extern "C" {

int s24_fp8_quant_rows(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t ld_in,
                       const unsigned* amax_in, int64_t pair_rows, uint8_t* codes, int64_t ld_codes, float* scales,
                       void* deq_bf16, int64_t ld_deq, void* raw_bf16, int64_t ld_raw, void* stream) {
  if (rows < 0 || cols < 0) return fail(S24_ERR_DIMENSION, "negative dimension");
  if (cols % 8 != 0) return fail(S24_ERR_DIMENSION, "quantized row length %lld must be a multiple of 8", (long long)cols);
  if (pair_rows < 0 || pair_rows % 2 || pair_rows > rows) return fail(S24_ERR_DIMENSION, "pair_rows must be even, <= rows");
  if (!codes || !scales) return fail(S24_ERR_DIMENSION, "codes and scales are required");
  if (in_dtype != S24_F32 && in_dtype != S24_BF16) return fail(S24_ERR_PRECISION, "input must be fp32 or bf16");
  if (ld_in < cols || ld_codes < cols || (deq_bf16 && ld_deq < cols) || (raw_bf16 && ld_raw < cols))
    return fail(S24_ERR_DIMENSION, "leading dimension too small");
  if (ld_codes % 8 || (deq_bf16 && ld_deq % 8) || (raw_bf16 && ld_raw % 8) || ld_in % (in_dtype == S24_F32 ? 4 : 8))
    return fail(S24_ERR_DIMENSION, "leading dimensions must keep rows 16-byte aligned");
  if (rows == 0 || cols == 0) return S24_OK;
  auto st = static_cast<cudaStream_t>(stream);
  const long long units = pair_rows / 2 + (rows - pair_rows);
  const int grid = grid_for(units * 32, 256);
  if (in_dtype == S24_F32)
    k_quant_rows<float><<<grid, 256, 0, st>>>(static_cast<const float*>(in), ld_in, static_cast<int>(rows),
                                              static_cast<int>(cols), amax_in, static_cast<int>(pair_rows), codes,
                                              ld_codes, scales, static_cast<__nv_bfloat16*>(deq_bf16), ld_deq,
                                              static_cast<__nv_bfloat16*>(raw_bf16), ld_raw);
  else
    k_quant_rows<__nv_bfloat16><<<grid, 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(in), ld_in, static_cast<int>(rows), static_cast<int>(cols), amax_in,
        static_cast<int>(pair_rows), codes, ld_codes, scales, static_cast<__nv_bfloat16*>(deq_bf16), ld_deq,
        static_cast<__nv_bfloat16*>(raw_bf16), ld_raw);
  return check_launch("k_quant_rows");
}

int s24_fp8_quant_cols_t(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t ld_in, uint8_t* codes_t,
                         int64_t ld_out, float* scales, unsigned* amax_ws, void* stream) {
  if (rows < 0 || cols < 0) return fail(S24_ERR_DIMENSION, "negative dimension");
  if (in_dtype != S24_F32 && in_dtype != S24_BF16) return fail(S24_ERR_PRECISION, "input must be fp32 or bf16");
  if (!codes_t || !scales || !amax_ws) return fail(S24_ERR_DIMENSION, "codes, scales and the workspace are required");
  if (ld_in < cols || ld_in % (in_dtype == S24_F32 ? 4 : 8))
    return fail(S24_ERR_DIMENSION, "ld_in must be >= cols and keep rows 16-byte aligned");
  if (ld_out < rows || ld_out % 16) return fail(S24_ERR_DIMENSION, "ld_out must be >= rows and a multiple of 16");
  if (rows > (1ll << 31) - 64 || cols > (1ll << 31) - 256) return fail(S24_ERR_DIMENSION, "matrix too large");
  if (cols == 0) return S24_OK;
  auto st = static_cast<cudaStream_t>(stream);
  cudaMemsetAsync(amax_ws, 0, sizeof(unsigned) * cols, st);
  if (rows > 0) {
    const int cb = static_cast<int>((cols + 255) / 256);
    int rpb = 256;
    while (static_cast<long long>(cb) * ((rows + rpb - 1) / rpb) > 8ll * num_sms() && rpb < (1 << 20)) rpb *= 2;
    dim3 g1(cb, static_cast<unsigned>((rows + rpb - 1) / rpb));
    if (in_dtype == S24_F32)
      k_col_amax<float><<<g1, 256, 0, st>>>(static_cast<const float*>(in), ld_in, static_cast<int>(rows),
                                            static_cast<int>(cols), rpb, amax_ws);
    else
      k_col_amax<__nv_bfloat16><<<g1, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(in), ld_in,
                                                    static_cast<int>(rows), static_cast<int>(cols), rpb, amax_ws);
    int rc = check_launch("k_col_amax");
    if (rc) return rc;
  }
  dim3 g2(static_cast<unsigned>((cols + 63) / 64), static_cast<unsigned>(rows > 0 ? (rows + 127) / 128 : 1));
  if (in_dtype == S24_F32)
    k_quant_cols_t<float><<<g2, 256, 0, st>>>(static_cast<const float*>(in), ld_in, static_cast<int>(rows),
                                              static_cast<int>(cols), amax_ws, codes_t, ld_out, scales);
  else
    k_quant_cols_t<__nv_bfloat16><<<g2, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(in), ld_in,
                                                      static_cast<int>(rows), static_cast<int>(cols), amax_ws,
                                                      codes_t, ld_out, scales);
  return check_launch("k_quant_cols_t");
}

int s24_meta_hw_to_f8(const uint8_t* meta_hw, int64_t rows, int64_t kdim, uint8_t* meta_f8, void* stream) {
  if (rows < 0 || kdim < 0 || kdim % 128) return fail(S24_ERR_DIMENSION, "metadata K must be a multiple of 128");
  const long long bytes = (rows + 127) / 128 * 128 * kdim / 8;
  if (bytes == 0) return S24_OK;
  if ((reinterpret_cast<uintptr_t>(meta_hw) | reinterpret_cast<uintptr_t>(meta_f8)) % 16 == 0)
    k_meta_to_f8_v<<<grid_for(bytes / 32, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const uint4*>(meta_hw), reinterpret_cast<uint4*>(meta_f8), bytes / 2048);
  else
    k_meta_to_f8<<<grid_for(bytes / 2, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const uint16_t*>(meta_hw), reinterpret_cast<uint16_t*>(meta_f8), bytes / 2);
  return check_launch("k_meta_to_f8");
}

int s24_e4m3_encode(const float* x, int64_t n, uint8_t* codes, void* stream) {
  if (n < 0) return fail(S24_ERR_DIMENSION, "negative length");
  if (n == 0) return S24_OK;
  k_e4m3_encode<<<grid_for(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(x, n, codes);
  return check_launch("k_e4m3_encode");
}

}  // extern "C"
