// C-ABI entry points for the tcgen05 GEMMs (dense, 2:4 sparse, fused K1/K3)
// plus the shared host utilities (error text, tensor maps, SM count).
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>

#include "epilogues.cuh"
#include "gemm.cuh"
#include "host_util.h"

namespace s24 {

std::string& last_error_ref() {
  static thread_local std::string msg;
  return msg;
}

int num_sms() {
  static std::mutex mu;
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  std::lock_guard<std::mutex> lock(mu);
  if (!cached[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 148;
  }
  return cached[dev];
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int make_map_2d(CUtensorMap* map, const void* base, bool bf16, uint64_t inner, uint64_t outer, uint64_t ld_bytes,
                uint32_t box_inner, uint32_t box_outer, int swizzle) {
  auto fn = encode_fn();
  if (!fn) return fail(S24_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (!aligned16(base) || ld_bytes % 16 != 0)
    return fail(S24_ERR_DIMENSION, "operand base/leading dimension must be 16-byte aligned");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 2,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                  : swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                  : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(S24_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
  return S24_OK;
}

int make_map_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
                  uint32_t box_inner, uint32_t box_outer, int swizzle) {
  return make_map_2d(map, base, true, inner, outer, ld * 2, box_inner, box_outer, swizzle);
}

// operands of one GEMM problem (the grouped launch takes two of equal shape)
template <class Epi>
struct GemmOperands {
  const void* A;
  int64_t lda;
  const void* B;
  int64_t ldb;
  const uint8_t* meta;
  typename Epi::Params ep;
};

template <class Cfg>
static int make_operand_maps(const void* A, int64_t lda, const void* B, int64_t ldb, const uint8_t* meta, int64_t M,
                             int64_t N, int64_t K, CUtensorMap* ma, CUtensorMap* mb, CUtensorMap* me) {
  int rc;
  if constexpr (Cfg::F8) {
    // e4m3 codes, both operands K-major (uint8 maps, 128-element boxes)
    if constexpr (Cfg::SPARSE) {
      const int64_t mpad = (M + 127) / 128 * 128;
      rc = make_map_2d(ma, A, false, K / 2, mpad, K / 2, 128, Cfg::BM, 128);
    } else {
      rc = make_map_2d(ma, A, false, K, M, lda, 128, Cfg::BM, 128);
    }
    if (rc) return rc;
    rc = make_map_2d(mb, B, false, K, N, ldb, 128, Cfg::B_BOX_ROWS, 128);
    if (rc) return rc;
    std::memset(me, 0, sizeof(*me));
    if constexpr (Cfg::SPARSE) {
      const int64_t atoms = (M + 127) / 128 * (K / 128);
      rc = make_map_2d(me, meta, false, 128, static_cast<uint64_t>(atoms) * 16, 128, 128, 16 * Cfg::E_ATOMS, 0);
    }
    return rc;
  }
  // A
  if constexpr (Cfg::A_MN) {
    rc = make_map_bf16(ma, A, M, K, lda, 64, Cfg::BK, 128);
  } else if constexpr (Cfg::SPARSE) {
    const int64_t mpad = (M + 127) / 128 * 128;
    rc = make_map_bf16(ma, A, K / 2, mpad, K / 2, 64, Cfg::BM, 128);
  } else {
    rc = make_map_bf16(ma, A, K, M, lda, 64, Cfg::BM, 128);
  }
  if (rc) return rc;
  // B
  if constexpr (Cfg::B_MN) {
    rc = make_map_bf16(mb, B, N, K, ldb, 64, Cfg::BK, 128);
  } else {
    rc = make_map_bf16(mb, B, K, N, ldb, 64, Cfg::B_BOX_ROWS, 128);
  }
  if (rc) return rc;
  std::memset(me, 0, sizeof(*me));
  if constexpr (Cfg::SPARSE) {
    // metadata atoms viewed as [atoms * 16 rows, 128 bytes]; one box = one atom
    const int64_t atoms = (M + 127) / 128 * (K / 128);
    rc = make_map_2d(me, meta, false, 128, static_cast<uint64_t>(atoms) * 16, 128, 128, 16, 0);
    if (rc) return rc;
  }
  return S24_OK;
}

template <class Cfg, class Epi>
static int launch_gemm(const void* A, int64_t lda, const void* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                       const uint8_t* meta, const typename Epi::Params& ep, cudaStream_t stream, int k_splits = 1,
                       const GemmOperands<Epi>* second = nullptr) {
  if (M <= 0 || N <= 0 || K <= 0) return S24_OK;
  if (M > (1 << 30) || N > (1 << 30) || K > (1 << 30)) return fail(S24_ERR_DIMENSION, "GEMM dims too large");
  CUtensorMap ma, mb, me, ma2, mb2, me2;
  int rc = make_operand_maps<Cfg>(A, lda, B, ldb, meta, M, N, K, &ma, &mb, &me);
  if (rc) return rc;
  if (second) {
    rc = make_operand_maps<Cfg>(second->A, second->lda, second->B, second->ldb, second->meta, M, N, K, &ma2, &mb2,
                                &me2);
    if (rc) return rc;
  } else {
    ma2 = ma;
    mb2 = mb;
    me2 = me;
  }

  GemmShape sh;
  sh.M = static_cast<int>(M);
  sh.N = static_cast<int>(N);
  sh.K = static_cast<int>(K);
  sh.tiles_m = static_cast<int>((M + Cfg::TILE_M - 1) / Cfg::TILE_M);
  sh.tiles_n = static_cast<int>((N + Cfg::BN - 1) / Cfg::BN);
  // raster: groups of 512 rows sweep N (measured best for the 2:4 GEMMs,
  // neutral for the dense ones; 2048-row groups cost up to 10%)
  sh.group_m = 4 / Cfg::CLUSTER;
  sh.k_splits = k_splits < 1 ? 1 : k_splits;
  sh.groups = second ? 2 : 1;
  const int tiles = sh.tiles_m * sh.tiles_n * sh.k_splits * sh.groups;
  if (static_cast<long long>(tiles) * 2 * Cfg::CLUSTER >= (1ll << 31)) return fail(S24_ERR_DIMENSION, "too many tiles");

  auto kern = gemm_kernel<Cfg, Epi>;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = Cfg::CLUSTER;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // critical-path priority (host_util.h high_priority): when a GEMM becomes
  // ready together with a side-stream kernel (K4), the block scheduler places
  // the GEMM's CTA pairs first and K4 fills the registers / warps they leave
  attr[1].id = cudaLaunchAttributePriority;
  attr[1].val.priority = high_priority();
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  // clusters resident at once (one CTA per SM: the stage ring fills smem)
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  });
  if (attr_err != cudaSuccess) return fail(S24_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(attr_err));
  const int resident = num_sms() / Cfg::CLUSTER;
  // L2 policies (see gemm.cuh): pin B when it fits, and only then let the
  // A panels stream through (measured: with a 64 MiB B, evict-first A panels
  // are lost before all N tiles of their row have read them)
  sh.b_keep = static_cast<long long>(K) * N * Cfg::EB * sh.groups <= (40ll << 20);
  sh.a_stream = sh.b_keep && sh.group_m * sh.tiles_n <= resident;
  // a partial last wave of at most half the clusters: its tiles run as two
  // N-halves each, so that wave takes half as long
  sh.tail_split = 0;
  if constexpr (Cfg::HALF_OK) {
    const int rem = tiles % resident;
    if (tiles > resident && rem > 0 && 2 * rem <= resident) sh.tail_split = rem;
  }
  // one cluster per work unit; running clusters steal the units of the ones
  // that have not started (cluster launch control, gemm.cuh)
  long long units = static_cast<long long>(tiles) + sh.tail_split;
  if (S24_STATIC_SCHED && units > resident) units = resident;  // (persistent grid, static round robin)
  cfg.gridDim = dim3(static_cast<unsigned>(units * Cfg::CLUSTER));
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, mb, me, ma2, mb2, me2, sh, ep, second ? second->ep : ep);
  if (e != cudaSuccess) return fail(S24_ERR_CUDA, "gemm launch: %s", cudaGetErrorString(e));
  return check_launch("gemm_kernel");
}

// tile configurations
// <sparse, A MN-major, B MN-major, BN, stages, CTA-group, epilogue warps, e4m3>
#ifndef S24_DN_STAGES
#define S24_DN_STAGES 6
#endif
using DenseKN = GemmCfg<false, false, true, 256, S24_DN_STAGES, 2, 8>;   // A K-major, B MN-major
using DenseKK = GemmCfg<false, false, false, 256, S24_DN_STAGES, 2, 8>;  // A K-major, B K-major
using DenseMM = GemmCfg<false, true, true, 256, S24_DN_STAGES, 2, 8>;    // A MN-major, B MN-major
using DenseMK = GemmCfg<false, true, false, 256, S24_DN_STAGES, 2, 8>;   // A MN-major, B K-major
// sparse: light epilogue, 4 epilogue warps and <= 128 registers/thread, leaving
// room for a co-resident side-stream kernel (the feature-wise split K4)
// (4 stages of 50 KB: 3 measured 18% slower; 8 half-K stages of 26 KB with
// SWIZZLE_64B A rows 25-37% slower)
#ifndef S24_SP_STAGES
#define S24_SP_STAGES 4
#endif
using SparseN = GemmCfg<true, false, true, 256, S24_SP_STAGES, 2, 4>;   // sparse A, B MN-major
using SparseK = GemmCfg<true, false, false, 256, S24_SP_STAGES, 2, 4>;  // sparse A, B K-major

// e4m3 (kind::f8f6f4): same byte geometry per stage as the bf16 configs
using F8DenseKK = GemmCfg<false, false, false, 256, 6, 2, 8, true>;
using F8SparseK = GemmCfg<true, false, false, 256, 4, 2, 4, true>;

// wide dense tiles: 256 x 512 per CTA pair, one 512-column accumulator (see
// gemm.cuh). A quarter fewer operand bytes per MAC than 256 x 256, but the
// accumulator drain is exposed. Measured at c2 (scripts/gpu_wide.sh): the
// MN-major-A weight-gradient GEMMs (K = tokens = 16384) gain 6-9%; the
// K-major-A GEMMs lose 1-6% (K1 0.400 -> 0.423 ms: its heavier epilogue is
// what gets exposed). Default: wide for MN-major A only.
using DenseKN_W = GemmCfg<false, false, true, 512, 4, 2, 8>;
using DenseKK_W = GemmCfg<false, false, false, 512, 4, 2, 8>;
using DenseMM_W = GemmCfg<false, true, true, 512, 4, 2, 8>;
using DenseMK_W = GemmCfg<false, true, false, 512, 4, 2, 8>;
using F8DenseKK_W = GemmCfg<false, false, false, 512, 4, 2, 8, true>;

static bool dense_wide(bool a_mn) { return a_mn; }

template <class Narrow, class Wide, class Epi>
static int launch_dense(const void* A, int64_t lda, const void* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                        const typename Epi::Params& ep, cudaStream_t st, int k_splits = 1) {
  if (dense_wide(Narrow::A_MN)) return launch_gemm<Wide, Epi>(A, lda, B, ldb, M, N, K, nullptr, ep, st, k_splits);
  return launch_gemm<Narrow, Epi>(A, lda, B, ldb, M, N, K, nullptr, ep, st, k_splits);
}

template <class Epi>
static int dispatch_dense(int a_mn, int b_mn, const void* A, int64_t lda, const void* B, int64_t ldb, int64_t M,
                          int64_t N, int64_t K, const typename Epi::Params& ep, cudaStream_t st, int k_splits = 1) {
  if (!a_mn && b_mn) return launch_dense<DenseKN, DenseKN_W, Epi>(A, lda, B, ldb, M, N, K, ep, st, k_splits);
  if (!a_mn && !b_mn) return launch_dense<DenseKK, DenseKK_W, Epi>(A, lda, B, ldb, M, N, K, ep, st, k_splits);
  if (a_mn && b_mn) return launch_dense<DenseMM, DenseMM_W, Epi>(A, lda, B, ldb, M, N, K, ep, st, k_splits);
  return launch_dense<DenseMK, DenseMK_W, Epi>(A, lda, B, ldb, M, N, K, ep, st, k_splits);
}

// split-K partial sums ws[ks][M][N] -> D (row map / transpose), fixed order.
// One thread per 4 consecutive columns (float4 partial reads; N % 32 == 0).
template <typename OutT>
__global__ void __launch_bounds__(256) k_splitk_reduce(const float* __restrict__ ws, int k_splits, long long M,
                                                       long long N, OutT* __restrict__ out, long long ldo,
                                                       const int* __restrict__ row_map, int transposed) {
  const long long total = M * N, quads = total / 4;
  for (long long qi = blockIdx.x * (long long)blockDim.x + threadIdx.x; qi < quads;
       qi += (long long)gridDim.x * blockDim.x) {
    const long long i = qi * 4;
    float4 acc = *reinterpret_cast<const float4*>(ws + i);
    for (int k = 1; k < k_splits; ++k) {
      const float4 p = *reinterpret_cast<const float4*>(ws + k * total + i);
      acc.x += p.x;
      acc.y += p.y;
      acc.z += p.z;
      acc.w += p.w;
    }
    const long long m = i / N, n = i - m * N;
    const long long r = row_map ? row_map[m] : m;
    const float v[4] = {acc.x, acc.y, acc.z, acc.w};
    if (transposed) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if constexpr (sizeof(OutT) == 4)
          out[(n + j) * ldo + r] = v[j];
        else
          out[(n + j) * ldo + r] = __float2bfloat16_rn(v[j]);
      }
    } else if constexpr (sizeof(OutT) == 4) {
      *reinterpret_cast<float4*>(out + r * ldo + n) = acc;
    } else {
      __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(out + r * ldo + n);
      o[0] = __floats2bfloat162_rn(v[0], v[1]);
      o[1] = __floats2bfloat162_rn(v[2], v[3]);
    }
  }
}

template <class Epi>
static int dispatch_sparse(int b_mn, const void* A, const uint8_t* meta, const void* B, int64_t ldb, int64_t M,
                           int64_t N, int64_t K, const typename Epi::Params& ep, cudaStream_t st,
                           const GemmOperands<Epi>* second = nullptr) {
  if (b_mn) return launch_gemm<SparseN, Epi>(A, K / 2, B, ldb, M, N, K, meta, ep, st, 1, second);
  return launch_gemm<SparseK, Epi>(A, K / 2, B, ldb, M, N, K, meta, ep, st, 1, second);
}

static int check_common(int64_t M, int64_t N, int64_t K, int64_t lda, int a_mn, int64_t ldb, int b_mn) {
  if (M < 0 || N < 0 || K < 0) return fail(S24_ERR_DIMENSION, "negative GEMM dimension");
  if (N % 32 != 0) return fail(S24_ERR_DIMENSION, "N = %lld must be a multiple of 32", (long long)N);
  if (lda < (a_mn ? M : K)) return fail(S24_ERR_DIMENSION, "lda too small");
  if (ldb < (b_mn ? N : K)) return fail(S24_ERR_DIMENSION, "ldb too small");
  return S24_OK;
}

template <class Fn>
static int with_out(int out_dtype, Fn&& fn) {
  if (out_dtype == S24_F32) return fn(static_cast<float*>(nullptr));
  if (out_dtype == S24_BF16) return fn(static_cast<__nv_bfloat16*>(nullptr));
  return fail(S24_ERR_PRECISION, "unsupported output dtype %d", out_dtype);
}

}  // namespace s24

using namespace s24;

extern "C" {

const char* s24_last_error(void) { return last_error_ref().c_str(); }
const char* s24_version(void) { return "s24-b200 0.1.0 (sm_100a)"; }

int64_t s24_meta_hw_bytes(int64_t rows, int64_t cols) {
  const int64_t rp = (rows + 127) / 128 * 128;
  return rp * cols / 8;
}

int s24_gemm(const void* A, int a_mn_major, int64_t lda, const void* B, int b_mn_major, int64_t ldb, int64_t M,
             int64_t N, int64_t K, void* D, int out_dtype, int64_t ldd, const int* d_row_map, int d_transposed,
             int64_t d_rows_valid, const int* d_row_valid, void* stream) {
  int rc = check_common(M, N, K, lda, a_mn_major, ldb, b_mn_major);
  if (rc) return rc;
  if (!d_transposed && ldd < N) return fail(S24_ERR_DIMENSION, "ldd too small");
  return with_out(out_dtype, [&](auto tag) {
    using OutT = std::remove_pointer_t<decltype(tag)>;
    typename EpiStore<OutT>::Params ep{static_cast<OutT*>(D), ldd, d_row_map, d_transposed,
                                       static_cast<int>(d_rows_valid < 0 ? M : d_rows_valid), d_row_valid, 0};
    return dispatch_dense<EpiStore<OutT>>(a_mn_major, b_mn_major, A, lda, B, ldb, M, N, K, ep,
                                          static_cast<cudaStream_t>(stream));
  });
}

int s24_gemm_splitk(const void* A, int a_mn_major, int64_t lda, const void* B, int b_mn_major, int64_t ldb,
                    int64_t M, int64_t N, int64_t K, int k_splits, float* workspace, void* D, int out_dtype,
                    int64_t ldd, const int* d_row_map, int d_transposed, void* stream) {
  int rc = check_common(M, N, K, lda, a_mn_major, ldb, b_mn_major);
  if (rc) return rc;
  if (k_splits < 1 || k_splits > 64) return fail(S24_ERR_CONFIG, "k_splits must be in [1, 64]");
  if (!workspace) return fail(S24_ERR_DIMENSION, "split-K needs a workspace of k_splits*M*N floats");
  if (ldd % 4 != 0 && !d_transposed) return fail(S24_ERR_DIMENSION, "split-K output needs ldd %% 4 == 0");
  if (out_dtype != S24_F32 && out_dtype != S24_BF16) return fail(S24_ERR_PRECISION, "unsupported output dtype");
  if (M == 0 || N == 0) return S24_OK;
  auto st = static_cast<cudaStream_t>(stream);
  EpiStore<float>::Params ep{workspace, N, nullptr, 0, static_cast<int>(M), nullptr, M * N};
  rc = dispatch_dense<EpiStore<float>>(a_mn_major, b_mn_major, A, lda, B, ldb, M, N, K, ep, st, k_splits);
  if (rc) return rc;
  long long blocks = (M * N / 4 + 255) / 256;
  if (blocks > 8L * num_sms()) blocks = 8L * num_sms();
  if (out_dtype == S24_F32)
    k_splitk_reduce<float><<<static_cast<int>(blocks), 256, 0, st>>>(workspace, k_splits, M, N, static_cast<float*>(D),
                                                                   ldd, d_row_map, d_transposed);
  else
    k_splitk_reduce<__nv_bfloat16><<<static_cast<int>(blocks), 256, 0, st>>>(
        workspace, k_splits, M, N, static_cast<__nv_bfloat16*>(D), ldd, d_row_map, d_transposed);
  return check_launch("k_splitk_reduce");
}

int s24_spmm(const void* a_vals, const uint8_t* a_meta, const void* B, int b_mn_major, int64_t ldb, int64_t M,
             int64_t N, int64_t K, void* D, int out_dtype, int64_t ldd, const int* d_row_map, int d_transposed,
             int64_t d_rows_valid, const int* d_row_valid, int64_t pair_rows, void* stream) {
  int rc = check_common(M, N, K, K, 0, ldb, b_mn_major);
  if (rc) return rc;
  if (K % 128 != 0) return fail(S24_ERR_DIMENSION, "sparse K = %lld must be a multiple of 128", (long long)K);
  if (!d_transposed && ldd < N) return fail(S24_ERR_DIMENSION, "ldd too small");
  if (pair_rows < 0 || pair_rows % 2 || pair_rows > M) return fail(S24_ERR_DIMENSION, "pair_rows must be even, <= M");
  return with_out(out_dtype, [&](auto tag) {
    using OutT = std::remove_pointer_t<decltype(tag)>;
    typename EpiStore<OutT>::Params ep{static_cast<OutT*>(D), ldd, d_row_map, d_transposed,
                                       static_cast<int>(d_rows_valid < 0 ? M : d_rows_valid), d_row_valid, 0,
                                       static_cast<int>(pair_rows)};
    return dispatch_sparse<EpiStore<OutT>>(b_mn_major, a_vals, a_meta, B, ldb, M, N, K, ep,
                                           static_cast<cudaStream_t>(stream));
  });
}

int s24_spmm_pair(int b_mn_major, int64_t M, int64_t N, int64_t K, int out_dtype, const void* a_vals0,
                  const uint8_t* a_meta0, const void* B0, int64_t ldb0, void* D0, int64_t ldd0, const int* d_row_map0,
                  int d_transposed0, const int* d_row_valid0, const void* a_vals1, const uint8_t* a_meta1,
                  const void* B1, int64_t ldb1, void* D1, int64_t ldd1, const int* d_row_map1, int d_transposed1,
                  const int* d_row_valid1, int64_t pair_rows, void* stream) {
  int rc = check_common(M, N, K, K, 0, ldb0, b_mn_major);
  if (rc) return rc;
  if ((rc = check_common(M, N, K, K, 0, ldb1, b_mn_major))) return rc;
  if (K % 128 != 0) return fail(S24_ERR_DIMENSION, "sparse K = %lld must be a multiple of 128", (long long)K);
  if ((!d_transposed0 && ldd0 < N) || (!d_transposed1 && ldd1 < N)) return fail(S24_ERR_DIMENSION, "ldd too small");
  if (pair_rows < 0 || pair_rows % 2 || pair_rows > M) return fail(S24_ERR_DIMENSION, "pair_rows must be even, <= M");
  return with_out(out_dtype, [&](auto tag) {
    using OutT = std::remove_pointer_t<decltype(tag)>;
    using Epi = EpiStore<OutT>;
    const int pr = static_cast<int>(pair_rows);
    typename Epi::Params ep0{static_cast<OutT*>(D0), ldd0, d_row_map0, d_transposed0, static_cast<int>(M),
                             d_row_valid0, 0, pr};
    GemmOperands<Epi> second{a_vals1, K / 2, B1, ldb1, a_meta1,
                             typename Epi::Params{static_cast<OutT*>(D1), ldd1, d_row_map1, d_transposed1,
                                                  static_cast<int>(M), d_row_valid1, 0, pr}};
    return dispatch_sparse<Epi>(b_mn_major, a_vals0, a_meta0, B0, ldb0, M, N, K, ep0,
                                static_cast<cudaStream_t>(stream), &second);
  });
}

int s24_fwd_gemm1_fused(const void* x, int64_t ldx, const void* w1, int64_t ldw1, int64_t M, int64_t N,
                        int64_t K, void* act_vals, uint8_t* act_meta, int* counts, unsigned long long* stats,
                        float* y_dbg, void* stream) {
  int rc = check_common(M, N, K, ldx, 0, ldw1, 1);
  if (rc) return rc;
  if (N % 128 != 0) return fail(S24_ERR_DIMENSION, "hidden width %lld must be a multiple of 128", (long long)N);
  if (!act_vals || !act_meta) return fail(S24_ERR_DIMENSION, "K1 needs the value and metadata buffers");
  EpiFwd1::Params ep{static_cast<__nv_bfloat16*>(act_vals), act_meta, counts, stats, y_dbg, static_cast<int>(N)};
  return launch_dense<DenseKN, DenseKN_W, EpiFwd1>(x, ldx, w1, ldw1, M, N, K, ep, static_cast<cudaStream_t>(stream));
}

int s24_bwd_dact_fused(const void* g, int64_t ldg, const void* w2, int64_t ldw2, int64_t M, int64_t N,
                       int64_t K, const void* act_vals, const uint8_t* act_meta, void* g_vals, void* stream) {
  int rc = check_common(M, N, K, ldg, 0, ldw2, 0);
  if (rc) return rc;
  if (N % 128 != 0) return fail(S24_ERR_DIMENSION, "hidden width %lld must be a multiple of 128", (long long)N);
  if (!act_vals || !act_meta || !g_vals) return fail(S24_ERR_DIMENSION, "K3 needs act, metadata and g_pre buffers");
  EpiBwd1::Params ep{static_cast<const __nv_bfloat16*>(act_vals), act_meta, static_cast<__nv_bfloat16*>(g_vals),
                     static_cast<int>(N)};
  return launch_gemm<DenseKK, EpiBwd1>(g, ldg, w2, ldw2, M, N, K, nullptr, ep, static_cast<cudaStream_t>(stream));
}

int s24_gemm_relu2(const void* x, int64_t ldx, const void* w1, int64_t ldw1, int64_t M, int64_t N, int64_t K,
                   void* act, int64_t ld_act, void* stream) {
  int rc = check_common(M, N, K, ldx, 0, ldw1, 1);
  if (rc) return rc;
  EpiRelu2::Params ep{static_cast<__nv_bfloat16*>(act), ld_act};
  return launch_dense<DenseKN, DenseKN_W, EpiRelu2>(x, ldx, w1, ldw1, M, N, K, ep, static_cast<cudaStream_t>(stream));
}

int s24_gemm_dact(const void* g, int64_t ldg, const void* w2, int64_t ldw2, int64_t M, int64_t N, int64_t K,
                  const void* act, int64_t ld_act, void* gpre, int64_t ld_g, void* stream) {
  int rc = check_common(M, N, K, ldg, 0, ldw2, 0);
  if (rc) return rc;
  EpiDact::Params ep{static_cast<const __nv_bfloat16*>(act), ld_act, static_cast<__nv_bfloat16*>(gpre), ld_g,
                     static_cast<int>(N)};
  return launch_gemm<DenseKK, EpiDact>(g, ldg, w2, ldw2, M, N, K, nullptr, ep, static_cast<cudaStream_t>(stream));
}


// ---------------------------------------------------------------------------
// e4m3 GEMMs (FfnConfig.fp8_emulation / fp8_backward on the tensor cores).
// Operands are e4m3 codes, K-major (A [M, K] or the 2:4 compressed [M, K/2]
// with e4m3-layout metadata, B as [N, K]); D = (row_scale x col_scale) * acc.

int s24_gemm_f8(const uint8_t* A, int64_t lda, const uint8_t* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                const float* row_scale, const float* col_scale, void* D, int out_dtype, int64_t ldd,
                const int* d_row_map, int d_transposed, int64_t d_rows_valid, void* stream) {
  int rc = check_common(M, N, K, lda, 0, ldb, 0);
  if (rc) return rc;
  if (!row_scale || !col_scale) return fail(S24_ERR_DIMENSION, "e4m3 GEMM needs row and column scales");
  if (K % 16 != 0) return fail(S24_ERR_DIMENSION, "e4m3 K = %lld must be a multiple of 16", (long long)K);
  if (!d_transposed && ldd < N) return fail(S24_ERR_DIMENSION, "ldd too small");
  return with_out(out_dtype, [&](auto tag) {
    using OutT = std::remove_pointer_t<decltype(tag)>;
    using Epi = EpiStore<OutT, true>;
    typename Epi::Params ep{static_cast<OutT*>(D), ldd, d_row_map, d_transposed,
                            static_cast<int>(d_rows_valid < 0 ? M : d_rows_valid), nullptr, 0, 0, row_scale,
                            col_scale};
    return launch_dense<F8DenseKK, F8DenseKK_W, Epi>(A, lda, B, ldb, M, N, K, ep, static_cast<cudaStream_t>(stream));
  });
}

int s24_spmm_f8(const uint8_t* a_codes, const uint8_t* a_meta_f8, const uint8_t* B, int64_t ldb, int64_t M,
                int64_t N, int64_t K, const float* row_scale, const float* col_scale, void* D, int out_dtype,
                int64_t ldd, const int* d_row_map, int d_transposed, int64_t d_rows_valid, const int* d_row_valid,
                int64_t pair_rows, void* stream) {
  int rc = check_common(M, N, K, K, 0, ldb, 0);
  if (rc) return rc;
  if (!row_scale || !col_scale) return fail(S24_ERR_DIMENSION, "e4m3 GEMM needs row and column scales");
  // (a stage spans 256 logical K; with K % 256 == 128 the last stage's second
  // half reads zero-filled A and B, whatever metadata sits next to it)
  if (K % 128 != 0) return fail(S24_ERR_DIMENSION, "sparse K = %lld must be a multiple of 128", (long long)K);
  if (!d_transposed && ldd < N) return fail(S24_ERR_DIMENSION, "ldd too small");
  if (pair_rows < 0 || pair_rows % 2 || pair_rows > M) return fail(S24_ERR_DIMENSION, "pair_rows must be even, <= M");
  return with_out(out_dtype, [&](auto tag) {
    using OutT = std::remove_pointer_t<decltype(tag)>;
    using Epi = EpiStore<OutT, true>;
    typename Epi::Params ep{static_cast<OutT*>(D), ldd, d_row_map, d_transposed,
                            static_cast<int>(d_rows_valid < 0 ? M : d_rows_valid), d_row_valid, 0,
                            static_cast<int>(pair_rows), row_scale, col_scale};
    return launch_gemm<F8SparseK, Epi>(a_codes, K / 2, B, ldb, M, N, K, a_meta_f8, ep,
                                       static_cast<cudaStream_t>(stream));
  });
}

int s24_spmm_pair_f8(int64_t M, int64_t N, int64_t K, int out_dtype, const uint8_t* a0, const uint8_t* meta0,
                     const uint8_t* B0, int64_t ldb0, const float* rs0, const float* cs0, void* D0, int64_t ldd0,
                     const int* d_row_map0, int d_transposed0, const int* d_row_valid0, const uint8_t* a1,
                     const uint8_t* meta1, const uint8_t* B1, int64_t ldb1, const float* rs1, const float* cs1,
                     void* D1, int64_t ldd1, const int* d_row_map1, int d_transposed1, const int* d_row_valid1,
                     int64_t pair_rows, void* stream) {
  int rc = check_common(M, N, K, K, 0, ldb0, 0);
  if (rc) return rc;
  if ((rc = check_common(M, N, K, K, 0, ldb1, 0))) return rc;
  if (!rs0 || !cs0 || !rs1 || !cs1) return fail(S24_ERR_DIMENSION, "e4m3 GEMM needs row and column scales");
  if (K % 128 != 0) return fail(S24_ERR_DIMENSION, "sparse K = %lld must be a multiple of 128", (long long)K);
  if ((!d_transposed0 && ldd0 < N) || (!d_transposed1 && ldd1 < N)) return fail(S24_ERR_DIMENSION, "ldd too small");
  if (pair_rows < 0 || pair_rows % 2 || pair_rows > M) return fail(S24_ERR_DIMENSION, "pair_rows must be even, <= M");
  return with_out(out_dtype, [&](auto tag) {
    using OutT = std::remove_pointer_t<decltype(tag)>;
    using Epi = EpiStore<OutT, true>;
    const int pr = static_cast<int>(pair_rows);
    typename Epi::Params ep0{static_cast<OutT*>(D0), ldd0, d_row_map0, d_transposed0, static_cast<int>(M),
                             d_row_valid0, 0, pr, rs0, cs0};
    GemmOperands<Epi> second{a1, K / 2, B1, ldb1, meta1,
                             typename Epi::Params{static_cast<OutT*>(D1), ldd1, d_row_map1, d_transposed1,
                                                  static_cast<int>(M), d_row_valid1, 0, pr, rs1, cs1}};
    return launch_gemm<F8SparseK, Epi>(a0, K / 2, B0, ldb0, M, N, K, meta0, ep0, static_cast<cudaStream_t>(stream),
                                       1, &second);
  });
}

int s24_fwd_gemm1_f8(const uint8_t* xq, int64_t ldx, const uint8_t* w1q, int64_t ldw1, int64_t M, int64_t N,
                     int64_t K, const float* x_scale, const float* w1_scale, float* act_vals32, unsigned* row_amax,
                     uint8_t* act_meta, int* counts, unsigned long long* stats, float* y_dbg, void* stream) {
  int rc = check_common(M, N, K, ldx, 0, ldw1, 0);
  if (rc) return rc;
  if (N % 128 != 0) return fail(S24_ERR_DIMENSION, "hidden width %lld must be a multiple of 128", (long long)N);
  if (K % 16 != 0) return fail(S24_ERR_DIMENSION, "e4m3 K = %lld must be a multiple of 16", (long long)K);
  if (!x_scale || !w1_scale || !act_vals32 || !row_amax)
    return fail(S24_ERR_DIMENSION, "e4m3 K1 needs scales, the fp32 value buffer and the row maxima");
  using Epi = EpiFwd1T<true>;
  Epi::Params ep{nullptr, act_meta, counts, stats, y_dbg, static_cast<int>(N), x_scale, w1_scale, act_vals32, row_amax};
  return launch_dense<F8DenseKK, F8DenseKK_W, Epi>(xq, ldx, w1q, ldw1, M, N, K, ep, static_cast<cudaStream_t>(stream));
}

int s24_bwd_dact_f8(const uint8_t* gq, int64_t ldg, const uint8_t* w2q, int64_t ldw2, int64_t M, int64_t N,
                    int64_t K, const float* g_scale, const float* w2_scale, const void* act_vals,
                    const uint8_t* act_meta, void* g_vals, void* stream) {
  int rc = check_common(M, N, K, ldg, 0, ldw2, 0);
  if (rc) return rc;
  if (N % 128 != 0) return fail(S24_ERR_DIMENSION, "hidden width %lld must be a multiple of 128", (long long)N);
  if (K % 16 != 0) return fail(S24_ERR_DIMENSION, "e4m3 K = %lld must be a multiple of 16", (long long)K);
  if (!g_scale || !w2_scale) return fail(S24_ERR_DIMENSION, "e4m3 K3 needs row and column scales");
  using Epi = EpiBwd1T<true>;
  Epi::Params ep{static_cast<const __nv_bfloat16*>(act_vals), act_meta, static_cast<__nv_bfloat16*>(g_vals),
                 static_cast<int>(N), g_scale, w2_scale};
  return launch_gemm<F8DenseKK, Epi>(gq, ldg, w2q, ldw2, M, N, K, nullptr, ep, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
