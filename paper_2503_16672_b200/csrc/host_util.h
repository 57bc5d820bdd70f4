// Host-side helpers shared by the C-ABI translation units: thread-local error
// text, status codes, TMA tensor-map encoding through the driver entry point
// (no link-time libcuda dependency) and device attribute caching.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <string>

#include "../../include/s24.h"

namespace s24 {

std::string& last_error_ref();

inline int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  last_error_ref() = buf;
  return code;
}

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(S24_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return S24_OK;
}

int num_sms();

// 2-D bf16 tensor map: inner dim (contiguous) `inner` elements, `outer` rows,
// row pitch `ld` elements; box {box_inner, box_outer}; `swizzle` = 128, 64
// (bytes) or 0 for none.
int make_map_2d(CUtensorMap* map, const void* base, bool bf16, uint64_t inner, uint64_t outer, uint64_t ld_bytes,
                uint32_t box_inner, uint32_t box_outer, int swizzle);
int make_map_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
                  uint32_t box_inner, uint32_t box_outer, int swizzle);

// The device's greatest (most urgent) launch priority. Every kernel of the
// FFN's critical path launches at it (the GEMMs, the row gathers, the plan);
// K4, which the recipe runs on side streams next to them, keeps the default,
// so the block scheduler places critical-path CTAs first and K4 fills the
// room they leave.
inline int high_priority() {
  static const int prio = [] {
    int least = 0, greatest = 0;
    if (cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) return 0;
    return greatest;
  }();
  return prio;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_high(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, size_t smem,
                               Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = st;
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributePriority;
  at[0].val.priority = high_priority();
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

struct K4Args;
int k4_prepare(const void* vals, const uint8_t* meta_hw, int64_t n, int64_t h, const int* feat_pos,
               int64_t n_sparse, int64_t n_dense, void* vs, uint8_t* es, void* vd, cudaStream_t st, K4Args* out,
               int64_t pair_rows = -1);

}  // namespace s24
