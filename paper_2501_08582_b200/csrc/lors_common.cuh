// Shared helpers for the LoRS B200 kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "../../include/lors_b200.h"

namespace lors {

// ---------------------------------------------------------------------------
// error plumbing (thread-local message, status codes of lors_b200.h)
// ---------------------------------------------------------------------------
void set_error(const std::string& msg);
extern std::atomic<uint64_t> g_launch_count;

inline void count_launch(uint64_t n = 1) { g_launch_count.fetch_add(n, std::memory_order_relaxed); }

#define LORS_CHECK_LAUNCH(what)                                              \
  do {                                                                       \
    cudaError_t e__ = cudaGetLastError();                                    \
    if (e__ != cudaSuccess) {                                                \
      ::lors::set_error(std::string(what) + ": " + cudaGetErrorString(e__)); \
      return LORS_ERR_CUDA;                                                  \
    }                                                                        \
    ::lors::count_launch();                                                  \
  } while (0)

#define LORS_CUDA_TRY(expr, what)                                            \
  do {                                                                       \
    cudaError_t e__ = (expr);                                                \
    if (e__ != cudaSuccess) {                                                \
      ::lors::set_error(std::string(what) + ": " + cudaGetErrorString(e__)); \
      return LORS_ERR_CUDA;                                                  \
    }                                                                        \
  } while (0)

// ---------------------------------------------------------------------------
// element access
// ---------------------------------------------------------------------------
__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// Round a float to the storage precision of T (identity for fp32).
template <typename T>
__device__ __forceinline__ float round_to(float v) { return to_f(from_f<T>(v)); }

// Mask predicate M(row, col): (W != 0) from the value itself, or a packed bit.
template <typename T>
__device__ __forceinline__ bool mask_at(const T w, const uint32_t* __restrict__ bits,
                                        int64_t words_per_row, int64_t row, int64_t col) {
  if (bits != nullptr) return (__ldg(bits + row * words_per_row + (col >> 5)) >> (col & 31)) & 1u;
  return to_f(w) != 0.0f;
}

// The effective-weight element of the FFMA kernels (fp32 mode, K6 fp32, shapes TMA
// cannot address), rounded to the storage type T by the caller:
//   fp32: select(M, fma(alpha, p, w), +0.0)
//   bf16: select(M, bf16(w + bf16(alpha p)), +0.0)  -- the tensor-core weff_pair's arithmetic
// `select`, not multiplication, so pruned entries are bit-exact +0.0 (reference
// merged_weight adapters.py:214-224 yields +0.0 there because W is normalised to +0.0,
// prune.py:47; (w + alpha*p)*0 could give -0.0).
template <typename T>
__device__ __forceinline__ float weff_value(bool keep, float w, float p, float alpha) {
  if (!keep) return 0.0f;
  if (sizeof(T) == 2) return w + round_to<T>(alpha * p);
  return fmaf(alpha, p, w);
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace lors
