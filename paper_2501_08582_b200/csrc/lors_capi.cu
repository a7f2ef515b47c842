// C-ABI entry points (include/lors_b200.h).  Validation mirrors the
// reference's error vocabulary (adapters.py:72-83, 117-137, 227-238):
// shape problems -> LORS_ERR_SHAPE, bad rank/alpha/mode -> LORS_ERR_ARGUMENT.
#include <cuda.h>

#include <cstdio>
#include <string>

#include "lors_common.cuh"
#include "lors_simt.cuh"
#include "lors_tc.cuh"

namespace lors {

static thread_local std::string t_last_error;
std::atomic<uint64_t> g_launch_count{0};

void set_error(const std::string& msg) { t_last_error = msg; }

static int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

// per-device capability cache: major*10+minor, 0 = unknown
static int g_cc[64];

static int device_cc() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return -1;
  if (g_cc[dev] == 0) {
    int maj = 0, min = 0;
    if (cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return -1;
    if (cudaDeviceGetAttribute(&min, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) return -1;
    g_cc[dev] = maj * 10 + min;
  }
  return g_cc[dev];
}

static int require_sm100() {
  const int cc = device_cc();
  if (cc != 100) {
    return fail(LORS_ERR_DEVICE, "lors_b200 kernels are built for sm_100a only; current device compute capability " +
                                     std::to_string(cc / 10) + "." + std::to_string(cc % 10));
  }
  return LORS_OK;
}

static int check_common(int64_t L, int64_t R, int64_t C, int64_t r, int32_t dtype, int32_t mask_mode,
                        float alpha, const uint32_t* bits) {
  if (L < 0 || R < 1 || C < 1) return fail(LORS_ERR_SHAPE, "dimensions must be positive (L >= 0, R, C >= 1)");
  if (r < 1 || r > (R < C ? R : C))
    return fail(LORS_ERR_ARGUMENT, "rank " + std::to_string(r) + " must satisfy 1 <= r <= min(" +
                                       std::to_string(R) + ", " + std::to_string(C) + ")");
  if (!(alpha > 0.0f)) return fail(LORS_ERR_ARGUMENT, "alpha must be positive");
  if (dtype != LORS_DTYPE_F32 && dtype != LORS_DTYPE_BF16) return fail(LORS_ERR_ARGUMENT, "unknown dtype");
  if (mask_mode != LORS_MASK_FROM_W && mask_mode != LORS_MASK_BITS)
    return fail(LORS_ERR_ARGUMENT, "unknown mask mode");
  if (mask_mode == LORS_MASK_BITS && bits == nullptr)
    return fail(LORS_ERR_ARGUMENT, "mask_mode BITS needs mask_bits");
  if (L > INT32_MAX || R > INT32_MAX || C > INT32_MAX || L * C > ((int64_t)1 << 40))
    return fail(LORS_ERR_SHAPE, "dimensions too large");
  return LORS_OK;
}

}  // namespace lors

using namespace lors;
using bf16 = __nv_bfloat16;

extern "C" {

const char* lors_last_error(void) { return t_last_error.c_str(); }
int lors_abi_version(void) { return LORS_ABI_VERSION; }
int lors_device_check(void) { return require_sm100(); }
uint64_t lors_launch_count(void) { return g_launch_count.load(); }
void lors_reset_launch_count(void) { g_launch_count.store(0); }

size_t lors_fwd_workspace(const lors_fwd_args* a) {
  if (a == nullptr) return 0;
  return tc_fwd_workspace(a);
}

size_t lors_bwd_workspace(const lors_bwd_args* a) {
  if (a == nullptr) return 0;
  if (a->flags & LORS_FLAG_DX_ONLY) return tc_bwd_workspace(a);
  // P (when not supplied) and Q, fp32-sized slots, 256-byte aligned
  const size_t slot = ((size_t)a->L * (size_t)a->r * sizeof(float) + 255) / 256 * 256;
  return 2 * slot + tc_bwd_workspace(a);
}

int lors_fwd(const lors_fwd_args* A, void* stream) {
  if (A == nullptr) return fail(LORS_ERR_ARGUMENT, "null args");
  int st = check_common(A->L, A->R, A->C, A->r, A->dtype, A->mask_mode, A->alpha, A->mask_bits);
  if (st) return st;
  if (!A->w || !A->a || !A->b) return fail(LORS_ERR_ARGUMENT, "null tensor pointer");
  if (A->L > 0 && (!A->x || !A->y)) return fail(LORS_ERR_ARGUMENT, "null tensor pointer");
  if (A->L > 0 && (A->flags & LORS_FLAG_EMIT_P) && !A->p) return fail(LORS_ERR_ARGUMENT, "EMIT_P needs p");
  if ((st = require_sm100())) return st;
  if (A->L == 0) return LORS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int L = (int)A->L, R = (int)A->R, C = (int)A->C, r = (int)A->r;
  const uint32_t* bits = A->mask_mode == LORS_MASK_BITS ? A->mask_bits : nullptr;
  if (A->dtype == LORS_DTYPE_F32) {
    if (A->flags & LORS_FLAG_SPARSE24) return fail(LORS_ERR_ARGUMENT, "2:4 sparse tensor cores need bf16");
    const float *x = (const float*)A->x, *w = (const float*)A->w, *a = (const float*)A->a, *b = (const float*)A->b;
    // tensor cores (3xTF32) where TMA can address the fp32 rows, else the FFMA kernels
    st = tf32x3_lors_gemm(false, x, w, a, b, bits, (const float*)A->bias, (float*)A->y, L, R, C, r, A->alpha, s);
    if (st == LORS_ERR_SHAPE)
      st = simt_lors_gemm<float>(false, x, w, bits, a, b, (const float*)A->bias, (float*)A->y, L, R, C, r, A->alpha, s);
    if (st) return st;
    if (A->flags & LORS_FLAG_EMIT_P) {  // P[l, j] = sum_c X_t[l, c] b[j, c], one warp a row (deterministic)
      st = s4_rank_project(x, C, b, C, 1, (float*)A->p, L, C, r, true, s);
      if (st == LORS_ERR_SHAPE)
        st = simt_strided_gemm<float, float, float>(x, C, 1, b, C, 1, (float*)A->p, r, 1, L, r, C, 1.0f, false, s);
    }
    return st;
  }
  return tc_fwd(A, s);
}

size_t lors_fwd_group_workspace(const lors_fwd_args* a, int32_t groups) {
  if (a == nullptr) return 0;
  return tc_fwd_group_workspace(a, groups);
}

int lors_fwd_group(const lors_fwd_args* A, int32_t groups, void* stream) {
  if (A == nullptr) return fail(LORS_ERR_ARGUMENT, "null args");
  int st = check_common(A->L, A->R, A->C, A->r, A->dtype, A->mask_mode, A->alpha, A->mask_bits);
  if (st) return st;
  if (!tc_fwd_group_ok(A, groups))
    return fail(LORS_ERR_ARGUMENT, "grouped forward needs bf16, FROM_W, no bias / SPARSE24 / EMIT_P, R % 256 == 0, "
                                   "C % 8 == 0, r in {16, 32, 64} and groups >= 1");
  if (!A->w || !A->a || !A->b) return fail(LORS_ERR_ARGUMENT, "null tensor pointer");
  if (A->L > 0 && (!A->x || !A->y)) return fail(LORS_ERR_ARGUMENT, "null tensor pointer");
  if ((st = require_sm100())) return st;
  if (A->L == 0) return LORS_OK;
  return tc_fwd_group(A, groups, (cudaStream_t)stream);
}

int lors_bwd(const lors_bwd_args* A, void* stream) {
  if (A == nullptr) return fail(LORS_ERR_ARGUMENT, "null args");
  int st = check_common(A->L, A->R, A->C, A->r, A->dtype, A->mask_mode, A->alpha, A->mask_bits);
  if (st) return st;
  if (A->grad_mode != LORS_GRAD_STE && A->grad_mode != LORS_GRAD_MASKED)
    return fail(LORS_ERR_ARGUMENT, "unknown grad_mode");
  const bool dx_only = (A->flags & LORS_FLAG_DX_ONLY) != 0;
  if (dx_only && (A->flags & LORS_FLAG_NO_DX)) return fail(LORS_ERR_ARGUMENT, "DX_ONLY and NO_DX together");
  if (!A->w || !A->a || !A->b || (!dx_only && (!A->da || !A->db)))
    return fail(LORS_ERR_ARGUMENT, "null tensor pointer");
  if (A->L > 0 && (!A->x || !A->dy)) return fail(LORS_ERR_ARGUMENT, "null tensor pointer");
  if (A->L > 0 && !(A->flags & LORS_FLAG_NO_DX) && !A->dx) return fail(LORS_ERR_ARGUMENT, "dx is null");
  if (A->workspace_bytes < lors_bwd_workspace(A) || (A->workspace == nullptr && lors_bwd_workspace(A) > 0))
    return fail(LORS_ERR_ARGUMENT, "workspace too small: need " + std::to_string(lors_bwd_workspace(A)) + " bytes");
  if ((st = require_sm100())) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const int L = (int)A->L, R = (int)A->R, C = (int)A->C, r = (int)A->r;
  if (L == 0) {
    if (dx_only) return LORS_OK;
    LORS_CUDA_TRY(cudaMemsetAsync(A->da, 0, sizeof(float) * R * r, s), "zero dA");
    LORS_CUDA_TRY(cudaMemsetAsync(A->db, 0, sizeof(float) * r * C, s), "zero dB");
    if (A->dbias) LORS_CUDA_TRY(cudaMemsetAsync(A->dbias, 0, sizeof(float) * R, s), "zero dbias");
    return LORS_OK;
  }
  const uint32_t* bits = A->mask_mode == LORS_MASK_BITS ? A->mask_bits : nullptr;
  if (A->dtype == LORS_DTYPE_F32) {
    const float *x = (const float*)A->x, *w = (const float*)A->w, *a = (const float*)A->a,
                *b = (const float*)A->b, *dy = (const float*)A->dy;
    if (!(A->flags & LORS_FLAG_NO_DX)) {  // dX_t = dY_t W_eff  (adapters.py:395)
      st = tf32x3_lors_gemm(true, dy, w, a, b, bits, nullptr, (float*)A->dx, L, R, C, r, A->alpha, s);
      if (st == LORS_ERR_SHAPE)
        st = simt_lors_gemm<float>(true, dy, w, bits, a, b, nullptr, (float*)A->dx, L, R, C, r, A->alpha, s);
      if (st) return st;
    }
    if (dx_only) return LORS_OK;
    if (A->grad_mode == LORS_GRAD_STE) {
      // fast mode splits every product along its reduction (fp32 atomics into a zeroed output;
      // P and Q have only L / 64 row tiles); LORS_FLAG_DETERMINISTIC keeps one CTA per output
      // tile, summed in k order, so dA / dB are bitwise reproducible
      const bool split = (A->flags & LORS_FLAG_DETERMINISTIC) == 0;
      const size_t slot = ((size_t)L * r * sizeof(float) + 255) / 256 * 256;
      float* P = (float*)A->p;
      float* Q = (float*)((char*)A->workspace + slot);
      // S4 streams X / dY once per product (P and Q: one warp a row, no atomics when deterministic;
      // dA and dB: L split with fp32 atomics, fast mode only); S2 covers the rest
      if (P == nullptr) {  // xt_bt = X^T b^T  (adapters.py:396)
        P = (float*)A->workspace;
        st = s4_rank_project(x, C, b, C, 1, P, L, C, r, !split, s);
        if (st == LORS_ERR_SHAPE)
          st = simt_strided_gemm<float, float, float>(x, C, 1, b, C, 1, P, r, 1, L, r, C, 1.0f, split, s);
        if (st) return st;
      }
      // at_dy = a^T dY (adapters.py:397): Q[l, j] = sum_n dY_t[l, n] a[n, j]
      st = s4_rank_project(dy, R, a, 1, r, Q, L, R, r, !split, s);
      if (st == LORS_ERR_SHAPE)
        st = simt_strided_gemm<float, float, float>(dy, R, 1, a, 1, r, Q, r, 1, L, r, R, 1.0f, split, s);
      if (st) return st;
      // da = alpha dY xt_bt (adapters.py:398): dA[n, j] = alpha sum_l dY_t[l, n] P[l, j]
      st = split ? s4_rank_accumulate(dy, R, P, A->da, r, 1, L, R, r, A->alpha, s) : LORS_ERR_SHAPE;
      if (st == LORS_ERR_SHAPE)
        st = simt_strided_gemm<float, float, float>(dy, 1, R, P, 1, r, A->da, r, 1, R, r, L, A->alpha, split, s);
      if (st) return st;
      // db = alpha at_dy X^T (adapters.py:399): dB[j, c] = alpha sum_l Q[l, j] X_t[l, c]
      st = split ? s4_rank_accumulate(x, C, Q, A->db, 1, C, L, C, r, A->alpha, s) : LORS_ERR_SHAPE;
      if (st == LORS_ERR_SHAPE)
        st = simt_strided_gemm<float, float, float>(Q, 1, r, x, 1, C, A->db, C, 1, r, C, L, A->alpha, split, s);
      if (st) return st;
    } else {
      st = simt_masked_grad<float>(dy, x, w, bits, a, b, A->da, A->db, L, R, C, r, A->alpha, s);
      if (st) return st;
    }
    if (A->dbias) {
      st = colsum<float>(dy, A->dbias, L, R, s);
      if (st) return st;
    }
    if (A->flags & LORS_FLAG_FAULT_DA_SIGN) return negate_f32(A->da, (int64_t)R * r, s);
    return LORS_OK;
  }
  return tc_bwd(A, s);
}

int lors_effective_weight(int64_t R, int64_t C, int64_t r, int32_t dtype, int32_t mask_mode, float alpha,
                          const void* w, const uint32_t* mask_bits, const void* a, const void* b, void* out,
                          void* stream) {
  int st = check_common(0, R, C, r, dtype, mask_mode, alpha, mask_bits);
  if (st) return st;
  if (!w || !a || !b || !out) return fail(LORS_ERR_ARGUMENT, "null tensor pointer");
  if ((st = require_sm100())) return st;
  const uint32_t* bits = mask_mode == LORS_MASK_BITS ? mask_bits : nullptr;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == LORS_DTYPE_F32)
    return effective_weight<float>((const float*)w, bits, (const float*)a, (const float*)b, (float*)out, (int)R,
                                   (int)C, (int)r, alpha, s);
  return tc_effective_weight((const bf16*)w, bits, (const bf16*)a, (const bf16*)b, (bf16*)out, (int)R, (int)C,
                             (int)r, alpha, s);
}

int lors_pack_mask(int64_t R, int64_t C, int32_t dtype, const void* w, uint32_t* bits, void* stream) {
  if (R < 1 || C < 1) return fail(LORS_ERR_SHAPE, "dimensions must be positive");
  if (!w || !bits) return fail(LORS_ERR_ARGUMENT, "null tensor pointer");
  int st;
  if ((st = require_sm100())) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == LORS_DTYPE_F32) return pack_mask<float>((const float*)w, bits, (int)R, (int)C, s);
  if (dtype == LORS_DTYPE_BF16) return pack_mask<bf16>((const bf16*)w, bits, (int)R, (int)C, s);
  return fail(LORS_ERR_ARGUMENT, "unknown dtype");
}

int lors_compress_24(int64_t R, int64_t C, int32_t dtype, const void* w, void* values, uint8_t* meta,
                     int32_t* invalid, void* stream) {
  if (R < 1 || C < 1) return fail(LORS_ERR_SHAPE, "dimensions must be positive");
  if (C % 8) return fail(LORS_ERR_SHAPE, "2:4 compression needs C % 8 == 0");
  if (!w || !values || !meta) return fail(LORS_ERR_ARGUMENT, "null tensor pointer");
  int st;
  if ((st = require_sm100())) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (invalid) LORS_CUDA_TRY(cudaMemsetAsync(invalid, 0, sizeof(int32_t), s), "zero invalid flag");
  if (dtype == LORS_DTYPE_F32)
    return compress24<float>((const float*)w, (float*)values, meta, invalid, (int)R, (int)C, s);
  if (dtype == LORS_DTYPE_BF16)
    return compress24<bf16>((const bf16*)w, (bf16*)values, meta, invalid, (int)R, (int)C, s);
  return fail(LORS_ERR_ARGUMENT, "unknown dtype");
}

int lors_grad_outer(int64_t L, int64_t R, int64_t C, int32_t dtype, int32_t masked, const void* dy, const void* x,
                    const void* w, float* dw, void* stream) {
  if (L < 1 || R < 1 || C < 1) return fail(LORS_ERR_SHAPE, "dimensions must be positive");
  if (!dy || !x || !dw || (masked && !w)) return fail(LORS_ERR_ARGUMENT, "null tensor pointer");
  int st;
  if ((st = require_sm100())) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == LORS_DTYPE_F32)
    return grad_outer<float>((const float*)dy, (const float*)x, (const float*)w, dw, (int)L, (int)R, (int)C, masked,
                             s);
  if (dtype == LORS_DTYPE_BF16)
    return grad_outer<bf16>((const bf16*)dy, (const bf16*)x, (const bf16*)w, dw, (int)L, (int)R, (int)C, masked, s);
  return fail(LORS_ERR_ARGUMENT, "unknown dtype");
}

}  // extern "C"
