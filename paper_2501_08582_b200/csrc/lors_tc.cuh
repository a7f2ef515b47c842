// bf16 tensor-core path (tcgen05 / TMA / TMEM), see lors_tc.cu.
#pragma once
#include "lors_common.cuh"

namespace lors {
size_t tc_fwd_workspace(const lors_fwd_args* a);
size_t tc_bwd_workspace(const lors_bwd_args* a);
int tc_fwd(const lors_fwd_args* a, cudaStream_t s);
bool tc_fwd_group_ok(const lors_fwd_args* a, int groups);
size_t tc_fwd_group_workspace(const lors_fwd_args* a, int groups);
int tc_fwd_group(const lors_fwd_args* a, int groups, cudaStream_t s);
int tc_bwd(const lors_bwd_args* a, cudaStream_t s);
bool tc_shape_ok(int64_t R, int64_t C, int64_t r);
// fp32 parity mode on the tensor cores (3xTF32): forward (dx = false, act = X_t) or dX (act = dY_t);
// LORS_ERR_SHAPE when the shapes need the FFMA kernels
int tf32x3_lors_gemm(bool dx, const float* act, const float* w, const float* a, const float* b, const uint32_t* bits,
                     const float* bias, float* out, int L, int R, int C, int r, float alpha, cudaStream_t s);
// bf16 W_eff through the forward's tensor-core prologue (FFMA kernel for shapes TMA cannot address)
int tc_effective_weight(const __nv_bfloat16* w, const uint32_t* bits, const __nv_bfloat16* a, const __nv_bfloat16* b,
                        __nv_bfloat16* out, int R, int C, int r, float alpha, cudaStream_t s);
}  // namespace lors
