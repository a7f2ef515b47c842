// Declarations of the SIMT (FFMA) kernels; see lors_simt.cu.
#pragma once
#include "lors_common.cuh"

namespace lors {

template <typename T>
int simt_lors_gemm(bool dx, const T* act, const T* w, const uint32_t* bits, const T* a, const T* b,
                   const T* bias, T* out, int L, int R, int C, int r, float alpha, cudaStream_t s);

template <typename TA, typename TB, typename TO>
int simt_strided_gemm(const TA* A, int64_t sam, int64_t sak, const TB* B, int64_t sbn, int64_t sbk,
                      TO* out, int64_t som, int64_t son, int M, int N, int K, float alpha,
                      bool allow_split, cudaStream_t s);

// S4: fp32 rank-r products streamed at the HBM rate (LORS_ERR_SHAPE when N, ldy or Y are not float4-aligned)
int s4_rank_project(const float* Y, int64_t ldy, const float* Fm, int64_t sfj, int64_t sfn, float* out, int L,
                    int N, int r, bool deterministic, cudaStream_t s);
int s4_rank_accumulate(const float* Y, int64_t ldy, const float* Sm, float* out, int64_t son, int64_t soj, int L,
                       int N, int r, float alpha, cudaStream_t s);

template <typename T>
int simt_masked_grad(const T* dy, const T* x, const T* w, const uint32_t* bits, const T* a,
                     const T* b, float* da, float* db, int L, int R, int C, int r, float alpha,
                     cudaStream_t s);

template <typename T>
int colsum(const T* dy, float* out, int L, int R, cudaStream_t s);
template <typename T>
int effective_weight(const T* w, const uint32_t* bits, const T* a, const T* b, T* out, int R, int C,
                     int r, float alpha, cudaStream_t s);
template <typename T>
int pack_mask(const T* w, uint32_t* bits, int R, int C, cudaStream_t s);
template <typename T>
int compress24(const T* w, T* vals, uint8_t* meta, int32_t* invalid, int R, int C, cudaStream_t s);
template <typename T>
int grad_outer(const T* dy, const T* x, const T* w, float* dw, int L, int R, int C, int masked,
               cudaStream_t s);
int negate_f32(float* p, int64_t n, cudaStream_t s);

}  // namespace lors
