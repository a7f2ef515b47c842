// bf16 path -- placeholder routing to the SIMT kernels until the tcgen05
// kernels land.
#include "lors_simt.cuh"
#include "lors_tc.cuh"

namespace lors {
using bf16 = __nv_bfloat16;

size_t tc_fwd_workspace(const lors_fwd_args*) { return 0; }
size_t tc_bwd_workspace(const lors_bwd_args*) { return 0; }

int tc_fwd(const lors_fwd_args* A, cudaStream_t s) {
  const int L = (int)A->L, R = (int)A->R, C = (int)A->C, r = (int)A->r;
  const uint32_t* bits = A->mask_mode == LORS_MASK_BITS ? A->mask_bits : nullptr;
  const bf16 *x = (const bf16*)A->x, *w = (const bf16*)A->w, *a = (const bf16*)A->a, *b = (const bf16*)A->b;
  int st = simt_lors_gemm<bf16>(false, x, w, bits, a, b, (const bf16*)A->bias, (bf16*)A->y, L, R, C, r, A->alpha, s);
  if (st) return st;
  if (A->flags & LORS_FLAG_EMIT_P)
    st = simt_strided_gemm<bf16, bf16, bf16>(x, C, 1, b, C, 1, (bf16*)A->p, r, 1, L, r, C, 1.0f, false, s);
  return st;
}

int tc_bwd(const lors_bwd_args* A, cudaStream_t s) {
  const int L = (int)A->L, R = (int)A->R, C = (int)A->C, r = (int)A->r;
  const uint32_t* bits = A->mask_mode == LORS_MASK_BITS ? A->mask_bits : nullptr;
  const bf16 *x = (const bf16*)A->x, *w = (const bf16*)A->w, *a = (const bf16*)A->a, *b = (const bf16*)A->b,
             *dy = (const bf16*)A->dy;
  int st;
  if (!(A->flags & LORS_FLAG_NO_DX)) {
    st = simt_lors_gemm<bf16>(true, dy, w, bits, a, b, nullptr, (bf16*)A->dx, L, R, C, r, A->alpha, s);
    if (st) return st;
  }
  if (A->grad_mode == LORS_GRAD_STE) {
    const size_t slot = ((size_t)L * r * sizeof(float) + 255) / 256 * 256;
    bf16* P = (bf16*)A->p;
    bf16* Q = (bf16*)((char*)A->workspace + slot);
    if (P == nullptr) {
      P = (bf16*)A->workspace;
      st = simt_strided_gemm<bf16, bf16, bf16>(x, C, 1, b, C, 1, P, r, 1, L, r, C, 1.0f, false, s);
      if (st) return st;
    }
    st = simt_strided_gemm<bf16, bf16, bf16>(dy, R, 1, a, 1, r, Q, r, 1, L, r, R, 1.0f, false, s);
    if (st) return st;
    st = simt_strided_gemm<bf16, bf16, float>(dy, 1, R, P, 1, r, A->da, r, 1, R, r, L, A->alpha, true, s);
    if (st) return st;
    st = simt_strided_gemm<bf16, bf16, float>(Q, 1, r, x, 1, C, A->db, C, 1, r, C, L, A->alpha, true, s);
    if (st) return st;
  } else {
    st = simt_masked_grad<bf16>(dy, x, w, bits, a, b, A->da, A->db, L, R, C, r, A->alpha, s);
    if (st) return st;
  }
  if (A->dbias) {
    st = colsum<bf16>(dy, A->dbias, L, R, s);
    if (st) return st;
  }
  if (A->flags & LORS_FLAG_FAULT_DA_SIGN) return negate_f32(A->da, (int64_t)R * r, s);
  return LORS_OK;
}
}  // namespace lors
