// bf16 tensor-core path (tcgen05 / TMA / TMEM), see lors_tc.cu.
#pragma once
#include "lors_common.cuh"

namespace lors {
size_t tc_fwd_workspace(const lors_fwd_args* a);
size_t tc_bwd_workspace(const lors_bwd_args* a);
int tc_fwd(const lors_fwd_args* a, cudaStream_t s);
int tc_bwd(const lors_bwd_args* a, cudaStream_t s);
}  // namespace lors
