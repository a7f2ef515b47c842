// Micro test: TMA load of a [128 rows x 16 bytes] uint8 box (no swizzle) into shared memory,
// in a 2-CTA cluster kernel, completing on an mbarrier.  nvcc -arch=sm_100a tma_u8.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void __cluster_dims__(2, 1, 1) k(const __grid_constant__ CUtensorMap m, int x, uint32_t* out) {
  __shared__ alignas(1024) uint8_t buf[2048];
  __shared__ alignas(8) uint64_t bar;
  uint32_t sb = (uint32_t)__cvta_generic_to_shared(&bar), sd = (uint32_t)__cvta_generic_to_shared(buf);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(2048));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(sd),
        "l"(reinterpret_cast<uint64_t>(&m)), "r"(sb), "r"(x), "r"(0));
  }
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(sb));
  if (blockIdx.x == 0) out[threadIdx.x] = reinterpret_cast<uint32_t*>(buf)[threadIdx.x * 4];
}

typedef CUresult (*enc_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const int R = 512, W = 48;
  std::vector<uint8_t> h(R * W);
  for (int i = 0; i < R * W; ++i) h[i] = (uint8_t)(i * 7 + 3);
  uint8_t* d;
  uint32_t* o;
  cudaMalloc(&d, R * W);
  cudaMalloc(&o, 128 * 4);
  cudaMemcpy(d, h.data(), R * W, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[2] = {W, R}, str[1] = {W};
  cuuint32_t box[2] = {16, 128}, es[2] = {1, 1};
  CUresult r = ((enc_t)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  for (int x : {0, 8, 40}) {
    k<<<2, 128>>>(m, x, o);
    cudaError_t e = cudaDeviceSynchronize();
    printf("x=%d: %s\n", x, cudaGetErrorString(e));
    if (e) return 1;
    std::vector<uint32_t> ho(128);
    cudaMemcpy(ho.data(), o, 512, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int row = 0; row < 128; ++row) {
      uint32_t want = 0;
      for (int b = 0; b < 4; ++b) want |= (uint32_t)(x + b < W ? h[row * W + x + b] : 0) << (8 * b);
      bad += ho[row] != want;
    }
    printf("  bad rows %d (row0 %08x)\n", bad, ho[0]);
  }
  return 0;
}
