// Experiment (tools only): HBM streaming rate of TMA box loads into a shared-memory
// ring, no compute -- what the HBM-bound rank-r kernels can expect per SM.
//   tma_bw <rows> <cols> <box_rows> <boxes_per_stage> <stages> <ctas_per_sm>
// Reads a [rows x cols] bf16 matrix once: CTA c takes row tiles c, c + grid, ...; per
// row tile it walks the columns in stages of boxes_per_stage adjacent 64-column boxes.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include "../../paper_2501_08582_b200/csrc/ptx_sm100.cuh"
using namespace lors::ptx;

__global__ void stream_kernel(const __grid_constant__ CUtensorMap m, int rows, int cols, int box_rows, int bps,
                              int stages, int col_chunks, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t box_bytes = box_rows * 128, stage_bytes = box_bytes * bps;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int n_rt = (rows + box_rows - 1) / box_rows, n_st_all = (cols / 64 + bps - 1) / bps;
  const int n_st = (n_st_all + col_chunks - 1) / col_chunks;
  int i = 0;
  unsigned long long acc = 0;
  // keep `stages` stages in flight: issue stage i, wait for stage i - stages + 1
  for (int u = blockIdx.x; u < n_rt * col_chunks; u += gridDim.x)
    for (int st = (u % col_chunks) * n_st, rt = u / col_chunks; st < min(n_st_all, (u % col_chunks + 1) * n_st); ++st, ++i) {
      const int s = i % stages;
      if (i >= stages) {
        mbar_wait(&full[s], ((i / stages) - 1) & 1);
        acc += smem[s * stage_bytes];
      }
      mbar_arrive_expect_tx(&full[s], stage_bytes);
      for (int b = 0; b < bps; ++b) tma_load_2d(smem + s * stage_bytes + b * box_bytes, &m, &full[s], (st * bps + b) * 64, rt * box_rows);
    }
  for (int j = (i > stages ? i - stages : 0); j < i; ++j) mbar_wait(&full[j % stages], (j / stages) & 1);
  if (acc == 12345) *sink = acc;
}

typedef CUresult (*PFN_encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                               const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  if (argc < 8) { printf("usage: tma_bw rows cols box_rows boxes_per_stage stages ctas_per_sm col_chunks\n"); return 1; }
  const int rows = atoi(argv[1]), cols = atoi(argv[2]), box_rows = atoi(argv[3]), bps = atoi(argv[4]),
            stages = atoi(argv[5]), cps = atoi(argv[6]), cc = atoi(argv[7]);
  void* d; cudaMalloc(&d, (size_t)rows * cols * 2); cudaMemset(d, 1, (size_t)rows * cols * 2);
  void* flush; cudaMalloc(&flush, 512ull << 20);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  PFN_encode enc = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows}, es[2] = {1, 1};
  if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n"); return 1;
  }
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = 1024 + (size_t)stages * box_rows * 128 * bps + 8 * stages;
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int it = 0; it < 6; ++it) {
    cudaMemsetAsync(flush, it, 512ull << 20);
    cudaEventRecord(e0);
    stream_kernel<<<nsm * cps, 32, smem>>>(m, rows, cols, box_rows, bps, stages, cc, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (it > 0 && ms < best) best = ms;
  }
  cudaError_t err = cudaGetLastError();
  printf("rows %d cols %d box %dx64 x%d stages %d ctas/sm %d col chunks %d smem %zu KB: %.1f us, %.0f GB/s (%s)\n",
         rows, cols, box_rows, bps, stages, cps, cc, smem / 1024, best * 1e3, (double)rows * cols * 2 / (best * 1e-3) / 1e9,
         cudaGetErrorString(err));
  return 0;
}
