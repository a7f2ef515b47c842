// Experiment (tools only): L2 -> SM rate of TMA box loads when the data is L2-resident (the
// regime of the LoRS GEMMs, whose W and activation panels are re-read from L2 by many CTAs).
//   l2_bw <rows> <cols> <box_rows> <stages> <ctas_per_sm> <reps> <stagger>
// Every CTA streams the whole [rows x cols] bf16 matrix `reps` times through a `stages`-deep
// ring of [box_rows x 64] SW128 boxes; stagger = 1 starts CTA c at box c (no two SMs ask for
// the same line at the same time), 0 = all CTAs walk the same sequence.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include "../../paper_2501_08582_b200/csrc/ptx_sm100.cuh"
using namespace lors::ptx;

__global__ void l2_kernel(const __grid_constant__ CUtensorMap m, int n_boxes, int col_boxes, int box_rows, int stages,
                          int reps, int stagger, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t box_bytes = box_rows * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * box_bytes);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  // `issuers` threads (one per warp) each own every issuers-th stage of the ring
  const int issuers = blockDim.x / 32, me = threadIdx.x / 32;
  if (threadIdx.x % 32 != 0) return;
  unsigned long long acc = 0;
  const int total = n_boxes * reps, start = stagger ? (int)(blockIdx.x * 7919) % n_boxes : 0;
  for (int i = me; i < total; i += issuers) {
    const int s = i % stages;
    if (i >= stages) {
      mbar_wait(&full[s], ((i / stages) - 1) & 1);
      acc += smem[s * box_bytes];
    }
    const int b = (start + i) % n_boxes;
    mbar_arrive_expect_tx(&full[s], box_bytes);
    tma_load_2d(smem + s * box_bytes, &m, &full[s], (b % col_boxes) * 64, (b / col_boxes) * box_rows);
  }
  for (int j = (total > stages ? total - stages : 0); j < total; ++j)
    if (j % issuers == me) mbar_wait(&full[j % stages], (j / stages) & 1);
  if (acc == 12345) *sink = acc;
}

typedef CUresult (*PFN_encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                               const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  if (argc < 8) { printf("usage: l2_bw rows cols box_rows stages ctas_per_sm reps stagger [issuers]\n"); return 1; }
  const int issuers = argc > 8 ? atoi(argv[8]) : 1;
  const int rows = atoi(argv[1]), cols = atoi(argv[2]), box_rows = atoi(argv[3]), stages = atoi(argv[4]),
            cps = atoi(argv[5]), reps = atoi(argv[6]), stagger = atoi(argv[7]);
  void* d; cudaMalloc(&d, (size_t)rows * cols * 2); cudaMemset(d, 1, (size_t)rows * cols * 2);
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
  const int col_boxes = cols / 64, n_boxes = col_boxes * (rows / box_rows);
  const size_t smem = 1024 + (size_t)stages * box_rows * 128 + 8 * stages;
  cudaFuncSetAttribute(l2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int it = 0; it < 5; ++it) {
    cudaEventRecord(e0);
    l2_kernel<<<nsm * cps, 32 * issuers, smem>>>(m, n_boxes, col_boxes, box_rows, stages, reps, stagger, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (it > 0 && ms < best) best = ms;
  }
  cudaError_t err = cudaGetLastError();
  const double bytes = (double)nsm * cps * rows * cols * 2 * reps;
  printf("l2 issuers %d rows %d cols %d box %dx64 stages %d ctas/sm %d reps %d stagger %d: %.1f us, %.0f GB/s delivered, %.1f B/clk/SM at 1.965 GHz (%s)\n",
         issuers, rows, cols, box_rows, stages, cps, reps, stagger, best * 1e3, bytes / (best * 1e-3) / 1e9,
         bytes / (best * 1e-3) / nsm / 1.965e9, cudaGetErrorString(err));
  return 0;
}
