// Experiment (tools only): tcgen05.mma issue-to-completion rate of back-to-back pair MMAs
// (cta_group::2, M = 256, K = 16, bf16 -> fp32) for N = 256 / 128 / 64, operands resident in
// shared memory (zeros), one CTA pair per SM pair -- is a small-N MMA as long as a large one?
//   mma_rate <N> <count> [mix]   mix = 1: alternate N = 256 and N = 128 (the LoRS K1 k-step);
//   mix = 2 / 3: a whole K2 (2:4, r = 64) / K1 (dense, r = 16) k-step's MMAs, recompute included
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include "../../paper_2501_08582_b200/csrc/ptx_sm100.cuh"
using namespace lors::ptx;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mma_kernel(int n, int count, int mix, int sp, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* A = smem;            // [128 rows][64 k] SW128, 16 KB
  uint8_t* B = smem + 16384;    // [128 rows][64 k] SW128, 16 KB
  uint64_t* done = reinterpret_cast<uint64_t*>(smem + 32768);
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 32768 + 16);
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    mbar_init(done, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  if (threadIdx.x / 32 == 1) tmem_alloc_pair<512>(slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (sp) {   // valid 2:4 metadata (kept positions 0 and 1 of every group) in columns 448..455
    const uint32_t lane_base = (uint32_t)((threadIdx.x / 32) * 32) << 16;
    for (int c = 0; c < 8; ++c) tmem_st_x1(tmem + lane_base + 448 + c, 0x44444444u);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (rank == 0 && threadIdx.x / 32 == 0) {
    const uint64_t ad = make_sdesc(smem_u32(A), 16, 1024, SW_128), bd = make_sdesc(smem_u32(B), 16, 1024, SW_128);
    const uint32_t i256 = make_idesc_bf16(256, 256, false, false), i128 = make_idesc_bf16(256, 128, false, false),
                   i64 = make_idesc_bf16(256, 64, false, false);
    const uint32_t idn = n == 256 ? i256 : n == 128 ? i128 : i64;
    unsigned long long t0 = clock64();
    if (elect_one()) {
      for (int c = 0; c < count; ++c) {
        const int kk = c & 3;
        if (mix >= 2) {
          // one K2 k-step (mix 2: 2:4, r = 64) or K1 k-step (mix 3: dense, r = 16): the main MMAs into
          // the two accumulators, then the recompute's N = 64 MMAs into column 384
          const int nrec = mix == 2 ? 4 : 1;
          if (mix == 2) {
            const uint32_t s256 = make_idesc_bf16(256, 256, false, false, true), s128 = make_idesc_bf16(256, 128, false, false, true);
            for (int h = 0; h < 2; ++h) mma_bf16_pair_sp(tmem, ad + h * 2, bd + h * 4, tmem + 448 + h * 4, s256, 1u);
            for (int h = 0; h < 2; ++h) mma_bf16_pair_sp(tmem + 256, ad + h * 2, bd + h * 4, tmem + 448 + h * 4, s128, 1u);
          } else {
            for (int q = 0; q < 4; ++q) mma_bf16_pair(tmem, ad + q * 2, bd + q * 2, i256, 1u);
            for (int q = 0; q < 4; ++q) mma_bf16_pair(tmem + 256, ad + q * 2, bd + q * 2, i128, 1u);
          }
          for (int q = 0; q < nrec; ++q) mma_bf16_pair(tmem + 384, ad + q * 2, bd + q * 2, i64, 1u);
        } else if (sp) {
          const uint32_t isp = make_idesc_bf16(256, n, false, false, true);
          mma_bf16_pair_sp(tmem + (c & 1) * (n == 256 ? 256 : 0), ad + (c & 1) * 2, bd + (c & 1) * 4, tmem + 448 + (c & 1) * 4,
                           isp, 1u);
        } else if (mix) {
          mma_bf16_pair(tmem, ad + kk * 2, bd + kk * 2, i256, 1u);
          mma_bf16_pair(tmem + 256, ad + kk * 2, bd + kk * 2, i128, 1u);
        } else {
          mma_bf16_pair(tmem + (c & 1) * (n == 256 ? 256 : 0), ad + kk * 2, bd + kk * 2, idn, 1u);
        }
      }
      mma_commit_pair(done, 0x3);
    }
    __syncwarp();
    mbar_wait(done, 0);
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x / 2] = t1 - t0;
  } else if (rank == 1 && threadIdx.x == 0) {
    mbar_wait(done, 0);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (threadIdx.x / 32 == 1) tmem_dealloc_pair<512>(tmem);
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 256, count = argc > 2 ? atoi(argv[2]) : 4096, mix = argc > 3 ? atoi(argv[3]) : 0;
  const int sp = argc > 4 ? atoi(argv[4]) : 0;   // 2:4 sparse MMAs (K = 32 logical each)
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* out; cudaMalloc(&out, 8 * nsm);
  const size_t smem = 1024 + 32768 + 64;
  cudaFuncSetAttribute(mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int it = 0; it < 4; ++it) {
    cudaEventRecord(e0);
    mma_kernel<<<nsm / 2 * 2, 128, smem>>>(n, count, mix, sp, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (it > 0 && ms < best) best = ms;
  }
  unsigned long long cyc; cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
  const double macs = (double)count * 256.0 * (mix ? 384.0 : (double)n) * (sp ? 32.0 : 16.0) * (nsm / 2);
  if (mix >= 2) {
    printf("%s k-step pattern count %d: %.1f cycles per k-step (SM 0 pair) (%s)\n", mix == 2 ? "K2 2:4 r=64" : "K1 dense r=16",
           count, (double)cyc / count, cudaGetErrorString(cudaGetLastError()));
    return 0;
  }
  printf("%sN %d%s count %d: %.1f us, %.1f cycles per MMA%s (SM 0 pair), %.0f TFLOP/s (%s)\n", sp ? "sparse " : "", n, mix ? " (256+128 mix)" : "",
         count, best * 1e3, (double)cyc / count / (mix ? 2 : 1), mix ? " instr" : "", 2 * macs / (best * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
