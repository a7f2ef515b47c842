// Experiment (tools only): throughput of warp-level mma.sync m16n8k16 bf16 (legacy HMMA path) on
// B200, all SMs, register operands -- is it a usable engine for small side contractions?
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__global__ void hmma_loop(float* out, int iters) {
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
  uint32_t b0 = threadIdx.x * 11u, b1 = threadIdx.x * 13u;
  float d[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int j = 0; j < 4; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
  if (s == 1234.5f) out[0] = s;
}
int main() {
  float* o; cudaMalloc(&o, 4);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int warps : {4, 8, 16}) {
    const int iters = 20000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    hmma_loop<<<nsm, 32 * warps>>>(o, 100);
    cudaEventRecord(e0);
    hmma_loop<<<nsm, 32 * warps>>>(o, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * 8 * 16 * 4 * (double)iters * warps * nsm;
    printf("warps/SM %d: %.1f TFLOP/s (mma.sync m16n8k16 bf16->f32)\n", warps, flops / (ms * 1e-3) / 1e12);
  }
  return 0;
}
