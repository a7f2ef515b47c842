// Standalone check of the tcgen05 A-operand-in-TMEM layout (kind::f16, bf16):
// lanes = rows m, element k of row m at column k/2, low half = even k.
// D[128 x 64] = A[128 x 64] (TMEM) . B[64 x 64]^T (smem, K-major SW128)
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstring>
#include "../../paper_2501_08582_b200/csrc/ptx_sm100.cuh"
using namespace lors::ptx;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a_tmem), "l"(bdesc),
               "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void st_x32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
               "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
               "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
               "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
               "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
               : "memory");
}

__global__ void kern(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D) {
  __shared__ __align__(1024) uint8_t sB[64 * 128];
  __shared__ __align__(1024) uint8_t sB16[64 * 128];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  // B [64 n][64 k] K-major SW128: row n, chunk (k/8) ^ (n & 7)
  for (int i = tid; i < 64 * 64; i += 128) {
    const int n = i / 64, k = i % 64;
    *reinterpret_cast<__nv_bfloat16*>(sB + n * 128 + ((((k >> 3) ^ (n & 7))) << 4) + (k & 7) * 2) = B[n * 64 + k];
    *reinterpret_cast<__half*>(sB16 + n * 128 + ((((k >> 3) ^ (n & 7))) << 4) + (k & 7) * 2) =
        __float2half(__bfloat162float(B[n * 64 + k]));
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  // A row m = tid into TMEM columns 128.. (32 columns = 64 bf16)
  uint32_t v[32];
  for (int c = 0; c < 32; ++c) {
    __nv_bfloat162 p = __halves2bfloat162(A[tid * 64 + 2 * c], A[tid * 64 + 2 * c + 1]);
    v[c] = *reinterpret_cast<uint32_t*>(&p);
  }
  st_x32(tmem + ((uint32_t)(warp * 32) << 16) + 128, v);
  for (int c = 0; c < 32; ++c) {
    __half2 p = __floats2half2_rn(__bfloat162float(A[tid * 64 + 2 * c]), __bfloat162float(A[tid * 64 + 2 * c + 1]));
    v[c] = *reinterpret_cast<uint32_t*>(&p);
  }
  st_x32(tmem + ((uint32_t)(warp * 32) << 16) + 192, v);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    constexpr uint32_t idesc = make_idesc_bf16(128, 64, false, false);
    for (int kk = 0; kk < 4; ++kk)
      mma_ts(tmem, tmem + 128 + kk * 8, make_sdesc(smem_u32(sB) + kk * 32, 16, 1024, SW_128), idesc, kk > 0);
    // same product with an f16 accumulator (c_format = 0) into columns 256..
    // f16 A/B (a_format = b_format = 0), f16 D (c_format = 0)
    constexpr uint32_t idesc16 = make_idesc_bf16(128, 64, false, false) & ~((3u << 4) | (7u << 7) | (7u << 10));
    for (int kk = 0; kk < 4; ++kk)
      mma_ts(tmem + 256, tmem + 192 + kk * 8, make_sdesc(smem_u32(sB16) + kk * 32, 16, 1024, SW_128), idesc16,
             kk > 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t d[32];
  tmem_ld_x32(tmem + ((uint32_t)(warp * 32) << 16), d);
  tmem_ld_wait();
  for (int j = 0; j < 32; ++j) D[tid * 64 + j] = __uint_as_float(d[j]);
  tmem_ld_x32(tmem + ((uint32_t)(warp * 32) << 16) + 32, d);
  tmem_ld_wait();
  for (int j = 0; j < 32; ++j) D[tid * 64 + 32 + j] = __uint_as_float(d[j]);
  tmem_ld_x32(tmem + ((uint32_t)(warp * 32) << 16) + 256, d);
  tmem_ld_wait();
  for (int j = 0; j < 32; ++j) D[128 * 64 + tid * 32 + j] = __uint_as_float(d[j]);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
  std::vector<__nv_bfloat16> A(128 * 64), B(64 * 64);
  std::vector<float> Af(128 * 64), Bf(64 * 64), D(128 * 64 + 128 * 32);
  srand(1);
  for (int i = 0; i < 128 * 64; ++i) { A[i] = __float2bfloat16((rand() % 17 - 8) / 8.0f); Af[i] = __bfloat162float(A[i]); }
  for (int i = 0; i < 64 * 64; ++i) { B[i] = __float2bfloat16((rand() % 13 - 6) / 4.0f); Bf[i] = __bfloat162float(B[i]); }
  __nv_bfloat16 *dA, *dB; float* dD;
  cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  kern<<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 64; ++n) {
      double ref = 0;
      for (int k = 0; k < 64; ++k) ref += Af[m * 64 + k] * Bf[n * 64 + k];
      maxerr = std::max(maxerr, std::abs(ref - D[m * 64 + n]));
    }
  printf("TMEM-A layout test: max abs err %.3e (%s)\n", maxerr, maxerr < 1e-3 ? "PASS" : "FAIL");
  // f16 accumulator: packed two per column (low half = even n)?
  double e_packed = 0, e_unpacked = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 64; ++n) {
      double ref = 0;
      for (int k = 0; k < 64; ++k) ref += Af[m * 64 + k] * Bf[n * 64 + k];
      float word = D[128 * 64 + m * 32 + n / 2];
      uint32_t u; memcpy(&u, &word, 4);
      __half_raw hr; hr.x = (unsigned short)((n & 1) ? (u >> 16) : (u & 0xFFFF));
      e_packed = std::max(e_packed, std::abs(ref - (double)__half2float(__half(hr))));
      if (n < 32) {
        float w2 = D[128 * 64 + m * 32 + n]; uint32_t u2; memcpy(&u2, &w2, 4);
        __half_raw h2; h2.x = (unsigned short)(u2 & 0xFFFF);
        e_unpacked = std::max(e_unpacked, std::abs(ref - (double)__half2float(__half(h2))));
      }
    }
  printf("f16 accumulator: packed-2-per-column err %.3e, one-per-column(low16) err %.3e\n", e_packed, e_unpacked);
  return maxerr < 1e-3 ? 0 : 2;
}
