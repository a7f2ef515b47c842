// FFMA (SIMT) kernels of the LoRS layer.
//
// These are the fp32 parity-mode path (TF32 fails the 1e-4 bar,
// FFMA does not) plus the small utility kernels shared by both dtypes
// (mask packing, 2:4 compression, effective weight, dbias).  The bf16 hot
// path lives in lors_tc.cu (tcgen05/TMA/TMEM).
//
// Reference semantics: lors_forward / lors_backward adapters.py:359-406,
// _sqft_grads adapters.py:303-312, merged_weight adapters.py:214-224.

#include "lors_common.cuh"
#include "lors_simt.cuh"
#include <algorithm>

namespace lors {

// ===========================================================================
// S1: GEMM with the effective weight rebuilt in the tile prologue.
//
//   FWD : out[l, m] = sum_k act[l, k] * Weff[m, k]   (act = X_t, m over R, k over C)
//   DX  : out[l, m] = sum_k act[l, k] * Weff[k, m]   (act = dY_t, m over C, k over R)
//
// Weff(row, col) = select(M, W + alpha * sum_j a[row, j] b[j, col], 0).
// The "fixed" adapter factor (a rows for FWD, b columns for DX) is staged in
// shared memory once per block; the "streamed" one per k-tile.  W_eff lives
// only in shared memory.
// Block tile 128 (m) x 128 (l), BK = 8, 256 threads, 8x8 outputs per thread.
// ===========================================================================
namespace {
constexpr int BM = 128, BL = 128, BK = 8, NT = 256;
}

template <typename T, bool DX>
__global__ void __launch_bounds__(NT) simt_lors_gemm_kernel(
    const T* __restrict__ act, const T* __restrict__ w, const uint32_t* __restrict__ bits,
    const T* __restrict__ a, const T* __restrict__ b, const T* __restrict__ bias,
    T* __restrict__ out, int L, int R, int C, int r, float alpha) {
  extern __shared__ float smem[];
  // fixed factor F[j][m] (r x BM), streamed factor S[k][j] (BK x r),
  // act tile sA[k][l] (BK x BL), weight tile sW[k][m] (BK x BM)
  float* sF = smem;
  float* sS = sF + (size_t)r * BM;
  float* sA = sS + (size_t)BK * r;
  float* sW = sA + BK * BL;

  const int tid = threadIdx.x;
  const int m0 = blockIdx.x * BM;
  const int l0 = blockIdx.y * BL;
  const int M = DX ? C : R;   // output feature count
  const int K = DX ? R : C;   // reduction length
  const int64_t words = (C + 31) / 32;

  // stage the fixed factor once: FWD F[j][m] = a[m0+m, j]; DX F[j][m] = b[j, m0+m]
  for (int i = tid; i < r * BM; i += NT) {
    int j, m;
    float v = 0.f;
    if (DX) {
      j = i / BM; m = i % BM;
      if (m0 + m < M) v = to_f(b[(int64_t)j * C + m0 + m]);
    } else {
      m = i / r; j = i % r;
      if (m0 + m < M) v = to_f(a[(int64_t)(m0 + m) * r + j]);
    }
    sF[j * BM + m] = v;
  }

  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  const int tx = tid % 16, ty = tid / 16;
  // weight-tile ownership for the prologue: one m, 4 consecutive k
  const int pm = tid % BM, pk = (tid / BM) * 4;

  for (int k0 = 0; k0 < K; k0 += BK) {
    __syncthreads();
    // streamed factor: FWD S[k][j] = b[j, k0+k]; DX S[k][j] = a[k0+k, j]
    for (int i = tid; i < BK * r; i += NT) {
      int k, j;
      float v = 0.f;
      if (DX) {
        k = i / r; j = i % r;
        if (k0 + k < K) v = to_f(a[(int64_t)(k0 + k) * r + j]);
      } else {
        j = i / BK; k = i % BK;
        if (k0 + k < K) v = to_f(b[(int64_t)j * C + k0 + k]);
      }
      sS[k * r + j] = v;
    }
    // activation tile, transposed into sA[k][l]
    for (int i = tid; i < BK * BL; i += NT) {
      int l = i / BK, k = i % BK;
      float v = 0.f;
      if (l0 + l < L && k0 + k < K) v = to_f(act[(int64_t)(l0 + l) * K + k0 + k]);
      sA[k * BL + l] = v;
    }
    __syncthreads();
    // prologue: rebuild W_eff for this k-tile
    {
      const int gm = m0 + pm;
      float p[4] = {0.f, 0.f, 0.f, 0.f};
      for (int j = 0; j < r; ++j) {
        float f = sF[j * BM + pm];
#pragma unroll
        for (int q = 0; q < 4; ++q) p[q] = fmaf(f, sS[(pk + q) * r + j], p[q]);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int gk = k0 + pk + q;
        float v = 0.f;
        if (gm < M && gk < K) {
          const int64_t row = DX ? gk : gm, col = DX ? gm : gk;
          const T wv = w[row * C + col];
          v = round_to<T>(weff_value<T>(mask_at(wv, bits, words, row, col), to_f(wv), p[q], alpha));
        }
        sW[(pk + q) * BM + pm] = v;
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float av[8], wv[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        av[i] = sA[k * BL + ty * 4 + i];
        av[4 + i] = sA[k * BL + 64 + ty * 4 + i];
        wv[i] = sW[k * BM + tx * 4 + i];
        wv[4 + i] = sW[k * BM + 64 + tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], wv[j], acc[i][j]);
    }
  }
  // epilogue: out[l, m] (+ bias[m] for the forward)
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int l = l0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (l >= L) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int m = m0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (m >= M) continue;
      float v = acc[i][j];
      if (!DX && bias != nullptr) v += to_f(bias[m]);
      out[(int64_t)l * M + m] = from_f<T>(v);
    }
  }
}

// S1v: the fp32 kernel when R and C are multiples of 4 (16-byte rows): 128 x 128 tiles, BK = 16,
// the next k-tile's activation and W fragments fetched into registers (float4) while the current
// one is multiplied, W_eff of the next tile built from those registers, two barriers a k-tile.
// Same arithmetic and summation order as S1 (p over j, then the k-ascending fma chain), so the
// two kernels agree bit for bit.
namespace {
constexpr int VBK = 16;
// two independent fp32 fmas in one instruction (fma.rn.f32x2, sm_100): a 3-register FFMA issues
// at half rate per SMSP, so the packed form doubles the FMA throughput; each lane rounds like fmaf
__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void fma2(uint64_t& d, uint64_t a, uint64_t b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}
__device__ __forceinline__ float2 unpack2(uint64_t v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  return make_float2(lo, hi);
}
}
template <bool DX>
__global__ void __launch_bounds__(NT, 2) simt_lors_gemm_v4_kernel(
    const float* __restrict__ act, const float* __restrict__ w, const uint32_t* __restrict__ bits,
    const float* __restrict__ a, const float* __restrict__ b, const float* __restrict__ bias,
    float* __restrict__ out, int L, int R, int C, int r, float alpha) {
  extern __shared__ float smem[];
  float* sF = smem;                              // [r][BM] fixed factor
  float* sS = sF + (size_t)r * BM;               // [2][VBK][r] streamed factor
  float* sA = sS + (size_t)2 * VBK * r;          // [2][VBK][BL] activation, k-major
  float* sW = sA + 2 * VBK * BL;                 // [2][VBK][BM] W_eff, k-major
  const int tid = threadIdx.x;
  const int m0 = blockIdx.x * BM, l0 = blockIdx.y * BL;
  const int M = DX ? C : R, K = DX ? R : C;
  const int64_t words = (C + 31) / 32;
  for (int i = tid; i < r * BM; i += NT) {
    int j, m;
    float v = 0.f;
    if (DX) {
      j = i / BM; m = i % BM;
      if (m0 + m < M) v = b[(int64_t)j * C + m0 + m];
    } else {
      m = i / r; j = i % r;
      if (m0 + m < M) v = a[(int64_t)(m0 + m) * r + j];
    }
    sF[j * BM + m] = v;
  }
  // fragment ownership: activation row al (8 k from ak); W: FWD row wm (8 k from wk), DX row wk
  // (m = wm .. wm+3 and wm+64 .. wm+67) -- a warp covers 32 rows (FWD / activation) or 2 rows of
  // 128 m (DX W), every shared-memory access 16 bytes apart across the lanes
  const int al = tid % BL, ak = (tid / BL) * 8;
  const int wm = DX ? (tid % 16) * 4 : tid % BM;
  const int wk = DX ? tid / 16 : (tid / BM) * 8;
  float ra[8], rw[8];
  uint32_t rb[2] = {0u, 0u};   // packed-mask words of the W fragment (FWD: one; DX: one per run of 4)
  auto fetch = [&](const int k0, const int buf) {
    const int gl = l0 + al;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int gk = k0 + ak + 4 * h;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gl < L && gk < K) v = __ldg(reinterpret_cast<const float4*>(act + (int64_t)gl * K + gk));
      ra[4 * h] = v.x; ra[4 * h + 1] = v.y; ra[4 * h + 2] = v.z; ra[4 * h + 3] = v.w;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (DX) {
        const int gk = k0 + wk, gm = m0 + wm + 64 * h;
        if (gk < K && gm < M) v = __ldg(reinterpret_cast<const float4*>(w + (int64_t)gk * C + gm));
      } else {
        const int gm = m0 + wm, gk = k0 + wk + 4 * h;
        if (gm < M && gk < K) v = __ldg(reinterpret_cast<const float4*>(w + (int64_t)gm * C + gk));
      }
      rw[4 * h] = v.x; rw[4 * h + 1] = v.y; rw[4 * h + 2] = v.z; rw[4 * h + 3] = v.w;
    }
    if (bits != nullptr) {   // the fragment's mask bits, fetched with it (8 k / 4 m share a word)
#pragma unroll
      for (int h = 0; h < (DX ? 2 : 1); ++h) {
        const int gk = DX ? k0 + wk : k0 + wk, gm = DX ? m0 + wm + 64 * h : m0 + wm;
        const int64_t row = DX ? gk : gm, col = DX ? gm : gk;
        rb[h] = (gk < K && gm < M) ? __ldg(bits + row * words + (col >> 5)) : 0u;
      }
    }
    // streamed factor, laid out for stage(): DX [k][j] (a rows), FWD [j][k] (b rows)
    float* ss = sS + (size_t)buf * VBK * r;
    for (int i = tid; i < VBK * r; i += NT) {
      int k, j;
      float v = 0.f;
      if (DX) {
        k = i / r; j = i % r;
        if (k0 + k < K) v = a[(int64_t)(k0 + k) * r + j];
        ss[k * r + j] = v;
      } else {
        j = i / VBK; k = i % VBK;
        if (k0 + k < K) v = b[(int64_t)j * C + k0 + k];
        ss[j * VBK + k] = v;
      }
    }
  };
  // W_eff of the fetched fragment (needs sS[buf]) and both fragments into shared memory
  auto stage = [&](const int k0, const int buf) {
    const float* ss = sS + (size_t)buf * VBK * r;
    float* sa = sA + (size_t)buf * VBK * BL;
    float* sw = sW + (size_t)buf * VBK * BM;
#pragma unroll
    for (int e = 0; e < 8; ++e) sa[(ak + e) * BL + al] = ra[e];
    // rank-r product of the thread's 8 elements, p[e] = sum_j F[j][m_e] S[k_e][j] in j order (S1's
    // fma chain); FWD: one m, 8 k (S row j as two float4); DX: one k, 8 m (F row j as two float4)
    uint64_t p2[4] = {0ull, 0ull, 0ull, 0ull};   // (p[2q], p[2q + 1]), packed fmas
    for (int j = 0; j < r; ++j) {
      if (DX) {
        const float4 f0 = *reinterpret_cast<const float4*>(sF + j * BM + wm);
        const float4 f1 = *reinterpret_cast<const float4*>(sF + j * BM + wm + 64);
        const float sk = ss[wk * r + j];
        const uint64_t sk2 = pack2(sk, sk);
        fma2(p2[0], pack2(f0.x, f0.y), sk2);
        fma2(p2[1], pack2(f0.z, f0.w), sk2);
        fma2(p2[2], pack2(f1.x, f1.y), sk2);
        fma2(p2[3], pack2(f1.z, f1.w), sk2);
      } else {
        const float fm = sF[j * BM + wm];
        const uint64_t fm2 = pack2(fm, fm);
        const float4 s0 = *reinterpret_cast<const float4*>(ss + j * VBK + wk);
        const float4 s1 = *reinterpret_cast<const float4*>(ss + j * VBK + wk + 4);
        fma2(p2[0], fm2, pack2(s0.x, s0.y));
        fma2(p2[1], fm2, pack2(s0.z, s0.w));
        fma2(p2[2], fm2, pack2(s1.x, s1.y));
        fma2(p2[3], fm2, pack2(s1.z, s1.w));
      }
    }
    float p[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 v = unpack2(p2[q]);
      p[2 * q] = v.x;
      p[2 * q + 1] = v.y;
    }
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int km = DX ? wk : wk + e;           // k of element e (tile-local)
      const int mm = DX ? wm + (e & 3) + 64 * (e >> 2) : wm;   // m of element e (tile-local)
      const int gk = k0 + km, gm = m0 + mm;
      v[e] = 0.f;
      if (gm < M && gk < K) {
        const int col = DX ? gm : gk;
        const bool keep = bits != nullptr ? ((rb[DX ? (e >> 2) : 0] >> (col & 31)) & 1u) != 0u : rw[e] != 0.0f;
        v[e] = weff_value<float>(keep, rw[e], p[e], alpha);
      }
      if (!DX) sw[km * BM + mm] = v[e];          // a warp: 32 consecutive m of one k row
    }
    if (DX) {                                    // the thread's two runs of 4 m in row wk
      *reinterpret_cast<float4*>(sw + wk * BM + wm) = make_float4(v[0], v[1], v[2], v[3]);
      *reinterpret_cast<float4*>(sw + wk * BM + wm + 64) = make_float4(v[4], v[5], v[6], v[7]);
    }
  };
  uint64_t acc2[4][8];   // (acc[2 ip][j], acc[2 ip + 1][j])
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc2[i][j] = 0ull;
  const int tx = tid % 16, ty = tid / 16;
  fetch(0, 0);
  __syncthreads();          // sF, sS[0]
  stage(0, 0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < K; k0 += VBK, buf ^= 1) {
    const bool more = k0 + VBK < K;
    if (more) fetch(k0 + VBK, buf ^ 1);
    const float* sa = sA + (size_t)buf * VBK * BL;
    const float* sw = sW + (size_t)buf * VBK * BM;
#pragma unroll
    for (int k = 0; k < VBK; ++k) {
      const float4 a0 = *reinterpret_cast<const float4*>(sa + k * BL + ty * 4);
      const float4 a1 = *reinterpret_cast<const float4*>(sa + k * BL + 64 + ty * 4);
      const float4 w0 = *reinterpret_cast<const float4*>(sw + k * BM + tx * 4);
      const float4 w1 = *reinterpret_cast<const float4*>(sw + k * BM + 64 + tx * 4);
      const uint64_t ap[4] = {pack2(a0.x, a0.y), pack2(a0.z, a0.w), pack2(a1.x, a1.y), pack2(a1.z, a1.w)};
      const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint64_t wj = pack2(wv[j], wv[j]);
#pragma unroll
        for (int ip = 0; ip < 4; ++ip) fma2(acc2[ip][j], ap[ip], wj);
      }
    }
    if (more) {
      __syncthreads();      // sS[buf ^ 1] written; everyone done with the other buffers' last use
      stage(k0 + VBK, buf ^ 1);
      __syncthreads();
    }
  }
  float acc[8][8];
#pragma unroll
  for (int ip = 0; ip < 4; ++ip)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float2 v = unpack2(acc2[ip][j]);
      acc[2 * ip][j] = v.x;
      acc[2 * ip + 1][j] = v.y;
    }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int l = l0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (l >= L) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int m = m0 + h * 64 + tx * 4;
      if (m >= M) continue;                     // M % 4 == 0: all four or none
      float4 v = make_float4(acc[i][4 * h], acc[i][4 * h + 1], acc[i][4 * h + 2], acc[i][4 * h + 3]);
      if (!DX && bias != nullptr) {
        v.x += bias[m]; v.y += bias[m + 1]; v.z += bias[m + 2]; v.w += bias[m + 3];
      }
      *reinterpret_cast<float4*>(out + (int64_t)l * M + m) = v;
    }
  }
}

template <typename T>
int simt_lors_gemm(bool dx, const T* act, const T* w, const uint32_t* bits, const T* a, const T* b,
                   const T* bias, T* out, int L, int R, int C, int r, float alpha, cudaStream_t s) {
  const int M = dx ? C : R;
  dim3 grid((unsigned)ceil_div(M, BM), (unsigned)ceil_div(L, BL));
  if (sizeof(T) == 4 && R % 4 == 0 && C % 4 == 0) {   // 16-byte rows: the vectorised, pipelined kernel
    const size_t sm = sizeof(float) * ((size_t)r * BM + (size_t)2 * VBK * r + 2 * VBK * BL + 2 * VBK * BM);
    auto kv = dx ? simt_lors_gemm_v4_kernel<true> : simt_lors_gemm_v4_kernel<false>;
    LORS_CUDA_TRY(cudaFuncSetAttribute(kv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm),
                  "simt_lors_gemm smem attribute");
    kv<<<grid, NT, sm, s>>>((const float*)act, (const float*)w, bits, (const float*)a, (const float*)b,
                            (const float*)bias, (float*)out, L, R, C, r, alpha);
    LORS_CHECK_LAUNCH("simt_lors_gemm");
    return LORS_OK;
  }
  size_t smem = sizeof(float) * ((size_t)r * BM + (size_t)BK * r + BK * BL + BK * BM);
  auto kern = dx ? simt_lors_gemm_kernel<T, true> : simt_lors_gemm_kernel<T, false>;
  LORS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                "simt_lors_gemm smem attribute");
  kern<<<grid, NT, smem, s>>>(act, w, bits, a, b, bias, out, L, R, C, r, alpha);
  LORS_CHECK_LAUNCH("simt_lors_gemm");
  return LORS_OK;
}

// ===========================================================================
// S2: strided "skinny" GEMM for the rank-r products (P, Q, dA, dB):
//   out[m*som + n*son] (= or +=) alpha * sum_k A[m*sam + k*sak] * B[n*sbn + k*sbk]
// 64x64 tiles, BK = 16, 256 threads, 4x4 per thread; gridDim.z splits K and
// accumulates with atomicAdd into a zeroed fp32 output.
// ===========================================================================
template <typename TA, typename TB, typename TO, int TM, int TN>
__global__ void __launch_bounds__(256) simt_strided_gemm_kernel(
    const TA* __restrict__ A, int64_t sam, int64_t sak, const TB* __restrict__ B, int64_t sbn,
    int64_t sbk, TO* __restrict__ out, int64_t som, int64_t son, int M, int N, int K,
    int k_per_split, float alpha, int atomic_out) {
  // TM x TN tile (64 x 64, or 256 x 16 / 16 x 256 when one side is the rank), 4 x 4 per thread
  __shared__ float sA[16][TM + 4];
  __shared__ float sB[16][TN + 4];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.x * TM, n0 = blockIdx.y * TN;
  const int kbeg = blockIdx.z * k_per_split;
  const int kend = min(K, kbeg + k_per_split);
  constexpr int TXN = TN / 4;
  const int tx = tid % TXN, ty = tid / TXN;
  uint64_t acc2[2][4] = {};   // (acc[2 ip][j], acc[2 ip + 1][j]): packed fmas, each lane rounds like fmaf
  for (int k0 = kbeg; k0 < kend; k0 += 16) {
    for (int i = tid; i < 16 * TM; i += 256) {
      int m, k;
      if (sak == 1) { k = i % 16; m = i / 16; } else { m = i % TM; k = i / TM; }
      float v = 0.f;
      if (m0 + m < M && k0 + k < kend) v = to_f(A[(int64_t)(m0 + m) * sam + (int64_t)(k0 + k) * sak]);
      sA[k][m] = v;
    }
    for (int i = tid; i < 16 * TN; i += 256) {
      int n, k;
      if (sbk == 1) { k = i % 16; n = i / 16; } else { n = i % TN; k = i / TN; }
      float v = 0.f;
      if (n0 + n < N && k0 + k < kend) v = to_f(B[(int64_t)(n0 + n) * sbn + (int64_t)(k0 + k) * sbk]);
      sB[k][n] = v;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { av[i] = sA[k][ty * 4 + i]; bv[i] = sB[k][tx * 4 + i]; }
      const uint64_t ap[2] = {pack2(av[0], av[1]), pack2(av[2], av[3])};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t bj = pack2(bv[j], bv[j]);
        fma2(acc2[0][j], ap[0], bj);
        fma2(acc2[1][j], ap[1], bj);
      }
    }
    __syncthreads();
  }
  float acc[4][4];
#pragma unroll
  for (int ip = 0; ip < 2; ++ip)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 v = unpack2(acc2[ip][j]);
      acc[2 * ip][j] = v.x;
      acc[2 * ip + 1][j] = v.y;
    }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      TO* dst = out + (int64_t)m * som + (int64_t)n * son;
      const float v = alpha * acc[i][j];
      if (atomic_out) atomicAdd(reinterpret_cast<float*>(dst), v);
      else *dst = from_f<TO>(v);
    }
  }
}

template <typename TA, typename TB, typename TO>
int simt_strided_gemm(const TA* A, int64_t sam, int64_t sak, const TB* B, int64_t sbn, int64_t sbk,
                      TO* out, int64_t som, int64_t son, int M, int N, int K, float alpha,
                      bool allow_split, cudaStream_t s) {
  // tile shape: the rank side (N or M <= 16) gets a 16-wide tile, no 64-wide padding
  const int shape = N <= 16 ? 1 : M <= 16 ? 2 : 0;   // 0: 64 x 64, 1: 256 x 16, 2: 16 x 256
  const int TMh = shape == 1 ? 256 : shape == 2 ? 16 : 64, TNh = shape == 1 ? 16 : shape == 2 ? 256 : 64;
  const int tiles = (int)(ceil_div(M, TMh) * ceil_div(N, TNh));
  int split = 1;
  if (allow_split && sizeof(TO) == sizeof(float)) {
    split = (int)ceil_div(296, tiles);
    split = max(1, min(split, (int)ceil_div(K, 256)));
  }
  int kps = (int)(ceil_div(ceil_div(K, split), 16) * 16);
  split = (int)ceil_div(K, kps);
  if (split > 1) {
    // atomic accumulation requires a zeroed fp32, densely addressed output
    LORS_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(float) * (size_t)M * N, s), "zero split-K output");
  }
  dim3 grid((unsigned)ceil_div(M, TMh), (unsigned)ceil_div(N, TNh), (unsigned)split);
  if (shape == 1)
    simt_strided_gemm_kernel<TA, TB, TO, 256, 16><<<grid, 256, 0, s>>>(A, sam, sak, B, sbn, sbk, out, som, son, M,
                                                                       N, K, kps, alpha, split > 1 ? 1 : 0);
  else if (shape == 2)
    simt_strided_gemm_kernel<TA, TB, TO, 16, 256><<<grid, 256, 0, s>>>(A, sam, sak, B, sbn, sbk, out, som, son, M,
                                                                       N, K, kps, alpha, split > 1 ? 1 : 0);
  else
    simt_strided_gemm_kernel<TA, TB, TO, 64, 64><<<grid, 256, 0, s>>>(A, sam, sak, B, sbn, sbk, out, som, son, M, N,
                                                                      K, kps, alpha, split > 1 ? 1 : 0);
  LORS_CHECK_LAUNCH("simt_strided_gemm");
  return LORS_OK;
}

// ===========================================================================
// S4: the fp32 rank-r products at the HBM rate (P = X b^T, Q = dY a, dA = dY^T P, dB = Q^T X).
// Each reads one L x N activation matrix once against an r-wide factor; S2's tiles stage the big
// operand through shared memory a 16-k slice at a time, S4 streams it with float4 loads straight into
// packed fmas and keeps the factor on chip.
//   project:    out[l, j]  = sum_n Y[l, n] F(j, n)            F(j, n) = Fm[j sfj + n sfn]
//   accumulate: out[n, j] += alpha sum_l Y[l, n] S[l, j]     written at out[n son + j soj]
// Requires N % 4 == 0, ldy % 4 == 0 and a 16-byte aligned Y (the caller falls back to S2 otherwise).
// project splits N over gridDim.y with fp32 atomics into a zeroed out, or (deterministic) runs each
// row's whole reduction in one warp; accumulate always splits L (atomics: fast mode only).
// ===========================================================================
namespace {
constexpr int S4_THREADS = 256;
template <int RP>
struct s4 {
  static constexpr int PR = 64 / RP;            // project: rows a warp (PR x RP accumulators)
  static constexpr int ROWS = 8 * PR;           // project: rows a CTA
  static constexpr int NCH = RP <= 16 ? 1024 : 512;   // project: factor rows staged a chunk (80 / 72 KB)
  static constexpr size_t SMEM = (size_t)NCH * (RP + 4) * sizeof(float);
};

// reduce-scatter of NV values over the warp: afterwards lane l holds NV / 32 fully reduced values,
// value t of lane l being index ((l >> 4 & 1) NV/2 + (l >> 3 & 1) NV/4 + ... ) + t
template <int NV>
__device__ __forceinline__ void warp_reduce_scatter(float (&v)[NV], int lane) {
#pragma unroll
  for (int off = 16, n = NV; off >= 1; off >>= 1, n >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < n / 2; ++i) {
      const float keep = up ? v[n / 2 + i] : v[i];
      const float give = up ? v[i] : v[n / 2 + i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, give, off);
    }
  }
}
__device__ __forceinline__ int scatter_index(int lane, int nv) {
  int idx = 0;
#pragma unroll
  for (int off = 16, h = nv / 2; off >= 1; off >>= 1, h >>= 1)
    if (lane & off) idx += h;
  return idx;
}
__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
}  // namespace

template <int RP>
__global__ void __launch_bounds__(S4_THREADS, 2) s4_project_kernel(const float* __restrict__ Y, int64_t ldy,
                                                                   const float* __restrict__ Fm, int64_t sfj,
                                                                   int64_t sfn, float* __restrict__ out, int L,
                                                                   int N, int r, int n_per_cta, int atomic_out) {
  // factor slice as sF[n][RP + 4]: lane l reads row n = l + 32 t, the 4-float pad makes the 16-byte
  // reads of 8 consecutive rows hit 8 distinct bank groups
  using S = s4<RP>;
  constexpr int FS = RP + 4;
  extern __shared__ __align__(16) float sF[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int row0 = blockIdx.x * S::ROWS + warp * S::PR;
  const int nbeg = blockIdx.y * n_per_cta, nend = min(N, nbeg + n_per_cta);
  uint64_t acc[S::PR][RP / 2] = {};   // (rank 2 jp, 2 jp + 1) of row p
  for (int c0 = nbeg; c0 < nend; c0 += S::NCH) {
    const int cn = min(S::NCH, nend - c0);
    __syncthreads();
    for (int i = threadIdx.x; i < RP * S::NCH; i += S4_THREADS) {
      int j, c;
      if (sfn == 1) { j = i / S::NCH; c = i % S::NCH; } else { c = i / RP; j = i % RP; }
      sF[c * FS + j] = (j < r && c < cn) ? Fm[(int64_t)j * sfj + (int64_t)(c0 + c) * sfn] : 0.f;
    }
    __syncthreads();
    const float* yr[S::PR];
#pragma unroll
    for (int p = 0; p < S::PR; ++p) yr[p] = Y + (int64_t)min(row0 + p, L - 1) * ldy + c0;
#pragma unroll 4
    for (int c = lane; c < cn; c += 32) {
      float y[S::PR];
#pragma unroll
      for (int p = 0; p < S::PR; ++p) y[p] = __ldg(yr[p] + c);
#pragma unroll
      for (int j4 = 0; j4 < RP / 4; ++j4) {
        const float4 f = *reinterpret_cast<const float4*>(&sF[c * FS + 4 * j4]);
        const uint64_t f01 = pack2(f.x, f.y), f23 = pack2(f.z, f.w);
#pragma unroll
        for (int p = 0; p < S::PR; ++p) {
          const uint64_t y2 = pack2(y[p], y[p]);
          fma2(acc[p][2 * j4], y2, f01);
          fma2(acc[p][2 * j4 + 1], y2, f23);
        }
      }
    }
  }
  float v[S::PR * RP];
#pragma unroll
  for (int p = 0; p < S::PR; ++p)
#pragma unroll
    for (int jp = 0; jp < RP / 2; ++jp) {
      const float2 h = unpack2(acc[p][jp]);
      v[p * RP + 2 * jp] = h.x;
      v[p * RP + 2 * jp + 1] = h.y;
    }
  warp_reduce_scatter<S::PR * RP>(v, lane);
  const int idx = scatter_index(lane, S::PR * RP);
#pragma unroll
  for (int t = 0; t < S::PR * RP / 32; ++t) {
    const int p = (idx + t) / RP, j = (idx + t) % RP;
    if (j < r && row0 + p < L) {
      float* dst = out + (int64_t)(row0 + p) * r + j;
      if (atomic_out) atomicAdd(dst, v[t]);
      else *dst = v[t];
    }
  }
}

// mode 0: scalar atomics; 1: v4 over j (soj == 1, r % 4 == 0); 2: v4 over n (son == 1, soj % 4 == 0)
template <int RP>
__global__ void __launch_bounds__(S4_THREADS) s4_accumulate_kernel(const float* __restrict__ Y, int64_t ldy,
                                                                   const float* __restrict__ Sm,
                                                                   float* __restrict__ out, int64_t son,
                                                                   int64_t soj, int L, int N, int r, int l_per_cta,
                                                                   float alpha, int mode) {
  constexpr int LMAX = 128;
  __shared__ __align__(16) float sS[LMAX][RP];
  const int n = (blockIdx.x * S4_THREADS + threadIdx.x) * 4;
  const int l0 = blockIdx.y * l_per_cta, ln = min(l_per_cta, L - l0);
  for (int i = threadIdx.x; i < ln * RP; i += S4_THREADS) {
    const int l = i / RP, j = i % RP;
    sS[l][j] = j < r ? Sm[(int64_t)(l0 + l) * r + j] : 0.f;
  }
  __syncthreads();
  if (n >= N) return;
  uint64_t acc[4][RP / 2] = {};   // (n + q; ranks 2 jp, 2 jp + 1)
  const float* yp = Y + (int64_t)l0 * ldy + n;
#pragma unroll 4
  for (int l = 0; l < ln; ++l) {
    const float4 y = __ldg(reinterpret_cast<const float4*>(yp + (int64_t)l * ldy));
    const float yq[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
    for (int j4 = 0; j4 < RP / 4; ++j4) {
      const float4 sv = *reinterpret_cast<const float4*>(&sS[l][4 * j4]);   // broadcast
      const uint64_t s01 = pack2(sv.x, sv.y), s23 = pack2(sv.z, sv.w);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint64_t y2 = pack2(yq[q], yq[q]);
        fma2(acc[q][2 * j4], y2, s01);
        fma2(acc[q][2 * j4 + 1], y2, s23);
      }
    }
  }
  float o[4][RP];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int jp = 0; jp < RP / 2; ++jp) {
      const float2 h = unpack2(acc[q][jp]);
      o[q][2 * jp] = alpha * h.x;
      o[q][2 * jp + 1] = alpha * h.y;
    }
  if (mode == 1) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int j4 = 0; j4 < RP / 4; ++j4)
        if (4 * j4 < r)
          red_add_v4(out + (int64_t)(n + q) * son + 4 * j4, o[q][4 * j4], o[q][4 * j4 + 1], o[q][4 * j4 + 2],
                     o[q][4 * j4 + 3]);
  } else if (mode == 2) {
#pragma unroll
    for (int j = 0; j < RP; ++j)
      if (j < r) red_add_v4(out + (int64_t)j * soj + n, o[0][j], o[1][j], o[2][j], o[3][j]);
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int j = 0; j < RP; ++j)
        if (j < r) atomicAdd(out + (int64_t)(n + q) * son + (int64_t)j * soj, o[q][j]);
  }
}

static bool s4_ok(const float* Y, int64_t ldy, int N, int r) {
  return r >= 1 && r <= 32 && N % 4 == 0 && ldy % 4 == 0 && (reinterpret_cast<uintptr_t>(Y) & 15) == 0;
}

int s4_rank_project(const float* Y, int64_t ldy, const float* Fm, int64_t sfj, int64_t sfn, float* out, int L,
                    int N, int r, bool deterministic, cudaStream_t s) {
  if (!s4_ok(Y, ldy, N, r)) return LORS_ERR_SHAPE;
  const int rows = r <= 16 ? s4<16>::ROWS : s4<32>::ROWS, nch = r <= 16 ? s4<16>::NCH : s4<32>::NCH;
  const int rtiles = (int)ceil_div(L, rows);
  // fast mode: one staged factor chunk a CTA (N split over gridDim.y, atomics); deterministic: whole rows
  int splits = deterministic ? 1 : (int)ceil_div(N, nch);
  const int npc = (int)(ceil_div(ceil_div(N, splits), 4) * 4);
  splits = (int)ceil_div(N, npc);
  if (splits > 1) LORS_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(float) * (size_t)L * r, s), "zero S4 output");
  dim3 grid((unsigned)rtiles, (unsigned)splits);
  if (r <= 16) {
    LORS_CUDA_TRY(cudaFuncSetAttribute(s4_project_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)s4<16>::SMEM), "S4 smem attribute");
    s4_project_kernel<16><<<grid, S4_THREADS, s4<16>::SMEM, s>>>(Y, ldy, Fm, sfj, sfn, out, L, N, r, npc,
                                                                  splits > 1);
  } else {
    LORS_CUDA_TRY(cudaFuncSetAttribute(s4_project_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)s4<32>::SMEM), "S4 smem attribute");
    s4_project_kernel<32><<<grid, S4_THREADS, s4<32>::SMEM, s>>>(Y, ldy, Fm, sfj, sfn, out, L, N, r, npc,
                                                                  splits > 1);
  }
  LORS_CHECK_LAUNCH("s4_project");
  return LORS_OK;
}

int s4_rank_accumulate(const float* Y, int64_t ldy, const float* Sm, float* out, int64_t son, int64_t soj, int L,
                       int N, int r, float alpha, cudaStream_t s) {
  if (!s4_ok(Y, ldy, N, r)) return LORS_ERR_SHAPE;
  const int ntiles = (int)ceil_div(N, 4 * S4_THREADS);
  int lpc = (int)std::min<int64_t>(128, std::max<int64_t>(8, ceil_div(ceil_div((int64_t)L * ntiles, 296), 4) * 4));
  const int ltiles = (int)ceil_div(L, lpc);
  const bool aligned = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  const int mode = !aligned ? 0 : (soj == 1 && r % 4 == 0 && son % 4 == 0) ? 1 : (son == 1 && soj % 4 == 0) ? 2 : 0;
  // out is a dense N x r (or r x N) block here: zero it, then every L slice adds its share
  LORS_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(float) * (size_t)N * r, s), "zero S4 output");
  dim3 grid((unsigned)ntiles, (unsigned)ltiles);
  if (r <= 16)
    s4_accumulate_kernel<16><<<grid, S4_THREADS, 0, s>>>(Y, ldy, Sm, out, son, soj, L, N, r, lpc, alpha, mode);
  else
    s4_accumulate_kernel<32><<<grid, S4_THREADS, 0, s>>>(Y, ldy, Sm, out, son, soj, L, N, r, lpc, alpha, mode);
  LORS_CHECK_LAUNCH("s4_accumulate");
  return LORS_OK;
}

// ===========================================================================
// S3: masked-gradient fused kernel (north_star 3, SIMT form for fp32 mode).
// Each block forms one G tile = (dY^T X)[64 rows of R x 64 cols of C] over
// all L tokens in registers, masks it, parks it in shared memory and
// contracts it immediately:  dA[n, :] += alpha G b^T,  dB[:, c] += alpha a^T G.
// G never reaches HBM.  Oracle: _sqft_grads adapters.py:303-312.
// ===========================================================================
template <typename T>
__global__ void __launch_bounds__(256) simt_masked_grad_kernel(
    const T* __restrict__ dy, const T* __restrict__ x, const T* __restrict__ w,
    const uint32_t* __restrict__ bits, const T* __restrict__ a, const T* __restrict__ b,
    float* __restrict__ da, float* __restrict__ db, int L, int R, int C, int r, float alpha) {
  __shared__ float sA[16][64 + 4];
  __shared__ float sB[16][64 + 4];
  __shared__ float sG[64][64 + 1];
  const int tid = threadIdx.x;
  const int n0 = blockIdx.x * 64, c0 = blockIdx.y * 64;
  const int tx = tid % 16, ty = tid / 16;
  const int64_t words = (C + 31) / 32;
  float acc[4][4] = {};
  for (int l0 = 0; l0 < L; l0 += 16) {
    for (int i = tid; i < 16 * 64; i += 256) {
      const int mm = i % 64, k = i / 64;
      float v = 0.f;
      if (n0 + mm < R && l0 + k < L) v = to_f(dy[(int64_t)(l0 + k) * R + n0 + mm]);
      sA[k][mm] = v;
      v = 0.f;
      if (c0 + mm < C && l0 + k < L) v = to_f(x[(int64_t)(l0 + k) * C + c0 + mm]);
      sB[k][mm] = v;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { av[i] = sA[k][ty * 4 + i]; bv[i] = sB[k][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  // mask in registers, park in shared memory
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + ty * 4 + i, c = c0 + tx * 4 + j;
      float g = 0.f;
      if (n < R && c < C) {
        const T wv = w[(int64_t)n * C + c];
        g = mask_at(wv, bits, words, n, c) ? acc[i][j] : 0.f;
      }
      sG[ty * 4 + i][tx * 4 + j] = g;
    }
  __syncthreads();
  // dA[n, j] += alpha * sum_c G[n, c] b[j, c]
  for (int i = tid; i < 64 * r; i += 256) {
    const int nn = i / r, j = i % r;
    if (n0 + nn >= R) continue;
    float s = 0.f;
    for (int cc = 0; cc < 64 && c0 + cc < C; ++cc) s = fmaf(sG[nn][cc], to_f(b[(int64_t)j * C + c0 + cc]), s);
    atomicAdd(da + (int64_t)(n0 + nn) * r + j, alpha * s);
  }
  // dB[j, c] += alpha * sum_n a[n, j] G[n, c]
  for (int i = tid; i < 64 * r; i += 256) {
    const int cc = i % 64, j = i / 64;
    if (c0 + cc >= C) continue;
    float s = 0.f;
    for (int nn = 0; nn < 64 && n0 + nn < R; ++nn) s = fmaf(to_f(a[(int64_t)(n0 + nn) * r + j]), sG[nn][cc], s);
    atomicAdd(db + (int64_t)j * C + c0 + cc, alpha * s);
  }
}

template <typename T>
int simt_masked_grad(const T* dy, const T* x, const T* w, const uint32_t* bits, const T* a,
                     const T* b, float* da, float* db, int L, int R, int C, int r, float alpha,
                     cudaStream_t s) {
  LORS_CUDA_TRY(cudaMemsetAsync(da, 0, sizeof(float) * (size_t)R * r, s), "zero dA");
  LORS_CUDA_TRY(cudaMemsetAsync(db, 0, sizeof(float) * (size_t)r * C, s), "zero dB");
  dim3 grid((unsigned)ceil_div(R, 64), (unsigned)ceil_div(C, 64));
  simt_masked_grad_kernel<T><<<grid, 256, 0, s>>>(dy, x, w, bits, a, b, da, db, L, R, C, r, alpha);
  LORS_CHECK_LAUNCH("simt_masked_grad");
  return LORS_OK;
}

// ===========================================================================
// utility kernels (both dtypes)
// ===========================================================================

// dbias[n] = sum_l dY_t[l, n]   (reduce_sum_rows, adapters.py:402)
template <typename T>
__global__ void colsum_kernel(const T* __restrict__ dy, float* __restrict__ out, int L, int R) {
  const int n = blockIdx.x * 32 + threadIdx.x;
  const int part = threadIdx.y;  // 8 partial sums over L
  __shared__ float red[8][33];
  float s = 0.f;
  if (n < R)
    for (int l = part; l < L; l += 8) s += to_f(dy[(int64_t)l * R + n]);
  red[part][threadIdx.x] = s;
  __syncthreads();
  if (part == 0 && n < R) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += red[i][threadIdx.x];
    out[n] = t;
  }
}

template <typename T>
int colsum(const T* dy, float* out, int L, int R, cudaStream_t s) {
  colsum_kernel<T><<<(unsigned)ceil_div(R, 32), dim3(32, 8), 0, s>>>(dy, out, L, R);
  LORS_CHECK_LAUNCH("colsum");
  return LORS_OK;
}

// out[n, c] = select(M, W + alpha * (a b)[n, c], +0) -- merged_weight / merge
template <typename T>
__global__ void effective_weight_kernel(const T* __restrict__ w, const uint32_t* __restrict__ bits,
                                        const T* __restrict__ a, const T* __restrict__ b,
                                        T* __restrict__ out, int R, int C, int r, float alpha) {
  extern __shared__ float sa[];  // 4 rows of a
  const int n0 = blockIdx.y * 4;
  for (int i = threadIdx.x; i < 4 * r; i += blockDim.x) {
    const int nn = i / r;
    sa[i] = (n0 + nn < R) ? to_f(a[(int64_t)(n0 + nn) * r + i % r]) : 0.f;
  }
  __syncthreads();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const int64_t words = (C + 31) / 32;
  float p[4] = {0.f, 0.f, 0.f, 0.f};
  for (int j = 0; j < r; ++j) {
    const float bv = to_f(b[(int64_t)j * C + c]);
#pragma unroll
    for (int q = 0; q < 4; ++q) p[q] = fmaf(sa[q * r + j], bv, p[q]);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int n = n0 + q;
    if (n >= R) break;
    const T wv = w[(int64_t)n * C + c];
    out[(int64_t)n * C + c] = from_f<T>(weff_value<T>(mask_at(wv, bits, words, n, c), to_f(wv), p[q], alpha));
  }
}

template <typename T>
int effective_weight(const T* w, const uint32_t* bits, const T* a, const T* b, T* out, int R, int C,
                     int r, float alpha, cudaStream_t s) {
  dim3 grid((unsigned)ceil_div(C, 256), (unsigned)ceil_div(R, 4));
  effective_weight_kernel<T><<<grid, 256, sizeof(float) * 4 * r, s>>>(w, bits, a, b, out, R, C, r, alpha);
  LORS_CHECK_LAUNCH("effective_weight");
  return LORS_OK;
}

// bits[n, k] : bit j = (W[n, 32k + j] != 0), one warp ballot per word
template <typename T>
__global__ void pack_mask_kernel(const T* __restrict__ w, uint32_t* __restrict__ bits, int R, int C) {
  const int64_t words = (C + 31) / 32;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;  // global word
  if (gw >= (int64_t)R * words) return;
  const int64_t n = gw / words, k = gw % words;
  const int lane = threadIdx.x & 31;
  const int64_t c = k * 32 + lane;
  const bool nz = c < C && to_f(w[n * C + c]) != 0.0f;
  const uint32_t word = __ballot_sync(0xffffffffu, nz);
  if (lane == 0) bits[gw] = word;
}

template <typename T>
int pack_mask(const T* w, uint32_t* bits, int R, int C, cudaStream_t s) {
  const int64_t words = (int64_t)R * ceil_div(C, 32);
  pack_mask_kernel<T><<<(unsigned)ceil_div(words, 8), 256, 0, s>>>(w, bits, R, C);
  LORS_CHECK_LAUNCH("pack_mask");
  return LORS_OK;
}

// 2:4 compression: per group of 4 along C keep the (<= 2) nonzero positions.
// Groups with fewer than 2 nonzeros are padded with zero-valued positions
// (lowest unused index first); groups with more set *invalid.
template <typename T>
__global__ void compress24_kernel(const T* __restrict__ w, T* __restrict__ vals, uint8_t* __restrict__ meta,
                                  int32_t* __restrict__ invalid, int R, int C) {
  const int64_t pair = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // two groups per thread
  const int64_t pairs_per_row = C / 8;
  if (pair >= (int64_t)R * pairs_per_row) return;
  const int64_t n = pair / pairs_per_row, gp = pair % pairs_per_row;
  uint8_t byte = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t c0 = gp * 8 + h * 4;
    int idx[2] = {-1, -1};
    int cnt = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (to_f(w[n * C + c0 + q]) != 0.0f) {
        if (cnt < 2) idx[cnt] = q;
        ++cnt;
      }
    }
    if (cnt > 2 && invalid != nullptr) *invalid = 1;
    // pad with unused positions
    for (int q = 0; q < 4 && (idx[0] < 0 || idx[1] < 0); ++q) {
      if (q == idx[0] || q == idx[1]) continue;
      if (idx[0] < 0) idx[0] = q;
      else if (idx[1] < 0) idx[1] = q;
    }
    if (idx[0] > idx[1]) { int t = idx[0]; idx[0] = idx[1]; idx[1] = t; }
    vals[n * (C / 2) + (c0 / 2)] = w[n * C + c0 + idx[0]];
    vals[n * (C / 2) + (c0 / 2) + 1] = w[n * C + c0 + idx[1]];
    byte |= (uint8_t)((idx[0] | (idx[1] << 2)) << (4 * h));
  }
  meta[n * (C / 8) + gp] = byte;
}

template <typename T>
int compress24(const T* w, T* vals, uint8_t* meta, int32_t* invalid, int R, int C, cudaStream_t s) {
  const int64_t pairs = (int64_t)R * (C / 8);
  compress24_kernel<T><<<(unsigned)ceil_div(pairs, 256), 256, 0, s>>>(w, vals, meta, invalid, R, C);
  LORS_CHECK_LAUNCH("compress24");
  return LORS_OK;
}

// dW = dY_t^T X_t (optionally masked), the probe gradient of gradient-SVD init
template <typename T>
__global__ void __launch_bounds__(256) grad_outer_kernel(const T* __restrict__ dy, const T* __restrict__ x,
                                                         const T* __restrict__ w, float* __restrict__ dw,
                                                         int L, int R, int C, int masked) {
  __shared__ float sA[16][64 + 4];
  __shared__ float sB[16][64 + 4];
  const int tid = threadIdx.x;
  const int n0 = blockIdx.x * 64, c0 = blockIdx.y * 64;
  const int tx = tid % 16, ty = tid / 16;
  float acc[4][4] = {};
  for (int l0 = 0; l0 < L; l0 += 16) {
    for (int i = tid; i < 16 * 64; i += 256) {
      const int mm = i % 64, k = i / 64;
      sA[k][mm] = (n0 + mm < R && l0 + k < L) ? to_f(dy[(int64_t)(l0 + k) * R + n0 + mm]) : 0.f;
      sB[k][mm] = (c0 + mm < C && l0 + k < L) ? to_f(x[(int64_t)(l0 + k) * C + c0 + mm]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(sA[k][ty * 4 + i], sB[k][tx * 4 + j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + ty * 4 + i, c = c0 + tx * 4 + j;
      if (n >= R || c >= C) continue;
      float g = acc[i][j];
      if (masked && to_f(w[(int64_t)n * C + c]) == 0.0f) g = 0.f;
      dw[(int64_t)n * C + c] = g;
    }
}

template <typename T>
int grad_outer(const T* dy, const T* x, const T* w, float* dw, int L, int R, int C, int masked, cudaStream_t s) {
  dim3 grid((unsigned)ceil_div(R, 64), (unsigned)ceil_div(C, 64));
  grad_outer_kernel<T><<<grid, 256, 0, s>>>(dy, x, w, dw, L, R, C, masked);
  LORS_CHECK_LAUNCH("grad_outer");
  return LORS_OK;
}

// negate in place (negative-control fault injection)
__global__ void negate_kernel(float* p, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = -p[i];
}
int negate_f32(float* p, int64_t n, cudaStream_t s) {
  negate_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(p, n);
  LORS_CHECK_LAUNCH("negate");
  return LORS_OK;
}

// ---------------------------------------------------------------------------
// explicit instantiations
// ---------------------------------------------------------------------------
#define LORS_INST(T)                                                                                       \
  template int simt_lors_gemm<T>(bool, const T*, const T*, const uint32_t*, const T*, const T*, const T*, \
                                 T*, int, int, int, int, float, cudaStream_t);                            \
  template int simt_masked_grad<T>(const T*, const T*, const T*, const uint32_t*, const T*, const T*,     \
                                   float*, float*, int, int, int, int, float, cudaStream_t);              \
  template int colsum<T>(const T*, float*, int, int, cudaStream_t);                                       \
  template int effective_weight<T>(const T*, const uint32_t*, const T*, const T*, T*, int, int, int,      \
                                   float, cudaStream_t);                                                  \
  template int pack_mask<T>(const T*, uint32_t*, int, int, cudaStream_t);                                 \
  template int compress24<T>(const T*, T*, uint8_t*, int32_t*, int, int, cudaStream_t);                   \
  template int grad_outer<T>(const T*, const T*, const T*, float*, int, int, int, int, cudaStream_t);

LORS_INST(float)
LORS_INST(__nv_bfloat16)

template int simt_strided_gemm<float, float, float>(const float*, int64_t, int64_t, const float*, int64_t,
                                                    int64_t, float*, int64_t, int64_t, int, int, int, float,
                                                    bool, cudaStream_t);
template int simt_strided_gemm<__nv_bfloat16, __nv_bfloat16, float>(const __nv_bfloat16*, int64_t, int64_t,
                                                                    const __nv_bfloat16*, int64_t, int64_t,
                                                                    float*, int64_t, int64_t, int, int, int,
                                                                    float, bool, cudaStream_t);
template int simt_strided_gemm<__nv_bfloat16, __nv_bfloat16, __nv_bfloat16>(
    const __nv_bfloat16*, int64_t, int64_t, const __nv_bfloat16*, int64_t, int64_t, __nv_bfloat16*, int64_t,
    int64_t, int, int, int, float, bool, cudaStream_t);
template int simt_strided_gemm<__nv_bfloat16, float, float>(const __nv_bfloat16*, int64_t, int64_t, const float*,
                                                            int64_t, int64_t, float*, int64_t, int64_t, int, int,
                                                            int, float, bool, cudaStream_t);
template int simt_strided_gemm<float, __nv_bfloat16, float>(const float*, int64_t, int64_t, const __nv_bfloat16*,
                                                            int64_t, int64_t, float*, int64_t, int64_t, int, int,
                                                            int, float, bool, cudaStream_t);

}  // namespace lors
