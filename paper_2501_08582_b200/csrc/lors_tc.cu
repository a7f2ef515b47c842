// bf16 tensor-core path of the LoRS layer: tcgen05.mma with TMEM accumulators,
// TMA-staged operands, mbarrier pipelines, warp-specialised CTAs.
//
//   K1 tc_lors_gemm<false>  Y_t  = X_t  . W_eff^T   (lors_forward,  adapters.py:359-373)
//   K3 tc_lors_gemm<true>   dX_t = dY_t . W_eff     (lors_backward, adapters.py:395)
//        W_eff tiles are rebuilt in the prologue of every k-step: a rank-r
//        tcgen05 MMA forms (a b) for the tile in TMEM, a transform warpgroup
//        adds W, applies M = (W != 0) (or the packed bits) with a select,
//        rounds to bf16 and writes the swizzled operand tile to shared memory,
//        which the main MMA consumes.  W_eff never touches HBM.
//        Dense kernels: 256 features x 384 tokens per CTA pair (two accumulators),
//        persistent over the tile raster, the last wave's tiles optionally cut
//        along K (tail split, off under LORS_FLAG_NO_TAIL_SPLIT); the 2:4 kernel
//        (tcgen05.mma.sp) runs the same persistent 384-token walk.  Grouped forward
//        (lors_fwd_group): the pair tiles of G projections of one X in one walk, the
//        outputs through a 3-D [G][L][R] TMA map.  DESIGN.md section 4 has the pipeline.
//   K4 tc_skinny            rank-r products P = X b^T and dB = alpha Q^T X
//        (adapters.py:396, 399), N = r, split-K into fp32 accumulators.
//   K4b tc_q_da             Q = dY a and dA = alpha dY^T P from one pass over dY
//        (adapters.py:397-398), partials by TMA bulk reduce-add.
//   K5 tc_masked_grad_pair  G = (dY^T X) . M in TMEM on CTA pairs, contracted into
//        dA / dB (the sqft_gc masked gradient, adapters.py:303-312).
//   LORS_FLAG_DETERMINISTIC: the rank-r products and K5 write split partials to
//        workspace slabs that one kernel sums in a fixed order (no atomics, no TMA
//        reduce-adds), so dA / dB are bitwise reproducible run to run.
//
// Shapes that the TMA path cannot address (rows not 16-byte multiples, or
// r > 64) run the FFMA kernels of lors_simt.cu instead.
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "lors_simt.cuh"
#include "lors_tc.cuh"
#include "ptx_sm100.cuh"

#ifdef LORS_TRACE
// timeline experiment (tools/trace_k1.py): globaltimer stamps of pipeline events of the first CTA
// pair, per flat k-step g < 512: g_lors_trace[(cta * 16 + event) * 512 + g]
__device__ unsigned long long g_lors_trace[2 * 24 * 512];
extern "C" int lors_trace_read(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_lors_trace, sizeof(unsigned long long) * 2 * 24 * 512);
}
#define LORS_TR(ev, g)                                                                          \
  do {                                                                                         \
    if (blockIdx.x < 2 && (g) < 512) g_lors_trace[(blockIdx.x * 24 + (ev)) * 512 + (g)] = clock64(); \
  } while (0)
#else
#define LORS_TR(ev, g) \
  do {                 \
  } while (0)
#endif
#ifdef LORS_DEBUG_HANG
extern "C" int lors_debug_hang_info(unsigned int* out) {
  return (int)cudaMemcpyFromSymbol(out, lors::ptx::g_lors_hang, sizeof(unsigned int) * 64);
}
#endif

namespace lors {
using bf16 = __nv_bfloat16;
using namespace ptx;

// ===========================================================================
// host: tensor maps
// ===========================================================================
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(p);
  }
  return fn;
}

static CUtensorMapSwizzle to_swizzle(uint32_t bytes) {
  switch (bytes) {
    case 128: return CU_TENSOR_MAP_SWIZZLE_128B;
    case 64: return CU_TENSOR_MAP_SWIZZLE_64B;
    case 32: return CU_TENSOR_MAP_SWIZZLE_32B;
    default: return CU_TENSOR_MAP_SWIZZLE_NONE;
  }
}

// 2-D bf16 tensor [outer, inner] row-major (row stride = inner elements).
static int make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
                    uint32_t box_outer, uint32_t swizzle_bytes, const char* what, bool f32 = false) {
  PFN_encodeTiled_t fn = encode_fn();
  if (fn == nullptr) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return LORS_ERR_CUDA;
  }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * (f32 ? sizeof(float) : sizeof(bf16))};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, to_swizzle(swizzle_bytes), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error(std::string("cuTensorMapEncodeTiled failed for ") + what + " (CUresult " + std::to_string((int)r) +
              ")");
    return LORS_ERR_CUDA;
  }
  return LORS_OK;
}

// 3-D bf16 tensor [depth][outer][inner] with a dense [outer][inner] plane per depth index (the
// grouped forward's [G][L][R] outputs), box depth 1
static int make_map_3d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t depth,
                       uint32_t box_inner, uint32_t box_outer, uint32_t swizzle_bytes, const char* what) {
  PFN_encodeTiled_t fn = encode_fn();
  if (fn == nullptr) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return LORS_ERR_CUDA;
  }
  cuuint64_t dims[3] = {inner, outer, depth};
  cuuint64_t strides[2] = {inner * sizeof(bf16), inner * outer * sizeof(bf16)};
  cuuint32_t box[3] = {box_inner, box_outer, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, to_swizzle(swizzle_bytes), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error(std::string("cuTensorMapEncodeTiled failed for ") + what + " (CUresult " + std::to_string((int)r) +
              ")");
    return LORS_ERR_CUDA;
  }
  return LORS_OK;
}

// 2-D byte tensor [outer][inner], no swizzle (the 2:4 metadata boxes)
static int make_map_u8(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
                       uint32_t box_outer, const char* what) {
  PFN_encodeTiled_t fn = encode_fn();
  if (fn == nullptr) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return LORS_ERR_CUDA;
  }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error(std::string("cuTensorMapEncodeTiled failed for ") + what + " (CUresult " + std::to_string((int)r) + ")");
    return LORS_ERR_CUDA;
  }
  return LORS_OK;
}

static int num_sms() {
  static int n[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (n[dev] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 1 ? v : 148;
  }
  return n[dev];
}

// fp32 -> bf16 of the split-K rank-r side products (P and Q in one launch)
__global__ void f32_to_bf16_pair_kernel(const float4* __restrict__ a32, __nv_bfloat16* __restrict__ a16, int64_t na4,
                                        const float4* __restrict__ b32, __nv_bfloat16* __restrict__ b16, int64_t nb4) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const float4* src = i < na4 ? a32 : b32;
  __nv_bfloat16* dst = i < na4 ? a16 : b16;
  const int64_t j = i < na4 ? i : i - na4;
  if (i >= na4 + nb4) return;
  const float4 v = src[j];
  uint2 o;
  o.x = ptx::pack_bf16x2(v.x, v.y);
  o.y = ptx::pack_bf16x2(v.z, v.w);
  reinterpret_cast<uint2*>(dst)[j] = o;
}

static inline uint32_t pad_rank(int r) { return r <= 16 ? 16 : r <= 32 ? 32 : 64; }
// alpha a (normal) power of two: bf16(alpha P) = alpha bf16(P), weff_pair's fused form applies
static inline bool alpha_pow2(float alpha) {
  uint32_t u;
  std::memcpy(&u, &alpha, sizeof u);
  const uint32_t e = (u >> 23) & 0xFFu;
  return (u & 0x7FFFFFu) == 0 && e > 0 && e < 255;
}

// ===========================================================================
// K4: skinny GEMM  D[M, BN] = sum_k A[m, k] B[n, k]   (M tile 128, BN = padded r)
//   A_MN / B_MN: operand stored MN-major (m resp. n contiguous) instead of K-major.
//   OUT 0: bf16 out[m*ldo + n]; 1: fp32 alpha*out[m*ldo + n]; 2: fp32 alpha*out[n*ldo + m]
//   out_mode 0: plain stores; 1: the grid splits K and 1/2 accumulate atomically (OUT 0:
//   fp32 red.add into a caller-zeroed accumulator); 2 (deterministic): split s stores its raw
//   fp32 partial to out[s][M][BN], summed in split order by skinny_reduce_kernel.
// warps: 0 TMA producer, 1 MMA issuer + TMEM owner, 2..5 epilogue.
// ===========================================================================
namespace sk {
constexpr int BM = 128, BK = 64, STAGES = 4, THREADS = 192;
template <int BN>
constexpr uint32_t b_bytes() { return BN * BK * 2; }
constexpr uint32_t A_BYTES = BM * BK * 2;
template <int BN>
constexpr size_t smem_bytes() { return 1024 + STAGES * (A_BYTES + b_bytes<BN>()) + 256; }
}  // namespace sk

template <int BN, bool A_MN, bool B_MN, int OUT>
__global__ void __launch_bounds__(sk::THREADS, 1)
    tc_skinny_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, void* out,
                     int M, int N, int K, int k_per_split, int ldo, float alpha, int out_mode) {
  using namespace sk;
  constexpr uint32_t B_BYTES = b_bytes<BN>();
  constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
  constexpr uint32_t SWB = B_MN ? BN * 2 : 128;  // B swizzle span (bytes)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* accf = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);

  const int warp = warp_id(), lane = lane_id();
  const int m0 = blockIdx.x * BM;
  const int kbeg = blockIdx.y * k_per_split;
  const int kend = min(K, kbeg + k_per_split);
  const int nk = (kend - kbeg + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accf, 1);
    fence_barrier_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < nk; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], A_BYTES + B_BYTES);
        const int k0 = kbeg + i * BK;
        uint8_t* a = sA + s * A_BYTES;
        uint8_t* b = sB + s * B_BYTES;
        if (A_MN) {  // two 64-wide MN atoms of [64 k-rows x 128 B]
          tma_load_2d(a, &tmA, &full[s], m0, k0);
          tma_load_2d(a + A_BYTES / 2, &tmA, &full[s], m0 + 64, k0);
        } else {
          tma_load_2d(a, &tmA, &full[s], k0, m0);
        }
        if (B_MN) {
          tma_load_2d(b, &tmB, &full[s], 0, k0);
        } else {
          tma_load_2d(b, &tmB, &full[s], k0, 0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(BM, BN, A_MN, B_MN);
      for (int i = 0; i < nk; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t a_base = smem_u32(sA + s * A_BYTES), b_base = smem_u32(sB + s * B_BYTES);
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk) {
          const uint64_t ad = A_MN ? make_sdesc(a_base + kk * 2048, A_BYTES / 2, 1024, SW_128)
                                   : make_sdesc(a_base + kk * 32, 16, 1024, SW_128);
          const uint64_t bd = B_MN ? make_sdesc(b_base + kk * 16 * SWB, 0, 8 * SWB, sw_layout(SWB))
                                   : make_sdesc(b_base + kk * 32, 16, 1024, SW_128);
          mma_bf16(tmem, ad, bd, idesc, (i > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(&empty[s]);
      }
      mma_commit(accf);
    }
  } else {
    mbar_wait(accf, 0);
    tc_fence_after();
    const int q = warp % 4;
    const int m = m0 + q * 32 + lane;
    const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16);
#pragma unroll
    for (int c0 = 0; c0 < BN; c0 += 16) {
      uint32_t v[16];
      tmem_ld_x16(taddr + c0, v);
      tmem_ld_wait();
      if (m < M) {
        if (out_mode == 2) {   // deterministic split: this split's partial row, plain stores
          float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) +
                                                ((int64_t)blockIdx.y * M + m) * BN + c0);
#pragma unroll
          for (int h = 0; h < 4; ++h)
            o[h] = make_float4(__uint_as_float(v[h * 4]), __uint_as_float(v[h * 4 + 1]), __uint_as_float(v[h * 4 + 2]),
                               __uint_as_float(v[h * 4 + 3]));
        } else if (OUT == 0 && out_mode) {  // split-K partial: fp32 sums, converted to bf16 afterwards
          float* o = reinterpret_cast<float*>(out) + (int64_t)m * ldo + c0;
#pragma unroll
          for (int h = 0; h < 4; ++h)
            if (c0 + h * 4 + 4 <= N)
              red_add_v4(o + h * 4, __uint_as_float(v[h * 4]), __uint_as_float(v[h * 4 + 1]),
                         __uint_as_float(v[h * 4 + 2]), __uint_as_float(v[h * 4 + 3]));
        } else if (OUT == 0) {
          bf16* o = reinterpret_cast<bf16*>(out) + (int64_t)m * ldo + c0;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (c0 + h * 8 + 8 <= N) {
              uint4 pk;
              pk.x = pack_bf16x2(__uint_as_float(v[h * 8 + 0]), __uint_as_float(v[h * 8 + 1]));
              pk.y = pack_bf16x2(__uint_as_float(v[h * 8 + 2]), __uint_as_float(v[h * 8 + 3]));
              pk.z = pack_bf16x2(__uint_as_float(v[h * 8 + 4]), __uint_as_float(v[h * 8 + 5]));
              pk.w = pack_bf16x2(__uint_as_float(v[h * 8 + 6]), __uint_as_float(v[h * 8 + 7]));
              *reinterpret_cast<uint4*>(o + h * 8) = pk;
            }
          }
        } else {
          float* o = reinterpret_cast<float*>(out);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int n = c0 + j;
            if (n < N) {
              const float val = alpha * __uint_as_float(v[j]);
              float* dst = OUT == 1 ? o + (int64_t)m * ldo + n : o + (int64_t)n * ldo + m;
              if (out_mode) atomicAdd(dst, val);
              else *dst = val;
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<TMEM_COLS>(tmem);
}

// host launcher for one skinny product.
//   A: K-major tensor [M, K] (A_MN=false) or MN-major [K, M] (A_MN=true), bf16
//   B: K-major [N, K] or MN-major [K, N]
// deterministic split: out[m, n] (OUT's layout) = alpha * sum over s in order of part[s][m][n]
template <int OUT>
__global__ void skinny_reduce_kernel(const float* __restrict__ part, int split, int M, int N, int BN, void* out,
                                     int ldo, float alpha) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)M * N) return;
  const int m = OUT == 2 ? (int)(i % M) : (int)(i / N);   // OUT 2 writes along m (coalesced)
  const int n = OUT == 2 ? (int)(i / M) : (int)(i % N);
  float acc = 0.f;
  for (int k = 0; k < split; ++k) acc += part[((int64_t)k * M + m) * BN + n];
  if (OUT == 0) reinterpret_cast<bf16*>(out)[(int64_t)m * ldo + n] = __float2bfloat16_rn(acc);
  else if (OUT == 1) reinterpret_cast<float*>(out)[(int64_t)m * ldo + n] = alpha * acc;
  else reinterpret_cast<float*>(out)[(int64_t)n * ldo + m] = alpha * acc;
}

// K split of a skinny product: the CTAs fill one wave at two resident per SM (never a
// second, mostly empty wave) and every split keeps >= 4 k-blocks
static int skinny_split(int M, int K) {
  const int mt = (int)ceil_div(M, sk::BM), kblocks = (int)ceil_div(K, sk::BK);
  const int split = (int)std::max<int64_t>(1, std::min<int64_t>((2 * num_sms()) / mt, kblocks / 4));
  const int kps = (int)ceil_div(kblocks, split) * sk::BK;
  return (int)ceil_div(K, kps);
}
// bytes of the deterministic partials of one skinny product (0 = no split)
static size_t skinny_partial_bytes(int M, int K, int bn) {
  const int split = skinny_split(M, K);
  return split > 1 ? (size_t)split * (size_t)M * (size_t)bn * sizeof(float) : 0;
}

template <int BN, bool A_MN, bool B_MN, int OUT>
static int launch_skinny(const bf16* A, const bf16* B, void* out, int M, int N, int K, int ldo, float alpha,
                         bool allow_split, cudaStream_t s, float* acc32 = nullptr, bool zeroed = false,
                         float* det_part = nullptr) {
  CUtensorMap tA, tB;
  int st;
  if (A_MN) st = make_map(&tA, A, M, K, 64, 64, 128, "skinny A (MN)");
  else st = make_map(&tA, A, K, M, 64, 128, 128, "skinny A (K)");
  if (st) return st;
  if (B_MN) st = make_map(&tB, B, N, K, BN, 64, BN * 2, "skinny B (MN)");
  else st = make_map(&tB, B, K, N, 64, BN, 128, "skinny B (K)");
  if (st) return st;
  const int mt = (int)ceil_div(M, sk::BM);
  const int kblocks = (int)ceil_div(K, sk::BK);
  // split K so that the CTAs fill one wave at two resident per SM (never a
  // second, mostly empty wave); OUT 0 splits only into a caller-zeroed fp32
  // accumulator (acc32)
  int split = 1;
  const bool can_split = allow_split && (OUT != 0 || acc32 != nullptr || det_part != nullptr);
  if (can_split) split = skinny_split(M, K);
  const int kps = (int)ceil_div(kblocks, split) * sk::BK;
  auto kern = tc_skinny_kernel<BN, A_MN, B_MN, OUT>;
  const size_t smem = sk::smem_bytes<BN>();
  LORS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                "skinny smem attribute");
  if (det_part != nullptr && split > 1) {   // deterministic: partials, then one ordered sum
    kern<<<dim3(mt, split), sk::THREADS, smem, s>>>(tA, tB, det_part, M, N, K, kps, ldo, alpha, 2);
    LORS_CHECK_LAUNCH("tc_skinny (partials)");
    const int64_t n = (int64_t)M * N;
    skinny_reduce_kernel<OUT><<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(det_part, split, M, N, BN, out, ldo, alpha);
    LORS_CHECK_LAUNCH("skinny_reduce");
    return LORS_OK;
  }
  if (split > 1 && OUT != 0 && !zeroed) {
    const size_t elems = OUT == 2 ? (size_t)N * ldo : (size_t)M * ldo;
    LORS_CUDA_TRY(cudaMemsetAsync(out, 0, elems * sizeof(float), s), "zero split-K output");
  }
  if (OUT == 0 && acc32 != nullptr && det_part == nullptr) out = acc32;  // fp32 sums; the caller converts to bf16
  const int atomic_out = (split > 1 || (OUT == 0 && acc32 != nullptr && det_part == nullptr)) ? 1 : 0;
  kern<<<dim3(mt, split), sk::THREADS, smem, s>>>(tA, tB, out, M, N, K, kps, ldo, alpha, atomic_out);
  LORS_CHECK_LAUNCH("tc_skinny");
  return LORS_OK;
}

// dispatch on the padded rank
template <bool A_MN, bool B_MN, int OUT>
static int skinny(int rp, const bf16* A, const bf16* B, void* out, int M, int N, int K, int ldo, float alpha,
                  bool allow_split, cudaStream_t s, float* acc32 = nullptr, bool zeroed = false,
                  float* det_part = nullptr) {
  switch (rp) {
    case 16:
      return launch_skinny<16, A_MN, B_MN, OUT>(A, B, out, M, N, K, ldo, alpha, allow_split, s, acc32, zeroed, det_part);
    case 32:
      return launch_skinny<32, A_MN, B_MN, OUT>(A, B, out, M, N, K, ldo, alpha, allow_split, s, acc32, zeroed, det_part);
    default:
      return launch_skinny<64, A_MN, B_MN, OUT>(A, B, out, M, N, K, ldo, alpha, allow_split, s, acc32, zeroed, det_part);
  }
}

// ===========================================================================
// K4b: Q and dA from one pass over dY (lors_backward at_dy and da, adapters.py:397-398)
//
//   Q[l, :]  = sum_R dY_t[l, R] a[R, :]          (fp32, red.add; rounded to bf16 after)
//   dA[R, :] = alpha sum_l dY_t[l, R] P[l, :]    (fp32, red.add)
//
// Every [128 tokens x 128 R] block of dY_t is staged once (two SW128 boxes) and
// feeds two MMAs: read K-major it is the A operand of Q (M = tokens, K = R), read
// MN-major it is the A operand of dA (M = R, K = tokens).  A CTA owns Tr R tiles
// (their a slices stay resident in shared memory, their dA accumulators in TMEM)
// and a run of token tiles (the P slice of the current one double-buffered, its Q
// accumulator double-buffered so that the flush overlaps the next tile).  Partial
// Q / dA tiles leave through a swizzled fp32 staging box and a TMA bulk reduce-add
// (one instruction per tile instead of a red.add per thread and row).
// warps: 0 TMA producer, 1 MMA issuer + TMEM owner, 2..5 flush.
// ===========================================================================
namespace qd {
constexpr int THREADS = 192, MAX_STAGES = 8, MIN_STAGES = 3;
constexpr uint32_t BLK_BYTES = 128 * 128 * 2;   // dY block, two [128 tokens][64 R] boxes
constexpr size_t SMEM_MAX = 232448;
template <int BN>
constexpr int tr_tmem() { return 512 / BN - 2; }                      // 30 / 14 / 6 (TMEM columns)
template <int BN>
constexpr uint32_t slice_bytes() { return 128 * BN * 2; }
// fp32 staging of one [128 rows][BN] accumulator for the TMA reduce-add: SW128
// boxes of [128 rows][32 floats] (one for BN <= 32)
template <int BN>
constexpr uint32_t stage_out_bytes() { return BN <= 32 ? 16384 : 32768; }
template <int BN>
constexpr size_t fixed_bytes(int tr) {
  return 1024 + (size_t)(tr + 2) * slice_bytes<BN>() + stage_out_bytes<BN>() + 512;
}
// the dY ring takes what the resident a slices, P and the staging leave
template <int BN>
constexpr int stages(int tr) {
  const int s = (int)((SMEM_MAX - fixed_bytes<BN>(tr)) / BLK_BYTES);
  return s < MAX_STAGES ? s : MAX_STAGES;
}
template <int BN>
constexpr int tr_max() {   // TMEM- and shared-memory-bound (keeps MIN_STAGES blocks in flight)
  int t = tr_tmem<BN>();
  while (t > 1 && stages<BN>(t) < MIN_STAGES) --t;
  return t;
}
template <int BN>
constexpr size_t smem_bytes(int tr) { return fixed_bytes<BN>(tr) + stages<BN>(tr) * BLK_BYTES; }
}  // namespace qd

template <int BN>
__global__ void __launch_bounds__(qd::THREADS, 1)
    tc_q_da_kernel(const __grid_constant__ CUtensorMap tmDY, const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmQ,
                   const __grid_constant__ CUtensorMap tmDA, int L, int R, int r, int tr, int tpg, int n_rg,
                   float alpha) {
  using namespace qd;
  constexpr uint32_t SL = slice_bytes<BN>();
  constexpr uint32_t SWB = BN * 2;               // swizzle span of the a / P slices (MN-major B)
  const int STAGES = stages<BN>(tr);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;                            // [tr] a slices
  uint8_t* sp = sa + tr * SL;                    // [2] P slices
  uint8_t* sout = sp + 2 * SL;                   // fp32 staging of a Q / dA tile (SW128 boxes)
  uint8_t* sdy = sout + stage_out_bytes<BN>();   // [STAGES] dY blocks
  uint64_t* full = reinterpret_cast<uint64_t*>(sdy + STAGES * BLK_BYTES);
  uint64_t* empty = full + MAX_STAGES;
  uint64_t* pfull = empty + MAX_STAGES;          // [2]
  uint64_t* pempty = pfull + 2;                  // [2]
  uint64_t* qfull = pempty + 2;                  // [2]
  uint64_t* qempty = qfull + 2;                  // [2]
  uint64_t* afull = qempty + 2;
  uint64_t* dafull = afull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dafull + 1);

  const int warp = warp_id(), lane = lane_id();
  const int n_rt = (R + 127) / 128, n_tt = (L + 127) / 128;
  const int rg = (int)blockIdx.x % n_rg, tg = (int)blockIdx.x / n_rg;
  const int r0 = rg * tr * 128, t0 = tg * tpg * 128;
  const int trc = min(tr, n_rt - rg * tr);       // R tiles of this CTA
  const int ntc = min(tpg, n_tt - tg * tpg);     // token tiles of this CTA
  // TMEM columns: Q accumulators 0 / BN, dA accumulator of R tile j at (2 + j) BN
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&pfull[b], 1);
      mbar_init(&pempty[b], 1);
      mbar_init(&qfull[b], 1);
      mbar_init(&qempty[b], 4);
    }
    mbar_init(afull, 1);
    mbar_init(dafull, 1);
    fence_barrier_init();
    tma_prefetch_desc(&tmDY);
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmP);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (trc <= 0 || ntc <= 0) {                    // (the planner never launches empty CTAs)
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<512>(tmem);
    return;
  }

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(afull, (uint32_t)trc * SL);
      for (int j = 0; j < trc; ++j) tma_load_2d(sa + j * SL, &tmA, afull, 0, r0 + 128 * j);
      for (int ti = 0, i = 0; ti < ntc; ++ti) {
        const int pb = ti & 1, tok = t0 + 128 * ti;
        mbar_wait(&pempty[pb], ((ti >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&pfull[pb], SL);
        tma_load_2d(sp + pb * SL, &tmP, &pfull[pb], 0, tok);
        for (int j = 0; j < trc; ++j, ++i) {
          const int s = i % STAGES;
          mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], BLK_BYTES);
          uint8_t* blk = sdy + s * BLK_BYTES;
          tma_load_2d(blk, &tmDY, &full[s], r0 + 128 * j, tok);
          tma_load_2d(blk + BLK_BYTES / 2, &tmDY, &full[s], r0 + 128 * j + 64, tok);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idq = make_idesc_bf16(128, BN, false, true);   // Q : A = dY (K = R)
      constexpr uint32_t ida = make_idesc_bf16(128, BN, true, true);    // dA: A = dY^T (K = tokens)
      mbar_wait(afull, 0);
      for (int ti = 0, i = 0; ti < ntc; ++ti) {
        const int pb = ti & 1;
        mbar_wait(&pfull[pb], (ti >> 1) & 1);
        mbar_wait(&qempty[pb], ((ti >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t p_base = smem_u32(sp + pb * SL);
        for (int j = 0; j < trc; ++j, ++i) {
          const int s = i % STAGES;
          mbar_wait(&full[s], (i / STAGES) & 1);
          tc_fence_after();
          const uint32_t blk = smem_u32(sdy + s * BLK_BYTES), a_base = smem_u32(sa + j * SL);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {   // Q += dY[128 tok x 128 R] . a[128 R x BN]
            const uint64_t ad = make_sdesc(blk + (kk >> 2) * (BLK_BYTES / 2) + (kk & 3) * 32, 16, 1024, SW_128);
            const uint64_t bd = make_sdesc(a_base + kk * 16 * SWB, 0, 8 * SWB, sw_layout(SWB));
            mma_bf16(tmem + pb * BN, ad, bd, idq, (j > 0 || kk > 0) ? 1u : 0u);
          }
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {   // dA_j += dY^T[128 R x 128 tok] . P[128 tok x BN]
            const uint64_t ad = make_sdesc(blk + kk * 2048, BLK_BYTES / 2, 1024, SW_128);
            const uint64_t bd = make_sdesc(p_base + kk * 16 * SWB, 0, 8 * SWB, sw_layout(SWB));
            mma_bf16(tmem + (2 + j) * BN, ad, bd, ida, (ti > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&qfull[pb]);
        mma_commit(&pempty[pb]);
      }
      mma_commit(dafull);
    }
  } else {
    // Flush: each thread owns one accumulator row (TMEM lane); the row's floats go
    // to the SW128 staging boxes (chunk j of row t at chunk j ^ (t & 7): the eight
    // rows of a bank group land in different banks), then one thread adds the
    // whole tile into global memory with a TMA bulk reduce (full-line L2 atomics,
    // rows / columns outside the tensor skipped by the tensor map).
    const int q = warp % 4;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    const int row = q * 32 + lane;
    const bool issuer = warp == 2 && lane == 0;
    auto stage = [&](const uint32_t col, const float scale) {
#pragma unroll
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t v[16];
        tmem_ld_x16(lane_base + col + c0, v);
        tmem_ld_wait();
        uint8_t* box = sout + (c0 >> 5) * 16384 + row * 128;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = ((c0 & 31) >> 2) + u;
          float4 f = make_float4(scale * __uint_as_float(v[4 * u]), scale * __uint_as_float(v[4 * u + 1]),
                                 scale * __uint_as_float(v[4 * u + 2]), scale * __uint_as_float(v[4 * u + 3]));
          *reinterpret_cast<float4*>(box + ((j ^ (row & 7)) << 4)) = f;
        }
      }
      fence_proxy_async_smem();
    };
    auto reduce_out = [&](const CUtensorMap* m, int row0) {   // after the staging barrier
      if (issuer) {
        tma_reduce_add_2d(m, sout, 0, row0);
        if (BN > 32) tma_reduce_add_2d(m, sout + 16384, 32, row0);
        tma_store_commit();
        tma_store_wait_all();                     // staging reusable (smem read done)
      }
    };
    for (int ti = 0; ti < ntc; ++ti) {            // Q of token tile ti
      const int pb = ti & 1;
      mbar_wait(&qfull[pb], (ti >> 1) & 1);
      tc_fence_after();
      stage(pb * BN, 1.0f);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&qempty[pb]);    // accumulator read: MMA may reuse it
      named_bar_sync(1, 128);
      reduce_out(&tmQ, t0 + 128 * ti);
      named_bar_sync(1, 128);
    }
    mbar_wait(dafull, 0);
    tc_fence_after();
    for (int j = 0; j < trc; ++j) {               // dA of the CTA's R tiles
      stage((2 + j) * BN, alpha);
      named_bar_sync(1, 128);
      reduce_out(&tmDA, r0 + 128 * j);
      named_bar_sync(1, 128);
    }
    if (issuer) tma_store_wait_done();            // the reductions landed in global memory
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// Grid of the Q / dA pass: Tr R tiles x tpg token tiles per CTA, one CTA per SM.
template <int BN>
static int launch_q_da(const bf16* dy, const bf16* a, const bf16* p, float* q32, float* da, int L, int R, int r,
                       float alpha, cudaStream_t s) {
  CUtensorMap tDY, tA, tP;
  int st;
  if ((st = make_map(&tDY, dy, R, L, 64, 128, 128, "dY (Q / dA pass)"))) return st;
  if ((st = make_map(&tA, a, r, R, BN, 128, BN * 2, "a slices (Q / dA pass)"))) return st;
  if ((st = make_map(&tP, p, r, L, BN, 128, BN * 2, "P slices (Q / dA pass)"))) return st;
  CUtensorMap tQ, tDA;   // fp32 outputs, reduce-added in [128 rows][32 floats] SW128 boxes
  if ((st = make_map(&tQ, q32, r, L, 32, 128, 128, "Q fp32 (Q / dA pass)", true))) return st;
  if ((st = make_map(&tDA, da, r, R, 32, 128, 128, "dA fp32 (Q / dA pass)", true))) return st;
  const int n_rt = (int)ceil_div(R, 128), n_tt = (int)ceil_div(L, 128), nsm = num_sms();
  // Tr minimising the blocks of the busiest CTA (the main loop streams ~27 GB/s per
  // SM whatever the rank; the TMA reductions of the partials are cheap); ties go to
  // the smallest Tr >= 2 (longer token runs per CTA, a shorter dA flush at the end).
  // Forced Tr: LORS_QDA_TR (experiments, tools/exp_qda_sweep.py).
  const int trm = std::min(qd::tr_max<BN>(), n_rt);
  int best_tr = trm, best_work = INT32_MAX;
  for (int tr = trm; tr >= 1; --tr) {
    const int n_rg = (int)ceil_div(n_rt, tr);
    if (n_rg > nsm) break;
    const int tpg = (int)ceil_div(n_tt, std::min(n_tt, std::max(1, nsm / n_rg)));
    if (tr * tpg < best_work || (tr * tpg == best_work && tr >= 2)) best_tr = tr, best_work = tr * tpg;
  }
  if (const char* force = getenv("LORS_QDA_TR")) best_tr = std::max(1, std::min(atoi(force), trm));
  while ((int)ceil_div(n_rt, best_tr) > nsm && best_tr < trm) ++best_tr;   // q_da_fits() holds
  const int best_tpg = (int)ceil_div(n_tt, std::min(n_tt, std::max(1, nsm / (int)ceil_div(n_rt, best_tr))));
  const int n_rg = (int)ceil_div(n_rt, best_tr);
  const int ctas = n_rg * (int)ceil_div(n_tt, best_tpg);
  auto kern = tc_q_da_kernel<BN>;
  const size_t smem = qd::smem_bytes<BN>(best_tr);
  LORS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                "q_da smem attribute");
  kern<<<ctas, qd::THREADS, smem, s>>>(tDY, tA, tP, tQ, tDA, L, R, r, best_tr, best_tpg, n_rg, alpha);
  LORS_CHECK_LAUNCH("tc_q_da");
  return LORS_OK;
}

// whether one wave of CTAs covers R at the largest Tr (else the separate skinny GEMMs run)
static bool q_da_fits(int rp, int R) {
  const int trm = rp == 16 ? qd::tr_max<16>() : rp == 32 ? qd::tr_max<32>() : qd::tr_max<64>();
  return ceil_div(R, 128) <= (int64_t)num_sms() * trm;
}

static int q_da(int rp, const bf16* dy, const bf16* a, const bf16* p, float* q32, float* da, int L, int R, int r,
                float alpha, cudaStream_t s) {
  switch (rp) {
    case 16: return launch_q_da<16>(dy, a, p, q32, da, L, R, r, alpha, s);
    case 32: return launch_q_da<32>(dy, a, p, q32, da, L, R, r, alpha, s);
    default: return launch_q_da<64>(dy, a, p, q32, da, L, R, r, alpha, s);
  }
}

// ===========================================================================
// K1 / K3: GEMM with W_eff rebuilt in the prologue, on CTA pairs.
//
//   out[l, m] = sum_k act[l, k] * Weff'(m, k)
//   FWD (DX=false): act = X_t [L, C], m over R, k over C, Weff'(m,k) = Weff[m,k]
//   DX  (DX=true) : act = dY_t [L, R], m over C, k over R, Weff'(m,k) = Weff[k,m]
//
// A cluster of two CTAs computes a 256 (features) x 256 (tokens) tile with
// tcgen05 cta_group::2: CTA c owns features m0 + 128c .. +127 (its TMEM lanes,
// its W / W_eff tiles) and stages tokens l0 + 128c .. +127 of the activation
// tile; the pair MMA (M = 256, N = 256, K = 16) reads both halves, so each SM
// streams half of the activation tile from L2.  Per 64-wide k-step:
//   TMA   : W tile (own rows), activation half, streamed adapter-factor half
//   MMA   : recompute D_re[256 x 64] = F . S^T (K = r) into TMEM (2 buffers)
//   xform : 8 warps per CTA read D_re (tcgen05.ld), add W, select on the mask,
//           round to bf16 and store the K-major SW128 W_eff tile (2 buffers)
//   MMA   : D[256 x 256] += W_eff . act^T (4 x K16), leader CTA issues
// The recompute of step i is issued before the main MMA of step i-1, so the
// transform of step i overlaps the tensor-core work of step i-1.
// warps 0-7: transform + epilogue, warp 8: TMA producer, warp 9: MMA issuer
// (leader CTA) and TMEM owner.
// ===========================================================================
struct alignas(16) Bar16 {
  uint64_t b;
  uint64_t pad;
};

namespace rg {
constexpr int BM = 128, BN = 256, BK = 64;
// warps 0 .. XW-1: transform + epilogue (one group of 8; the non-persistent build,
// LORS_PERSIST=0, can run two groups on alternate k-steps).  Then the roles:
// factor-ring producer, MMA issuer / relay, activation producer, activation
// relay, W-ring producer.
#ifndef LORS_XW_DENSE
#define LORS_XW_DENSE 8
#endif
#ifndef LORS_N2
#define LORS_N2 128
#endif
#ifndef LORS_NW_DENSE
#define LORS_NW_DENSE 4
#endif
#ifndef LORS_NW_SP
#define LORS_NW_SP 4
#endif
#ifndef LORS_PERSIST
#define LORS_PERSIST 1
#endif

// Persistent kernels (dense-masked and 2:4): one CTA pair per SM pair walks its
// tiles; the producers and the recompute run ahead into the next tile while the
// epilogue drains the accumulator through the (then idle) W_eff ring.
template <bool SP>
constexpr bool persist() { return LORS_PERSIST; }
template <bool SP>
constexpr int xw() { return LORS_PERSIST ? LORS_XW_DENSE : (SP ? 16 : LORS_XW_DENSE); }
template <bool SP>
constexpr int threads() { return 32 * (xw<SP>() + 4); }
// Token tile of a CTA pair: 256 + N2 tokens per W_eff tile -- one N = 256 MMA and
// one N = N2 MMA per k-step into two accumulators -- so each on-chip W_eff tile (its
// rank-r recompute, transform and W load) serves 1.5x the tokens.  TMEM: acc 256 + N2
// columns, then NE recompute buffers of 64 (dense: two; 2:4: one), then for 2:4 the
// sparse metadata of the NA W_eff buffers at e_col.  (A 352-token 2:4 tile, N2 = 96,
// fits two recompute buffers next to the metadata; it measured slower, 684 vs 645 us at
// cfg2: the 2:4 pipeline is paced by the transform warps' ~1300-cycle k-step, not by the
// single recompute buffer, tools/trace_k1.py.)
#ifndef LORS_N2_SP
#define LORS_N2_SP 128
#endif
template <bool SP>
constexpr int n2() { return (SP && !LORS_PERSIST) ? 0 : (SP ? LORS_N2_SP : LORS_N2); }
template <bool SP>
constexpr int bnt() { return 256 + n2<SP>(); }            // tokens per pair tile
// TMEM recompute buffers, and the factor ring (streamed adapter-factor half) with its
// own depth NS: a factor slot is free once its recompute committed, a recompute
// buffer once the transform has read it.  The W ring is separate too: the recompute
// of step j needs only its factor slice, W(j) is first read by the transform.
template <bool SP>
constexpr int ne() { return SP ? (LORS_PERSIST ? (512 - 256 - n2<SP>() - 32) / 64 : 3) : (512 - 256 - n2<SP>()) / 64; }
template <bool SP>
constexpr int ns() { return SP ? 3 : 2; }
template <bool SP>
constexpr int nw() { return SP ? (LORS_PERSIST ? LORS_NW_SP : 6) : LORS_NW_DENSE; }  // W ring
#ifndef LORS_NA_SP
#define LORS_NA_SP 3
#endif
template <bool SP>
constexpr int na() { return SP ? (LORS_PERSIST ? LORS_NA_SP : 4) : 3; }  // W_eff buffers
#ifndef LORS_NACT
#define LORS_NACT 3
#endif
// activation ring, its own depth (barriers afull / a_empty) apart from the W_eff ring: an
// activation half is requested when the MMA of the step NACT earlier has finished with its
// slot.  4 slots (with a 3-deep W ring to fit 227 KB) measured no faster than 3 (tools/ab_gemm.py)
template <bool SP>
constexpr int nact() { return LORS_PERSIST ? LORS_NACT : na<SP>(); }
// recompute lookahead D: recompute(j) is issued with main(j - D), so (tcgen05 ops run in
// issue order) it completes right after main(j - D - 1) and the transform of step j has D
// main MMAs to finish before main(j) is due.  tools/trace_k1.py measured the chain
// main(j - 2) done -> recompute(j) -> transform(j) -> issuer sees it -> main(j) at ~1200
// cycles against ~900 for one step's MMAs, so D = 1 left the tensor pipe idle ~25% of the
// time; D = 2 (dense: NE = 2) hides it.
#ifndef LORS_LOOKAHEAD
#define LORS_LOOKAHEAD 2
#endif
// (recompute(j) waits for the transform of j - NE to release its buffer; in the first D
// steps of a tile that transform may sit behind the previous tile's epilogue, so there the
// issuer puts the previous tile's pending main MMAs first, see `flip`)
template <bool SP>
constexpr int lookahead() { return LORS_LOOKAHEAD; }
// 2:4 index nibble (idx0 | idx1 << 2, idx0 < idx1) for each 4-bit keep mask;
// groups with fewer than two kept entries are padded with zero-valued slots,
// masks with more than two are not 2:4 (prune.py:72-77) and never reach here.
constexpr uint64_t nibble_lut() {
  uint64_t lut = 0;
  for (int m = 0; m < 16; ++m) {
    int idx[2] = {-1, -1}, n = 0;
    for (int i = 0; i < 4; ++i)
      if (((m >> i) & 1) && n < 2) idx[n++] = i;
    for (int i = 0; i < 4 && n < 2; ++i)
      if (i != idx[0]) idx[n++] = i;
    if (idx[0] > idx[1]) { int tmp = idx[0]; idx[0] = idx[1]; idx[1] = tmp; }
    lut |= (uint64_t)(idx[0] | (idx[1] << 2)) << (4 * m);
  }
  return lut;
}
constexpr uint64_t kNibbleLut = nibble_lut();
constexpr uint32_t E_COL_NP = 448;  // non-persistent 2:4 build: metadata columns
#ifndef LORS_GROUP_T
#define LORS_GROUP_T 8
#endif
constexpr int GROUP_T = LORS_GROUP_T;  // raster: token tiles per group (clusters of a wave share W and activation tiles)
template <bool SP>
constexpr uint32_t act_bytes() { return (bnt<SP>() / 2) * BK * 2; }   // this CTA's tokens: 24 KB / 16 KB
constexpr uint32_t W_BYTES = BM * BK * 2;           // 16 KB
// W_eff buffer stride: 16 KB (the 2:4 kernel's compressed tile uses the first half; the
// persistent epilogue stages 16 KB output blocks through these buffers)
template <bool SP>
constexpr uint32_t weff_bytes() { return (SP && !LORS_PERSIST) ? BM * BK : BM * BK * 2; }
constexpr uint32_t TMEM_COLS = 512;
template <bool SP>
constexpr uint32_t re_col() { return 256 + n2<SP>(); }  // recompute buffers at TMEM cols re_col + 64 e
// 2:4 metadata: W_eff buffer b, MMA h at column e_col + 8 b + 4 h
template <bool SP>
constexpr uint32_t e_col() { return LORS_PERSIST ? re_col<SP>() + ne<SP>() * 64 : E_COL_NP; }
// accumulator drain: chunks of 128 tokens (the last one BNT - 128 (nch - 1)), stored in
// boxes of out_rows token rows (32 when a chunk is partial, so no store crosses the tile)
template <bool SP>
constexpr int nch() { return (bnt<SP>() + 127) / 128; }
template <bool SP>
constexpr int out_rows() { return bnt<SP>() % 128 ? 32 : 128; }
template <int RP>
constexpr uint32_t sf_bytes() { return 32 * RP * 2; }   // streamed factor half (32 k x RP)
template <int RP>
constexpr uint32_t ff_bytes() { return 128 * RP * 2; }  // fixed factor tile (128 m x RP)
// 2:4 with precomputed metadata: each W slot carries the TMA box of meta24 rows m0 .. m0+127,
// bytes [16 (kq / 2), +16) (the 16 index nibbles a row of k-steps kq & ~1 and kq | 1), and a
// 256-entry table maps a metadata byte (two groups' nibbles) to the two groups' prmt selectors
template <bool SP>
constexpr uint32_t meta_bytes() { return SP ? 128 * 16 : 0; }
template <bool SP>
constexpr uint32_t sel_lut_bytes() { return SP ? 256 * 4 : 0; }
template <int RP, bool SP>
constexpr size_t smem_bytes() {
  return 1024 + ns<SP>() * sf_bytes<RP>() + nw<SP>() * (W_BYTES + meta_bytes<SP>()) + nact<SP>() * act_bytes<SP>() +
         na<SP>() * weff_bytes<SP>() + ff_bytes<RP>() + sel_lut_bytes<SP>() + 1024;
}
}  // namespace rg

// EX (K6 export, forward orientation only): no activations, no main MMA, no
// accumulator -- each transformed W_eff tile is TMA-stored to W_eff [R, C]
// instead of being consumed, so lors_effective_weight / merge() return exactly
// the tiles the forward's tensor cores multiply (same recompute MMA, same
// weff_pair).
// P2: alpha is a power of two (the default 2.0) -- weff_pair's fused three-instruction form;
// the host picks the instantiation from alpha (alpha_pow2), so the transform carries one form.
template <bool DX, int RP, bool BITS, bool SP, bool EX = false, bool P2 = true>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(rg::threads<SP>(), 1)
    tc_lors_gemm_kernel(const __grid_constant__ CUtensorMap tmAct, const __grid_constant__ CUtensorMap tmAct2,
                        const __grid_constant__ CUtensorMap tmW,
                        const __grid_constant__ CUtensorMap tmS, const __grid_constant__ CUtensorMap tmF,
                        const __grid_constant__ CUtensorMap tmOut, const __grid_constant__ CUtensorMap tmMeta,
                        const bf16* __restrict__ bias,
                        const uint32_t* __restrict__ bits, const uint8_t* __restrict__ meta24, int words_per_row,
                        int Mout, int Kred, int n_t, int n_f, int split, float* __restrict__ partials,
                        unsigned int* __restrict__ counters, float alpha, int n_tok, int grp_rows, int grp_r) {
  using namespace rg;
  static_assert(!(SP && DX), "2:4 sparse tensor cores apply to the forward only (SURVEY C6)");
  // Grouped forward (lors_fwd_group; grp_rows < Mout): G projections of one input whose W [G R, C],
  // a [G R, r] and b [G r, C] are consecutive and whose outputs are the 3-D [G][L][R] tmOut; a pair
  // tile never straddles two projections (R % 256 == 0).  grp_rows = Mout: one projection.
  const bool grouped = grp_rows < Mout;
  auto store_out = [&](const void* src, int m, int l) {
    if (grouped) tma_store_3d(&tmOut, src, m % grp_rows, l, m / grp_rows);
    else tma_store_2d(&tmOut, src, m, l);
  };
  static_assert(!EX || (!DX && !SP && LORS_PERSIST), "W_eff export runs the persistent forward prologue");
  constexpr int XW = xw<SP>(), XFORM_THREADS = 32 * XW;
  constexpr int W_SF = XW, W_MMA = XW + 1, W_ACT = XW + 2, W_RELAY = XW + 3;   // W ring: lane 1 of W_SF
  constexpr int NE = ne<SP>(), NS = ns<SP>(), NW = nw<SP>(), NA = na<SP>(), NACT = nact<SP>(), D = lookahead<SP>();
  constexpr int NGRP = XW / 8;          // transform groups (alternate k-steps)
  constexpr bool PERSIST = persist<SP>();
  static_assert(!PERSIST || NGRP == 1, "persistent schedule assumes one transform group");
  static_assert(smem_bytes<RP, SP>() <= 232448, "shared memory: rings exceed 227 KB");
  constexpr uint32_t E_COL = e_col<SP>();
  static_assert(re_col<SP>() + NE * 64 <= (SP ? E_COL : TMEM_COLS) && (!SP || E_COL + NA * 8 <= TMEM_COLS),
                "TMEM: accumulators, recompute buffers and 2:4 metadata must fit 512 columns");
  constexpr int N2 = n2<SP>(), BNT = bnt<SP>();
  constexpr uint32_t ACT_BYTES = act_bytes<SP>(), ACT1_BYTES = 128 * BK * 2;
  constexpr uint32_t RE_COL = re_col<SP>();
  constexpr uint32_t WEFF_BYTES = weff_bytes<SP>();
  // a ring used by the transform groups round robin: the period (in k-steps)
  // between two uses of one slot by the same group, so phase parities of the
  // per-group barrier sets stay sequential for odd ring sizes
  constexpr int RE_PERIOD = (NE % NGRP) ? NGRP * NE : NE;
  constexpr int W_PERIOD = (NW % NGRP) ? NGRP * NW : NW;
  constexpr int A_PERIOD = (NA % NGRP) ? NGRP * NA : NA;
  constexpr uint32_t SF = sf_bytes<RP>(), FF = ff_bytes<RP>();
  constexpr uint32_t SWR = RP * 2;  // swizzle span of the K-major rank-r tiles
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sfr = smem;                       // [NS] streamed factor halves
  uint8_t* wring = sfr + NS * SF;            // [NW] W tiles
  uint8_t* actb = wring + NW * W_BYTES;      // [NACT] activation halves
  uint8_t* weff = actb + NACT * ACT_BYTES;   // [NA] W_eff tiles
  uint8_t* ffac = weff + NA * WEFF_BYTES;    // fixed factor
  uint8_t* mring = ffac + FF;                // [NW] 2:4 metadata boxes (meta24 != nullptr), one per W slot
  uint32_t* sel_lut = reinterpret_cast<uint32_t*>(mring + NW * meta_bytes<SP>());  // 2:4: byte -> 2 selectors
  // mbarriers, one per 16 bytes.  sready / afull count 2 in the leader (own TMA
  // load with its bytes + the peer's relayed landing), 1 in the peer (its own
  // landing); refree / wready count the 16 transform warps of both CTAs.
  Bar16* bars = reinterpret_cast<Bar16*>(mring + NW * meta_bytes<SP>() + sel_lut_bytes<SP>());
  Bar16* sready = bars;                 // [NS] factor slot landed (both CTAs, in the leader)
  Bar16* s_empty = sready + NS;         // [NS] local: recompute committed (factor slot free)
  Bar16* refree = s_empty + NS;         // [NE] leader: 16 transform warps read the recompute buffer
  Bar16* afull = refree + NE;           // [NACT] activation half landed (both CTAs, in the leader)
  Bar16* wready = afull + NACT;         // [NA] leader: W_eff buffer written by the 16 transform warps
  Bar16* a_empty = wready + NA;         // [NACT] local: pair MMA done with the activation half
  // [2][NE] local: recompute landed in TMEM, one set per transform group so that
  // with an odd NE (buffers alternate between the groups) no waiter runs two
  // phases ahead of a barrier
  Bar16* refull = a_empty + NACT;
  // [2][NA] local: pair MMA done with the W_eff buffer, set = group of the next writer
  Bar16* wempty = refull + 2 * NE;
  uint64_t* ffull = &(wempty + 2 * NA)->b;      // local: own fixed factor landed
  uint64_t* pffull = &(wempty + 2 * NA + 1)->b; // leader: peer's fixed factor landed (relayed)
  uint64_t* accf = &(wempty + 2 * NA + 2)->b;   // local: accumulator complete
  Bar16* wfull = wempty + 2 * NA + 3;   // [2][NW] local: W tile landed, set = group of the reader
  Bar16* wfree = wfull + 2 * NW;        // [NW] local: 8 transform warps done reading the W tile
  uint64_t* ff_empty = &(wfree + NW)->b;      // local (PERSIST): the tile's last recompute committed
  uint64_t* acc_empty = &(wfree + NW + 1)->b; // leader (PERSIST): 16 transform warps drained the accumulator
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wfree + NW + 2);

  const int warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  // grouped raster over (token tile, feature pair): GROUP_T token tiles x all
  // feature pairs per group, token tile fastest, so the ~74 clusters of a wave
  // read ~9 W panels and <= 8 activation panels and both stay L2-resident.
  // Tile n of this cluster: non-persistent = the cluster's own tile; persistent =
  // tiles cl, cl + n_cl, ... of the same raster (static schedule).
  //
  // Work units (persistent): the first n_tiles - tail tiles whole, then each of
  // the last `tail` tiles split into `split` k-ranges, so the last round of a
  // GEMM whose tile count is not a multiple of the co-resident clusters is
  // spread over idle clusters instead of leaving them waiting (a stream-K
  // style tail).  Split parts add fp32 partial accumulators through global
  // memory; the last part to finish writes the tile.
  const int nk = (Kred + BK - 1) / BK;
  const int cl = (int)(blockIdx.x >> 1), n_cl = (int)(gridDim.x >> 1);
  const int n_tiles = n_t * n_f;
  const int tail = (PERSIST && split > 1) ? (n_tiles > n_cl ? n_tiles % n_cl : n_tiles) : 0;
  const int n_full = n_tiles - tail;
  const int n_units = n_full + tail * split;
  const int my_units = PERSIST ? (n_units > cl ? (n_units - cl + n_cl - 1) / n_cl : 0) : 1;
  // unit n of this cluster: features m0, tokens l0, k-steps [kb, ke), tail tile index ut (-1 =
  // whole tile) and part
  auto unit = [&](int n, int& m0_, int& l0_, int& kb_, int& ke_, int& ut_, int& part_) {
    const int uid = PERSIST ? cl + n * n_cl : (int)blockIdx.y * n_f + cl;
    int cid = uid;
    ut_ = -1;
    part_ = 0;
    if (uid >= n_full) {
      ut_ = (uid - n_full) / split;
      part_ = (uid - n_full) - ut_ * split;
      cid = n_full + ut_;
    }
    const int per_group = GROUP_T * n_f;
    const int grp_ = cid / per_group, idx = cid % per_group;
    const int gt = min(GROUP_T, n_t - grp_ * GROUP_T);
    const int fp = idx / gt, tt = grp_ * GROUP_T + idx % gt;
    m0_ = fp * (2 * BM) + rank * BM;   // this CTA's features
    l0_ = tt * BNT;                    // the pair's tokens
    kb_ = ut_ < 0 ? 0 : part_ * nk / split;
    ke_ = ut_ < 0 ? nk : (part_ + 1) * nk / split;
  };
  int m0, l0, kb0, ke0, ut0, pt0;
  unit(0, m0, l0, kb0, ke0, ut0, pt0);
  // this CTA's rows of the two MMAs' B operands: tokens l0 + 128 rank .. +127
  // (N = 256 MMA) and l0 + 256 + (N2 / 2) rank .. (N = N2 MMA)

  if (warp == W_SF) {
    // lane-parallel barrier initialisation over the flat Bar16 array (layout above):
    // sready / afull count the merged arrivals in the leader, refree / wready and
    // acc_empty the 16 transform warps of the pair, wfree the 8 of the CTA, the rest one
    constexpr int NBARS = 2 * NS + 3 * NE + 2 * NACT + 3 * NA + 3 + 3 * NW + 2;
    constexpr int AFULL0 = 2 * NS + NE, WREADY0 = AFULL0 + NACT;
    for (int k = lane; k < NBARS; k += 32) {
      uint32_t cnt = 1;
      if (k < NS) cnt = leader ? 2u : 1u;                              // sready
      if (k >= 2 * NS && k < AFULL0) cnt = 16;                         // refree
      if (k >= AFULL0 && k < WREADY0) cnt = leader ? 2u : 1u;          // afull
      if (k >= WREADY0 && k < WREADY0 + NA) cnt = 16;                  // wready
      if (k >= NBARS - 2 - NW && k < NBARS - 2) cnt = 8;   // wfree
      if (k == NBARS - 1) cnt = 16;                       // acc_empty
      mbar_init(&bars[k].b, cnt);
    }
    fence_barrier_init();
    __syncwarp();
    // first use of every recompute buffer: nobody has read it yet
    if (leader && lane < NE) mbar_arrive_count(&refree[lane].b, 16);
    if (lane == 0) {
      tma_prefetch_desc(&tmAct);
      if (N2) tma_prefetch_desc(&tmAct2);
      tma_prefetch_desc(&tmW);
      tma_prefetch_desc(&tmS);
      tma_prefetch_desc(&tmF);
      tma_prefetch_desc(&tmOut);
      if (SP && meta24 != nullptr) tma_prefetch_desc(&tmMeta);
    }
  }
  if (warp == W_MMA) tmem_alloc_pair<TMEM_COLS>(tmem_slot);
  if (SP && threadIdx.x < 256) {
    // prmt selector keeping entries i0 < i1 of a group of four bf16 (index nibble i0 | i1 << 2)
    auto sel = [](uint32_t n) { return 0x1010u + (n & 3u) * 0x22u + (n >> 2) * 0x2200u; };
    sel_lut[threadIdx.x] = sel(threadIdx.x & 0xFu) | (sel(threadIdx.x >> 4) << 16);
  }
  tc_fence_before();
  // Local barrier only: the producers start their TMA loads (which complete on
  // this CTA's own barriers) at once; every role that touches the peer CTA
  // (remote arrives, pair MMAs, multicast commits) waits on the cluster
  // barrier first, so the peer's barrier initialisation overlaps the loads.
  __syncthreads();
  tc_fence_after();
  cluster_arrive();
  const uint32_t tmem = *tmem_slot;
  // Every TMA completes on a barrier of the CTA that issued it; the peer
  // relays its landings to the leader, and the transform warps of both CTAs
  // arrive on the leader's merged barriers.  Remote arrives go through mapa.
  const uint32_t sready_l = mapa_shared(smem_u32(sready), 0);
  const uint32_t refree_l = mapa_shared(smem_u32(refree), 0);
  const uint32_t afull_l = mapa_shared(smem_u32(afull), 0);
  const uint32_t wready_l = mapa_shared(smem_u32(wready), 0);
  const uint32_t pffull_l = mapa_shared(smem_u32(pffull), 0);
  const uint32_t acc_empty_l = mapa_shared(smem_u32(acc_empty), 0);

  if (warp == W_SF) {
    // ------------------------------------------------------------ factor-ring producer (both CTAs)
    if (lane == 0) {
      for (int n = 0, g = 0; n < my_units; ++n) {
      int kb, ke, ut, part;
      unit(n, m0, l0, kb, ke, ut, part);
      if (PERSIST && n > 0) mbar_wait(ff_empty, (n - 1) & 1);   // every recompute of the previous unit committed
      mbar_arrive_expect_tx(ffull, FF);
      if (DX) {  // b [r, C] as MN-major A of the recompute: two 64-wide atoms of this CTA's columns
        tma_load_2d(ffac, &tmF, ffull, m0, 0);
        tma_load_2d(ffac + FF / 2, &tmF, ffull, m0 + 64, 0);
      } else {   // a [R, r] K-major, this CTA's rows
        tma_load_2d(ffac, &tmF, ffull, 0, m0);
      }
      for (int i = kb; i < ke; ++i, ++g) {
        const int sl = g % NS;
        mbar_wait(&s_empty[sl].b, ((g / NS) & 1) ^ 1);
        uint8_t* st = sfr + sl * SF;
        const int k0 = i * BK;
        mbar_arrive_expect_tx(&sready[sl].b, SF);
        if (DX) tma_load_2d(st, &tmS, &sready[sl].b, 0, k0 + 32 * rank);   // a rows, K-major
        else tma_load_2d(st, &tmS, &sready[sl].b, k0 + 32 * rank, (m0 / grp_rows) * grp_r);  // b cols, MN-major
      }
      }
    } else if (lane == 1) {
      // ---------------------------------------------------------- W-ring producer (both CTAs), a
      // second lane of this warp: one fewer warp keeps the kernel at 12 warps, whose register
      // budget is 168 a thread instead of 128 at 13
      for (int n = 0, g = 0; n < my_units; ++n) {
      int kb, ke, ut, part;
      unit(n, m0, l0, kb, ke, ut, part);
      for (int i = kb; i < ke; ++i, ++g) {
        const int wi = g % NW;
        mbar_wait(&wfree[wi].b, ((g / NW) & 1) ^ 1);
        LORS_TR(8, g);
        uint8_t* st = wring + wi * W_BYTES;
        const int k0 = i * BK;
        uint64_t* wf = &wfull[(g % NGRP) * NW + wi].b;   // the set of the group that reads step g
        mbar_arrive_expect_tx(wf, W_BYTES + (SP && meta24 != nullptr ? meta_bytes<SP>() : 0u));
        // (a box's first byte must be 16-byte aligned: the box of k-steps 2j, 2j + 1)
        if (SP && meta24 != nullptr) tma_load_2d(mring + wi * meta_bytes<SP>(), &tmMeta, wf, (k0 / 8) & ~15, m0);
        if (DX) {  // W[k0:k0+64, m0:m0+128] as two SW128 boxes of 64 columns
          tma_load_2d(st, &tmW, wf, m0, k0);
          tma_load_2d(st + W_BYTES / 2, &tmW, wf, m0 + 64, k0);
        } else {   // W[m0:m0+128, k0:k0+64], SW128
          tma_load_2d(st, &tmW, wf, k0, m0);
        }
      }
      }
    }
    cluster_wait();
  } else if (warp == W_ACT) {
    // ------------------------------------------------------------ activation-ring producer (both CTAs)
    if (lane == 0 && !EX) {
      for (int n = 0, g = 0; n < my_units; ++n) {
      int kb, ke, ut, part;
      unit(n, m0, l0, kb, ke, ut, part);
      const int lh = l0 + rank * 128, lh2 = l0 + 256 + rank * (N2 / 2);
      for (int i = kb; i < ke; ++i, ++g) {
        const int a = g % NACT;
        mbar_wait(&a_empty[a].b, ((g / NACT) & 1) ^ 1);
        LORS_TR(7, g);
        mbar_arrive_expect_tx(&afull[a].b, ACT_BYTES);   // both halves' bytes
        tma_load_2d(actb + a * ACT_BYTES, &tmAct, &afull[a].b, i * BK, lh);
        if (N2) tma_load_2d(actb + a * ACT_BYTES + ACT1_BYTES, &tmAct2, &afull[a].b, i * BK, lh2);
      }
      }
    }
    cluster_wait();
  } else if (warp == W_RELAY) {
    cluster_wait();
    // ------------------------------------------------------------ activation relay (peer CTA)
    if (!leader && lane == 0 && !EX) {
      int total = 0;
      for (int n = 0; n < my_units; ++n) {
        int m_, l_, kb, ke, ut, part;
        unit(n, m_, l_, kb, ke, ut, part);
        total += ke - kb;
      }
      for (int g = 0; g < total; ++g) {
        const int a = g % NACT;
        mbar_wait(&afull[a].b, (g / NACT) & 1);
        mbar_arrive_cluster(afull_l + a * 16);
      }
    }
  } else if (warp == W_MMA) {
    cluster_wait();
    if (!leader) {
      // ---------------------------------------------------------- early relay (peer CTA)
      if (lane == 0) {
        for (int n = 0, g = 0; n < my_units; ++n) {
          int m_, l_, kb, ke, ut, part;
          unit(n, m_, l_, kb, ke, ut, part);
          mbar_wait(ffull, n & 1);
          mbar_arrive_cluster(pffull_l);
          for (int i = kb; i < ke; ++i, ++g) {
            const int sl = g % NS;
            mbar_wait(&sready[sl].b, (g / NS) & 1);
            mbar_arrive_cluster(sready_l + sl * 16);
          }
        }
      }
    } else {
      // ---------------------------------------------------------- MMA issuer (leader CTA, converged warp)
      constexpr uint32_t idesc_re = make_idesc_bf16(256, 64, DX, !DX);
      constexpr uint32_t idesc_main = make_idesc_bf16(256, 256, false, false);
      constexpr uint32_t idesc_n2 = make_idesc_bf16(256, N2 ? N2 : 256, false, false);
      constexpr uint32_t idesc_sp = make_idesc_bf16(256, 256, false, false, true);
      constexpr uint32_t idesc_sp_n2 = make_idesc_bf16(256, N2 ? N2 : 256, false, false, true);
      // descriptor bases; a descriptor's start-address field is addr >> 4, so
      // byte offsets inside shared memory are added as (offset >> 4)
      const uint64_t ff_desc = DX ? make_sdesc(smem_u32(ffac), FF / 2, 1024, SW_128)
                                  : make_sdesc(smem_u32(ffac), 16, 8 * SWR, sw_layout(SWR));
      const uint64_t sf_desc = DX ? make_sdesc(smem_u32(sfr), 16, 8 * SWR, sw_layout(SWR))
                                  : make_sdesc(smem_u32(sfr), 0, 8 * 64, SW_64);
      const uint64_t weff_desc = SP ? make_sdesc(smem_u32(weff), 16, 512, SW_64)    // compressed, 64 B rows
                                    : make_sdesc(smem_u32(weff), 16, 1024, SW_128);
      const uint64_t act_desc = make_sdesc(smem_u32(actb), 16, 1024, SW_128);
      constexpr uint32_t FF_KSTEP = DX ? 2048 >> 4 : 32 >> 4;   // per K16 of the recompute
      constexpr uint32_t SF_KSTEP = DX ? 32 >> 4 : 1024 >> 4;
      auto do_rec = [&](const int j, const int rk, const int rn, const int rlen) {
        if (rk == 0) {  // this tile's fixed factor, both CTAs
          mbar_wait(ffull, rn & 1);
          mbar_wait(pffull, rn & 1);
        }
        const int e = j % NE, sl = j % NS;
        LORS_TR(0, j);
        // factor slice of step j landed in both CTAs; recompute buffer e read by the transform of j - NE
        mbar_wait2(&sready[sl].b, (j / NS) & 1, &refree[e].b, (j / NE) & 1);
        LORS_TR(2, j);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t sfd = sf_desc + (uint64_t)(sl * (SF >> 4));
#pragma unroll
          for (int kk = 0; kk < RP / 16; ++kk)
            mma_bf16_pair(tmem + RE_COL + e * 64, ff_desc + kk * FF_KSTEP, sfd + kk * SF_KSTEP, idesc_re,
                          kk > 0 ? 1u : 0u);
          mma_commit_pair(&refull[(j % NGRP) * NE + e].b, 0x3);
          mma_commit_pair(&s_empty[sl].b, 0x3);
          if (PERSIST && rk == rlen - 1) mma_commit_pair(ff_empty, 0x3);   // fixed factor may be replaced
        }
        __syncwarp();
      };
      bool main_n2 = true;   // the second MMA's tokens (l0 + 256 ..) hold valid rows in this unit
      // the main MMAs of step jm (activation slot a, W_eff buffer wb) and the commits that free
      // both slots; called from the elected lane
      auto main_mmas = [&](const int jm, const int mk, const int a, const int wb) {
        const uint64_t ad = weff_desc + (uint64_t)(wb * (WEFF_BYTES >> 4));
        const uint64_t bd = act_desc + (uint64_t)(a * (ACT_BYTES >> 4));
        if (SP) {
          // two K = 32 sparse MMAs: compressed A advances 32 B, B 64 B, metadata one column each
#pragma unroll
          for (int hh = 0; hh < 2; ++hh)
            mma_bf16_pair_sp(tmem, ad + hh * 2, bd + hh * 4, tmem + E_COL + wb * 8 + hh * 4, idesc_sp,
                             (mk > 0 || hh > 0) ? 1u : 0u);
          if (N2 && main_n2) {  // tokens 256 .. 256 + N2 into the second accumulator, same A and metadata
            const uint64_t bd2 = bd + (ACT1_BYTES >> 4);
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
              mma_bf16_pair_sp(tmem + 256, ad + hh * 2, bd2 + hh * 4, tmem + E_COL + wb * 8 + hh * 4, idesc_sp_n2,
                               (mk > 0 || hh > 0) ? 1u : 0u);
          }
        } else {
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            mma_bf16_pair(tmem, ad + kk * 2, bd + kk * 2, idesc_main, (mk > 0 || kk > 0) ? 1u : 0u);
          if (N2 && main_n2) {  // tokens 256 .. 256 + N2 into the second accumulator
            const uint64_t bd2 = bd + (ACT1_BYTES >> 4);
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
              mma_bf16_pair(tmem + 256, ad + kk * 2, bd2 + kk * 2, idesc_n2, (mk > 0 || kk > 0) ? 1u : 0u);
          }
        }
        mma_commit_pair(&a_empty[a].b, 0x3);
        mma_commit_pair(&wempty[((jm + NA) % NGRP) * NA + wb].b, 0x3);   // next writer's group
      };
      auto do_main = [&](const int jm, const int mk, const int mn, const int mlen) {
        if (PERSIST && mk == 0 && mn > 0) {
          LORS_TR(20, mn);
          mbar_wait(acc_empty, (mn - 1) & 1);  // previous tile drained
          LORS_TR(21, mn);
        }
        if (N2 && mk == 0) {   // a ragged last token tile: skip the all-padding N2 MMA (a third of it)
          int m_, l_, kb_, ke_, ut_, pt_;
          unit(mn, m_, l_, kb_, ke_, ut_, pt_);
          main_n2 = l_ + 256 < n_tok;
        }
        const int a = jm % NACT, wb = jm % NA;
        LORS_TR(3, jm);
        // activation halves of both CTAs landed; W_eff tiles of both CTAs written
        mbar_wait2(&afull[a].b, (jm / NACT) & 1, &wready[wb].b, (jm / NA) & 1);
        LORS_TR(5, jm);
        tc_fence_after();
        if (elect_one()) {
          main_mmas(jm, mk, a, wb);
          if (mk == mlen - 1) mma_commit_pair(accf, 0x3);
        }
        __syncwarp();
        LORS_TR(6, jm);
      };
      // Flat schedule over this CTA pair's tiles: the recompute of step j runs D
      // steps ahead of its main MMA and into the next tile.  At a tile boundary
      // the previous tile's last main MMA goes first (the new tile's recompute
      // waits for its fixed factor); incremental counters, no division by nk.
      auto unit_len = [&](int n) {
        int m_, l_, kb, ke, ut, part;
        unit(n, m_, l_, kb, ke, ut, part);
        return ke - kb;
      };
      int total = 0;
      for (int n = 0; n < my_units; ++n) total += unit_len(n);
      int rk = 0, rn = 0, mk = 0, mn = 0;
      int rlen = my_units > 0 ? unit_len(0) : 1, mlen = rlen;
      for (int j = 0; j < total + (EX ? 0 : D); ++j) {
        const bool has_rec = j < total, has_main = !EX && j >= D;
        // the first D steps of a tile: the previous tile's main MMA goes first (its accumulator
        // must be complete before the transform warps, after their epilogue, release the
        // recompute buffers of the new tile; and the new tile's first recompute waits for its
        // fixed factor)
        const bool flip = has_rec && rk < D && j > 0;
        if (has_rec && has_main && rk >= D && mk != 0) {
          // steady state (no tile boundary on either side): all four barriers of rec(j) and
          // main(j - D) probed at once, then both issued from one elected lane -- each barrier
          // probe costs ~100 cycles and each elect / __syncwarp region ~150, and this loop paces
          // the pipeline (tools/trace_k1.py: 1570 -> ~1030 cycles a k-step at cfg3)
          const int jm = j - D, e = j % NE, sl = j % NS, a = jm % NACT, wb = jm % NA;
          LORS_TR(0, j);
#ifdef LORS_TRACE
          // which barrier the issue loop waits for: one at a time, in the order they usually complete
          mbar_wait(&wready[wb].b, (jm / NA) & 1);
          LORS_TR(1, jm);
          mbar_wait(&afull[a].b, (jm / NACT) & 1);
          LORS_TR(2, jm);
          mbar_wait(&sready[sl].b, (j / NS) & 1);
          LORS_TR(4, jm);
          mbar_wait(&refree[e].b, (j / NE) & 1);
#else
          mbar_wait4(&sready[sl].b, (j / NS) & 1, &refree[e].b, (j / NE) & 1, &afull[a].b, (jm / NACT) & 1,
                     &wready[wb].b, (jm / NA) & 1);
#endif
          LORS_TR(5, jm);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t sfd = sf_desc + (uint64_t)(sl * (SF >> 4));
#pragma unroll
            for (int kk = 0; kk < RP / 16; ++kk)
              mma_bf16_pair(tmem + RE_COL + e * 64, ff_desc + kk * FF_KSTEP, sfd + kk * SF_KSTEP, idesc_re,
                            kk > 0 ? 1u : 0u);
            mma_commit_pair(&refull[(j % NGRP) * NE + e].b, 0x3);
            mma_commit_pair(&s_empty[sl].b, 0x3);
            if (PERSIST && rk == rlen - 1) mma_commit_pair(ff_empty, 0x3);   // fixed factor may be replaced
            main_mmas(jm, mk, a, wb);
            if (mk == mlen - 1) mma_commit_pair(accf, 0x3);
          }
          __syncwarp();
          LORS_TR(6, jm);
          if (++rk == rlen) { rk = 0; if (++rn < my_units) rlen = unit_len(rn); }
          if (++mk == mlen) { mk = 0; if (++mn < my_units) mlen = unit_len(mn); }
          continue;
        }
        if (flip && has_main) {
          do_main(j - D, mk, mn, mlen);
          if (++mk == mlen) { mk = 0; if (++mn < my_units) mlen = unit_len(mn); }
        }
        if (has_rec) {
          do_rec(j, rk, rn, rlen);
          if (++rk == rlen) { rk = 0; if (++rn < my_units) rlen = unit_len(rn); }
        }
        if (!flip && has_main) {
          do_main(j - D, mk, mn, mlen);
          if (++mk == mlen) { mk = 0; if (++mn < my_units) mlen = unit_len(mn); }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ transform warps 0..7
    cluster_wait();
    const int q = warp & 3;        // TMEM lane quarter
    const int h = (warp >> 2) & 1; // column half of the 64-wide k-step
    const int grp = warp >> 3;     // group: k-step parity this warp transforms (SP), else 0
    const int t = q * 32 + lane;   // feature row inside the tile (TMEM lane)
    int gm = m0 + t;               // global output feature (per tile)
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    const WeffAlpha walpha = weff_alpha(alpha);      // weff_pair's alpha operands
    // Per k-step: the TMEM load of the rank-r product (load_p), the W loads (load_w),
    // release of the recompute buffer, then transform and store (finish).  (Issuing the
    // next step's TMEM load at the end of a step measured 0-2% slower, tools/ab_gemm.py.)
    auto load_p = [&](const int i, uint32_t (&p)[32]) {
      const int rb = i % NE;
      if (warp == 0 && lane == 0) LORS_TR(9, i);
      mbar_wait(&refull[(i % NGRP) * NE + rb].b, (i / RE_PERIOD) & 1);
      if (warp == 0 && lane == 0) LORS_TR(10, i);
      tc_fence_after();
      const uint32_t re_col = RE_COL + rb * 64 + h * 32;
      if (!DX) {
        tmem_ld_x32(tmem + lane_addr + re_col, p);
      } else {  // fragment layout matching ldmatrix.trans, two 16-lane groups
        uint32_t (&p0)[16] = *reinterpret_cast<uint32_t(*)[16]>(&p[0]);
        uint32_t (&p1)[16] = *reinterpret_cast<uint32_t(*)[16]>(&p[16]);
        tmem_ld_16x256b_x4(tmem + lane_addr + re_col, p0);
        tmem_ld_16x256b_x4(tmem + lane_addr + (16u << 16) + re_col, p1);
      }
    };
    auto load_w = [&](const int i, const int kq, uint32_t (&wv)[16], uint32_t& mw) {
      // W tile landed: all of this thread's W loads are issued before any result is
      // needed, so their latency overlaps the TMEM load's
      const int wi = i % NW;
      mbar_wait(&wfull[(i % NGRP) * NW + wi].b, (i / W_PERIOD) & 1);
      if (warp == 0 && lane == 0) LORS_TR(11, i);
      const uint32_t wt = smem_u32(wring + wi * W_BYTES);
      // 2:4 with precomputed metadata: this row's 8 index nibbles of the half, from the
      // slot's meta24 box (lors_compress_24 layout [R, C/8]; rows past R were zero-filled)
      if (SP && meta24 != nullptr) {
        mw = lds32(smem_u32(mring + wi * meta_bytes<SP>()) + (uint32_t)t * 16 + (kq & 1) * 8 + h * 4);
        if (gm >= Mout) mw = 0x44444444u;   // rows past R: zero-filled box -> a valid (unused) pattern
      }
      if (!DX) {
        // thread = W row t; chunks 4h .. 4h+3 of 8 k-values (SW128)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          lds128(wt + (uint32_t)t * 128 + ((((uint32_t)h * 4 + c) ^ ((uint32_t)t & 7)) << 4),
                 *reinterpret_cast<uint32_t(*)[4]>(&wv[4 * c]));
      } else {
        // W tile [64 k][128 c] as two SW128 boxes of 64 c; ldmatrix.trans
        const int mi = lane >> 3, rr = lane & 7;
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
          for (int jp = 0; jp < 2; ++jp) {
            const int sa = mi & 1, ja = 2 * jp + (mi >> 1);
            const uint32_t k = h * 32 + 8 * ja + rr;
            const uint32_t c = q * 32 + 16 * g + 8 * sa;
            ldsm_x4_trans(wt + (c >> 6) * 8192 + k * 128 + ((((c & 63) >> 3) ^ (k & 7)) << 4),
                          *reinterpret_cast<uint32_t(*)[4]>(&wv[4 * (2 * g + jp)]));
          }
      }
    };
    auto release = [&](const int i) {
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(refree_l + (i % NE) * 16);  // RE buffer free for step i + NE
      if (warp == 0 && lane == 0) LORS_TR(22, i);
    };
    // hold_w: keep the W slot (no wfree arrival): the epilogue stages its output blocks there
    auto finish = [&](const int i, const int kq, uint32_t (&p)[32], uint32_t (&wv)[16], uint32_t mw,
                      const bool hold_w = false) {
      constexpr bool POW2 = P2;
      const int wb = i % NA, wi = i % NW;
      // 3. destination buffer drained by the MMA of step i - NA
      // waits for the commit of main(i - NA), the previous user of this buffer
      if (!EX && i >= NA) mbar_wait(&wempty[(i % NGRP) * NA + wb].b, ((i - NA) / A_PERIOD) & 1);
      if (warp == 0 && lane == 0) LORS_TR(12, i);
      const uint32_t dst = smem_u32(weff + wb * WEFF_BYTES);
      if (SP && meta24 != nullptr) {
        // 2:4 with precomputed index nibbles: the kept pair of each group of four is
        // selected first (one prmt on W, one on the rounded product, the selectors from
        // sel_lut), then weff_combine runs once per pair -- W_eff is elementwise, so this
        // is the dense prologue's value at the kept positions, compressed
        uint32_t comp[8];
#pragma unroll
        for (int g2 = 0; g2 < 4; ++g2) {
          const uint32_t sels = lds32_table(smem_u32(sel_lut) + ((mw >> (8 * g2)) & 0xFFu) * 4);
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int g = 2 * g2 + e;
            const uint32_t sel = e ? (sels >> 16) : sels;
            const uint32_t w2 = prmt(wv[2 * g], wv[2 * g + 1], sel);
            const uint32_t s2 = prmt(weff_scaled_p<POW2>(__uint_as_float(p[4 * g]), __uint_as_float(p[4 * g + 1]), walpha),
                                     weff_scaled_p<POW2>(__uint_as_float(p[4 * g + 2]), __uint_as_float(p[4 * g + 3]), walpha),
                                     sel);
            comp[g] = weff_combine<POW2>(w2, s2, walpha, nonzero_mask_bf16x2(w2));
          }
        }
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const uint32_t off = (uint32_t)t * 64 + (((uint32_t)(2 * h + cc) ^ (((uint32_t)t >> 1) & 3u)) << 4);
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(dst + off), "r"(comp[4 * cc]),
                       "r"(comp[4 * cc + 1]), "r"(comp[4 * cc + 2]), "r"(comp[4 * cc + 3])
                       : "memory");
        }
        const uint32_t pm = __shfl_xor_sync(0xffffffffu, mw, 8);
        const uint32_t word = (lane & 8) ? ((pm >> 16) | (mw & 0xFFFF0000u)) : ((mw & 0xFFFFu) | (pm << 16));
        tmem_st_x1(tmem + lane_addr + E_COL + wb * 8 + h * 4, word);
        tmem_st_wait();
        tc_fence_before();
      } else if (!DX) {
        // thread = W row; 4 chunks of 8 k-values, same swizzled position in and out
        uint32_t mword = 0;
        uint32_t comp[8], meta = 0;  // 2:4: compressed pairs and index nibbles of this half
        if (BITS) mword = (gm < Mout) ? __ldg(bits + (int64_t)gm * words_per_row + ((kq * BK + h * 32) >> 5)) : 0u;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t off = (uint32_t)t * 128 + ((((uint32_t)h * 4 + c) ^ ((uint32_t)t & 7)) << 4);
          uint32_t o[4], keepm[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t w2 = wv[4 * c + u];
            const uint32_t keep = BITS ? bits2_to_mask((mword >> (c * 8 + 2 * u)) & 3u) : nonzero_mask_bf16x2(w2);
            keepm[u] = keep;
            o[u] = weff_pair<POW2>(w2, __uint_as_float(p[c * 8 + 2 * u]), __uint_as_float(p[c * 8 + 2 * u + 1]), walpha,
                             keep);
          }
          if (SP) {
            // compress each group of 4 to its two kept values (select on the mask,
            // so padded slots of sparser groups carry +0) and a 4-bit index nibble
#pragma unroll
            for (int gi = 0; gi < 2; ++gi) {
              const uint32_t k0 = keepm[2 * gi], k1 = keepm[2 * gi + 1];
              const uint32_t m = (k0 & 1u) | ((k0 >> 15) & 2u) | ((k1 & 1u) << 2) | ((k1 >> 13) & 8u);
              const uint32_t nib = (uint32_t)(kNibbleLut >> (4 * m)) & 0xFu;
              const uint32_t sel = 0x1010u + (nib & 3u) * 0x22u + (nib >> 2) * 0x2200u;
              comp[c * 2 + gi] = prmt(o[2 * gi], o[2 * gi + 1], sel);
              meta |= nib << (4 * (c * 2 + gi));
            }
          } else {
            asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(dst + off), "r"(o[0]), "r"(o[1]), "r"(o[2]),
                         "r"(o[3])
                         : "memory");
          }
        }
        if (SP) {
          // compressed K-major SW64 tile: row t, bytes [32h, 32h + 32)
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const uint32_t off = (uint32_t)t * 64 + (((uint32_t)(2 * h + cc) ^ (((uint32_t)t >> 1) & 3u)) << 4);
            asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(dst + off), "r"(comp[4 * cc]),
                         "r"(comp[4 * cc + 1]), "r"(comp[4 * cc + 2]), "r"(comp[4 * cc + 3])
                         : "memory");
          }
          // metadata in the tcgen05 sparse layout: lane L = a + 8b + 16c holds, for the
          // MMA's k-half b, rows (L & ~8) in bits 0-15 and (L | 8) in bits 16-31
          const uint32_t pm = __shfl_xor_sync(0xffffffffu, meta, 8);
          const uint32_t word = (lane & 8) ? ((pm >> 16) | (meta & 0xFFFF0000u)) : ((meta & 0xFFFFu) | (pm << 16));
          tmem_st_x1(tmem + lane_addr + E_COL + wb * 8 + h * 4, word);
          tmem_st_wait();
          tc_fence_before();
        }
      } else {
        // ldmatrix.trans handed thread l the pair (k = 32h + 8j + 2(l%4) + {0,1},
        // c = 32q + 16g + 8s + l/4), the positions p[16g + 4j + 2s + {0,1}] hold;
        // results go to the K-major W_eff^T tile (row c) as 32-bit pairs.
        uint32_t bword[8];
        if (BITS) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e2 = 0; e2 < 2; ++e2) {
              const int64_t kr = (int64_t)kq * BK + h * 32 + 8 * j + 2 * (lane & 3) + e2;
              bword[j * 2 + e2] = kr < Kred ? __ldg(bits + kr * words_per_row + ((m0 + q * 32) >> 5)) : 0u;
            }
        }
#pragma unroll
        for (int g = 0; g < 2; ++g) {
#pragma unroll
          for (int jp = 0; jp < 2; ++jp) {
            const uint32_t* wq = &wv[4 * (2 * g + jp)];
            uint32_t o4[4];
#pragma unroll
            for (int mm = 0; mm < 4; ++mm) {
              const int sm = mm & 1, j = 2 * jp + (mm >> 1);
              const uint32_t ct = q * 32 + 16 * g + 8 * sm + (lane >> 2);   // k = 32h + 8j + 2(lane % 4)
              uint32_t keep;
              if (BITS) {
                const uint32_t cb = ct & 31;
                keep = bits2_to_mask(((bword[j * 2] >> cb) & 1u) | (((bword[j * 2 + 1] >> cb) & 1u) << 1));
              } else {
                keep = nonzero_mask_bf16x2(wq[mm]);
              }
              const uint32_t o = weff_pair<POW2>(wq[mm], __uint_as_float(p[16 * g + 4 * j + 2 * sm]),
                                           __uint_as_float(p[16 * g + 4 * j + 2 * sm + 1]), walpha, keep);
              o4[mm] = o;   // W_eff^T(ct, k .. k + 1): row lane / 4, column pair lane % 4 of 8x8 block mm
            }
            {  // one stmatrix per four blocks: matrix mm = lane / 8 (rows ct .. ct + 7 of the K-major
               // W_eff^T tile, 16-byte k chunk 4h + j), this lane's row address lane % 8
              const int mi = lane >> 3;
              const uint32_t ct = q * 32 + 16 * g + 8 * (mi & 1) + (lane & 7);
              const uint32_t chunk = 4 * h + 2 * jp + (mi >> 1);
              stsm_x4(dst + ct * 128 + ((chunk ^ (ct & 7)) << 4), o4[0], o4[1], o4[2], o4[3]);
            }
          }
        }
      }
      if (warp == 0 && lane == 0) LORS_TR(23, i);
      fence_proxy_async_smem();
      __syncwarp();
      if (EX) {
        // export: the whole [128 rows][64 k] SW128 tile is the TMA box of W_eff at
        // (k0, m0); the store has read the buffer before anyone rewrites it
        named_bar_sync(1, XFORM_THREADS);
        if (warp == 0 && lane == 0) {
          tma_store_2d(&tmOut, weff + wb * WEFF_BYTES, kq * BK, m0);
          tma_store_commit();
          tma_store_wait_all();
        }
        named_bar_sync(1, XFORM_THREADS);
        if (lane == 0) mbar_arrive(&wfree[wi].b);
        return;
      }
      if (lane == 0) {
        if (!hold_w) mbar_arrive(&wfree[wi].b);      // done reading the W tile
        mbar_arrive_cluster(wready_l + wb * 16);     // W_eff half ready for the pair MMA
        if (warp == 0) LORS_TR(13, i);
        if (warp == 3) LORS_TR(14, i);   // arrival skew across the transform warps
        if (warp == 5) LORS_TR(15, i);
        if (warp == 7) LORS_TR(16, i);
      }
    };
    // Accumulator -> bf16 -> transposed staging: the accumulator is read in the MMA
    // fragment layout (tcgen05.ld.16x256b: a thread holds two adjacent tokens of a
    // feature), rounded to bf16 pairs (+bias) and written by stmatrix.trans into a
    // [128 tokens][64 features] SW128 block (bank-conflict free).  Warp (q, hh):
    // features 32q .. 32q+31 (feature half q >> 1), tokens hh*TSL .. of chunk c.
    constexpr int TSL = 128 / (XW / 4);              // tokens of a chunk per warp (64 or 32)
    const int hh = warp >> 2;
    // split-K partials: fragment f = (chunk, 32-token slice, 16-lane group) of this thread,
    // 16 floats at ((f * XFORM_THREADS + tid) * 16) of the part's slot -- coalesced, and
    // read back by the same thread of the CTA that finishes the tile
    constexpr int NCH = nch<SP>(), OUT_ROWS = out_rows<SP>();
    constexpr int PSLOT = 128 * 128 * NCH;           // floats per CTA and part
    const int tid_x = (int)threadIdx.x;
    auto frag_off = [&](int c, int tb, int g16) {
      return ((int64_t)((c * (TSL / 32) + tb / 32) * 2 + g16) * XFORM_THREADS + tid_x) * 16;
    };
    auto stage_chunk = [&](const int c, uint8_t* blk, const float (&bvals)[2][2], const float* const* adds,
                           const int n_adds) {
#pragma unroll 1
      for (int tb = 0; tb < TSL; tb += 32) {
        const int tok = hh * TSL + tb;                // token offset inside the chunk
        if (c * 128 + tok >= BNT) continue;           // past a partial last chunk
        uint32_t v[2][16];
#pragma unroll
        for (int g16 = 0; g16 < 2; ++g16)
          tmem_ld_16x256b_x4(tmem + ((uint32_t)(q * 32 + 16 * g16) << 16) + (uint32_t)(c * 128 + tok), v[g16]);
        tmem_ld_wait();
        // a split tile: the sum of all its parts' partials in part order (run-to-run
        // deterministic whichever part finished last), replacing the accumulator
        // (two parts: all 16 loads issued before the first add, one L2 round trip)
        if (n_adds == 2) {
          float4 x0[2][4], x1[2][4];
#pragma unroll
          for (int g16 = 0; g16 < 2; ++g16)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              x0[g16][u] = __ldcg(reinterpret_cast<const float4*>(adds[0] + frag_off(c, tb, g16)) + u);
              x1[g16][u] = __ldcg(reinterpret_cast<const float4*>(adds[1] + frag_off(c, tb, g16)) + u);
            }
#pragma unroll
          for (int g16 = 0; g16 < 2; ++g16)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              v[g16][4 * u] = __float_as_uint(x0[g16][u].x + x1[g16][u].x);
              v[g16][4 * u + 1] = __float_as_uint(x0[g16][u].y + x1[g16][u].y);
              v[g16][4 * u + 2] = __float_as_uint(x0[g16][u].z + x1[g16][u].z);
              v[g16][4 * u + 3] = __float_as_uint(x0[g16][u].w + x1[g16][u].w);
            }
        }
#pragma unroll
        for (int g16 = 0; g16 < 2; ++g16) {
          const int F = q * 32 + 16 * g16;
#pragma unroll
          for (int bp = 0; bp < 2; ++bp) {           // token blocks 2bp, 2bp+1 (8 tokens each)
            uint32_t m[4];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int bb = 2 * bp + u;
              m[2 * u] = pack_bf16x2(__uint_as_float(v[g16][4 * bb]) + bvals[g16][0],
                                     __uint_as_float(v[g16][4 * bb + 1]) + bvals[g16][0]);
              m[2 * u + 1] = pack_bf16x2(__uint_as_float(v[g16][4 * bb + 2]) + bvals[g16][1],
                                         __uint_as_float(v[g16][4 * bb + 3]) + bvals[g16][1]);
            }
            // matrix mi = lane / 8: token block 2bp + (mi >> 1), feature block F + 8 (mi & 1);
            // this lane addresses stored row (token) lane % 8 of it
            const int mi = lane >> 3, tr = tok + 8 * (2 * bp + (mi >> 1)) + (lane & 7);
            const int fu = ((F & 63) >> 3) + (mi & 1);   // 16-byte unit of the 128-byte row
            stsm_x4_trans(smem_u32(blk + tr * 128 + ((fu ^ (tr & 7)) << 4)), m[0], m[1], m[2], m[3]);
          }
        }
      }
    };
    auto bias_of = [&](float (&bvals)[2][2], const int m0) {   // bias of features (16 g + l/4) and (+8)
#pragma unroll
      for (int g16 = 0; g16 < 2; ++g16)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int f = m0 + q * 32 + 16 * g16 + 8 * e + (lane >> 2);
          bvals[g16][e] = (!DX && bias != nullptr && f < Mout) ? __bfloat162float(bias[f]) : 0.f;
        }
    };
    if constexpr (PERSIST) {
      // Per unit n: its remaining k-steps; then (when unit n + 1 has >= 3 k-steps) the first three
      // k-steps of unit n + 1, whose W_eff buffers free up as unit n's last main MMAs complete and
      // whose W slots, read and held, stage unit n's epilogue; then the epilogue.  The MMAs of unit
      // n + 1 restart the moment the accumulator is handed back (tools/trace_k1.py: transforming
      // after the epilogue left the tensor pipe idle ~5000 cycles a tile on top of the drain).
      __shared__ int last_flag;
      constexpr int PRE = 3;
      int g = 0, pre = 0, kb = 0, ke = 0, ut = -1, part = 0;
      if (my_units > 0) unit(0, m0, l0, kb, ke, ut, part);
      auto step = [&](const int kq, const bool hold_w) {
        uint32_t p[32], wv[16], mw = 0;
        load_p(g, p);
        load_w(g, kq, wv, mw);
        release(g);
        finish(g, kq, p, wv, mw, hold_w);
        ++g;
      };
      for (int n = 0; n < my_units; ++n) {
        gm = m0 + t;
        for (int kq = kb + pre; kq < ke; ++kq) step(kq, false);
        const int em0 = m0, el0 = l0, eut = ut, epart = part;   // this unit, for its epilogue
        int stage_g = -1;       // flat step of the first held W slot (-1: stage in the W_eff ring)
        pre = 0;
        if (n + 1 < my_units) {
          unit(n + 1, m0, l0, kb, ke, ut, part);
          if (!EX && ke - kb >= PRE) {
            gm = m0 + t;
            stage_g = g;
            pre = PRE;
            for (int i = 0; i < PRE; ++i) step(kb + i, true);
          }
        }
        if (EX) continue;   // no accumulator
        // staging block b of the epilogue: a held W slot, or the (then idle) W_eff ring
        auto stage_buf = [&](const int b) {
          return stage_g >= 0 ? wring + ((stage_g + b % 3) % NW) * W_BYTES : weff + (b % 3) * WEFF_BYTES;
        };
        if (stage_g >= 0) named_bar_sync(1, XFORM_THREADS);   // every warp done reading the held W tiles
        // -------------------------------------------------------- epilogue of unit n
        if (warp == 0 && lane == 0) LORS_TR(17, n);
        mbar_wait(accf, n & 1);
        if (warp == 0 && lane == 0) LORS_TR(18, n);
        tc_fence_after();
        const float* adds[2];
        int n_adds = 0;
        if (eut >= 0) {
          // part of a split tile: publish this part's fp32 accumulator, then the last
          // part to arrive (per CTA of the pair) adds the others and writes the tile
          float* mine = partials + ((int64_t)(eut * split + epart) * 2 + rank) * PSLOT;
#pragma unroll 1
          for (int c = 0; c < NCH; ++c)
#pragma unroll 1
            for (int tb = 0; tb < TSL; tb += 32) {
              uint32_t v[2][16];
              const int tok = hh * TSL + tb;
              if (c * 128 + tok >= BNT) continue;         // past a partial last chunk
#pragma unroll
              for (int g16 = 0; g16 < 2; ++g16)
                tmem_ld_16x256b_x4(tmem + ((uint32_t)(q * 32 + 16 * g16) << 16) + (uint32_t)(c * 128 + tok), v[g16]);
              tmem_ld_wait();
#pragma unroll
              for (int g16 = 0; g16 < 2; ++g16) {
                float4* dst = reinterpret_cast<float4*>(mine + frag_off(c, tb, g16));
#pragma unroll
                for (int u = 0; u < 4; ++u)
                  __stcg(dst + u, make_float4(__uint_as_float(v[g16][4 * u]), __uint_as_float(v[g16][4 * u + 1]),
                                              __uint_as_float(v[g16][4 * u + 2]), __uint_as_float(v[g16][4 * u + 3])));
              }
            }
          __threadfence();
          named_bar_sync(1, XFORM_THREADS);
          if (threadIdx.x == 0) {
            const unsigned int old = atomicAdd(&counters[eut * 2 + rank], 1u);
            last_flag = old == (unsigned int)(split - 1);
            if (last_flag) counters[eut * 2 + rank] = 0u;   // reusable without a memset
          }
          named_bar_sync(1, XFORM_THREADS);
          if (!last_flag) {                                  // done: hand the accumulator back
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(acc_empty_l);
            if (stage_g >= 0 && lane == 0)             // the held W slots were not needed
              for (int k = 0; k < PRE; ++k) mbar_arrive(&wfree[(stage_g + k) % NW].b);
            continue;
          }
          __threadfence();
          for (int p2 = 0; p2 < split; ++p2) adds[n_adds++] = partials + ((int64_t)(eut * split + p2) * 2 + rank) * PSLOT;
        }
        // Staged through three 16 KB buffers (held W slots or the W_eff ring): six
        // [128 tokens][64 features] blocks in two batches of three; the accumulator is handed
        // back to the MMA issuer after the last TMEM read.
        float bvals[2][2];
        bias_of(bvals, em0);
#pragma unroll 1
        for (int batch = 0; batch < 2; ++batch) {
#pragma unroll 1
          for (int c = 0; c < NCH; ++c) {
            const int b = 2 * c + (q >> 1);            // block (chunk c, feature half q >> 1)
            if (b / 3 == batch) stage_chunk(c, stage_buf(b), bvals, adds, n_adds);
          }
          if (batch == 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(acc_empty_l);
            if (warp == 0 && lane == 0) LORS_TR(19, n);
          }
          fence_proxy_async_smem();
          named_bar_sync(1, XFORM_THREADS);
          if (warp == 0 && lane == 0) {
            for (int b = 3 * batch; b < 3 * batch + 3; ++b)
              for (int rr = 0; rr < 128 && (b >> 1) * 128 + rr < BNT; rr += OUT_ROWS)
                store_out(stage_buf(b) + rr * 128, em0 + 64 * (b & 1), el0 + 128 * (b >> 1) + rr);
            tma_store_commit();
            tma_store_wait_all();                      // the blocks are rewritten next
          }
          named_bar_sync(1, XFORM_THREADS);
        }
        if (stage_g >= 0 && lane == 0)                 // the stores have read the held W slots
          for (int k = 0; k < PRE; ++k) mbar_arrive(&wfree[(stage_g + k) % NW].b);
      }
      if (EX && warp == 0 && lane == 0) tma_store_wait_done();
    } else {
    for (int i = grp; i < nk; i += NGRP) {
      uint32_t p[32], wv[16], mw = 0;
      load_p(i, p);
      load_w(i, i, wv, mw);
      release(i);
      finish(i, i, p, wv, mw);
    }
    // ------------------------------------------------------------ epilogue
    mbar_wait(accf, 0);
    tc_fence_after();
    // Per 128-token chunk: the accumulator is read in the MMA fragment layout
    // (tcgen05.ld.16x256b: a thread holds two adjacent tokens of a feature),
    // rounded to bf16 pairs and written transposed by stmatrix.trans into
    // [token][64 features] SW128 blocks (one 16 KB block per chunk and feature
    // half, bank-conflict free); the chunk's two TMA stores are issued while the
    // next chunk is staged.  Warp (q, hh): features 32q .. 32q+31, tokens hh*64 ..
    // of each chunk (XW / 4 token slices of 128 / (XW / 4)).
    uint8_t* stg = smem;
    constexpr int TSL = 128 / (XW / 4);              // tokens of a chunk per warp (64 or 32)
    const int hh = warp >> 2;
    float bvals[2][2];                               // bias of features (16 g + l/4) and (+8)
#pragma unroll
    for (int g16 = 0; g16 < 2; ++g16)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int f = m0 + q * 32 + 16 * g16 + 8 * e + (lane >> 2);
        bvals[g16][e] = (!DX && bias != nullptr && f < Mout) ? __bfloat162float(bias[f]) : 0.f;
      }
#pragma unroll 1
    for (int c = 0; c < BNT / 128; ++c) {
#pragma unroll 1
      for (int tb = 0; tb < TSL; tb += 32) {
        const int tok = hh * TSL + tb;                // token offset inside the chunk
        uint32_t v[2][16];
#pragma unroll
        for (int g16 = 0; g16 < 2; ++g16)
          tmem_ld_16x256b_x4(tmem + ((uint32_t)(q * 32 + 16 * g16) << 16) + (uint32_t)(c * 128 + tok), v[g16]);
        tmem_ld_wait();
#pragma unroll
        for (int g16 = 0; g16 < 2; ++g16) {
          // features F = 32q + 16 g16 (+8 for the second row block); 64-feature half of the staging
          const int F = q * 32 + 16 * g16, fh = F >> 6;
          uint8_t* blk = stg + (size_t)((c * 2 + fh) * 16384);
#pragma unroll
          for (int bp = 0; bp < 2; ++bp) {           // token blocks 2bp, 2bp+1 (8 tokens each)
            uint32_t m[4];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int bb = 2 * bp + u;
              m[2 * u] = pack_bf16x2(__uint_as_float(v[g16][4 * bb]) + bvals[g16][0],
                                     __uint_as_float(v[g16][4 * bb + 1]) + bvals[g16][0]);
              m[2 * u + 1] = pack_bf16x2(__uint_as_float(v[g16][4 * bb + 2]) + bvals[g16][1],
                                         __uint_as_float(v[g16][4 * bb + 3]) + bvals[g16][1]);
            }
            // matrix mi = lane / 8: token block 2bp + (mi >> 1), feature block F + 8 (mi & 1);
            // this lane addresses stored row (token) lane % 8 of it
            const int mi = lane >> 3, tr = tok + 8 * (2 * bp + (mi >> 1)) + (lane & 7);
            const int fu = ((F & 63) >> 3) + (mi & 1);   // 16-byte unit of the 128-byte row
            stsm_x4_trans(smem_u32(blk + tr * 128 + ((fu ^ (tr & 7)) << 4)), m[0], m[1], m[2], m[3]);
          }
        }
      }
      fence_proxy_async_smem();
      named_bar_sync(1, XFORM_THREADS);
      if (warp == 0 && lane == 0) {
        store_out(stg + (c * 2) * 16384, m0, l0 + 128 * c);
        store_out(stg + (c * 2 + 1) * 16384, m0 + 64, l0 + 128 * c);
        tma_store_commit();
      }
    }
    if (warp == 0 && lane == 0) {
      tma_store_wait_all();
    }
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == W_MMA) tmem_dealloc_pair<TMEM_COLS>(tmem);
}

// Co-resident clusters of the persistent kernel (cached per kernel once it is known;
// 74 while no device answers, e.g. a workspace query on a host without a GPU).
template <bool DX, int RP, bool SP>
static int persistent_clusters() {
  using namespace rg;
  static int max_clusters = 0;
  if (max_clusters > 0) return max_clusters;
  auto kern = tc_lors_gemm_kernel<DX, RP, false, SP>;
  const size_t smem = smem_bytes<RP, SP>();
  int v = 0;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * (unsigned)(num_sms() / 2));
    cfg.blockDim = dim3(threads<SP>());
    cfg.dynamicSmemBytes = smem;
    if (cudaOccupancyMaxActiveClusters(&v, (void*)kern, &cfg) != cudaSuccess) v = 0;
  }
  (void)cudaGetLastError();
  if (v <= 0) return 74;
  max_clusters = v;
  return v;
}

// Tail split of the persistent walk: the n_tiles % clusters tiles of the last wave
// are cut along K into `split` units (parts), so that the last wave is as long as
// a part instead of a tile.  Parts publish fp32 partials; the last to finish adds.
struct TailSplit {
  int split = 1, tail = 0, clusters = 0;
  size_t bytes = 0;        // workspace: tail * 2 counters, then tail * split * 2 partial slots
  size_t counter_bytes = 0;
};

template <bool DX, int RP, bool SP>
static TailSplit plan_tail_split(int L, int R, int C) {
  using namespace rg;
  TailSplit p;
  if (!persist<SP>() || getenv("LORS_NO_TAIL_SPLIT")) return p;
  constexpr int BNT = bnt<SP>();
  const int Mout = DX ? C : R, Kred = DX ? R : C;
  const int n_tiles = (int)(ceil_div(Mout, 2 * BM) * ceil_div(L, BNT)), nk = (int)ceil_div(Kred, BK);
  const int mc = persistent_clusters<DX, RP, SP>();
  p.clusters = mc;
  const int tail = n_tiles > mc ? n_tiles % mc : n_tiles;
  if (tail == 0 || 2 * tail > mc) return p;
  // two parts when the tail fits twice and each part keeps enough k-steps to cover
  // its fixed cost (partials out, the last part's reads, the extra epilogue, and the
  // power the idle tail would have left to the busy SMs): measured a loss with 32
  // k-steps per part (K = 4096) and +6..14% with >= 86 (K >= 11008), tools/exp_split.py;
  // LORS_SPLIT_MIN_KSTEPS for experiments
  static const int min_ksteps = getenv("LORS_SPLIT_MIN_KSTEPS") ? atoi(getenv("LORS_SPLIT_MIN_KSTEPS")) : 64;
  const int split = (2 * tail <= mc && nk >= 2 * min_ksteps) ? 2 : 1;
  if (split < 2) return p;
  p.split = split;
  p.tail = tail;
  p.counter_bytes = ((size_t)tail * 2 * sizeof(unsigned int) + 255) / 256 * 256;
  p.bytes = p.counter_bytes + (size_t)tail * split * 2 * 128 * 128 * nch<SP>() * sizeof(float);
  return p;
}

template <bool DX, int RP, bool SP>
static int launch_lors_gemm(const bf16* act, const bf16* w, const bf16* a, const bf16* b, const bf16* bias,
                            const uint32_t* bits, const uint8_t* meta24, bf16* out, int L, int R, int C, int r,
                            float alpha, cudaStream_t s, void* ws, size_t ws_bytes, int groups = 1) {
  using namespace rg;
  // groups > 1 (forward only): R rows per projection, W / a / b / out of the G projections consecutive
  const int G = DX ? 1 : groups, Rt = R * G;
  const int Mout = DX ? C : Rt, Kred = DX ? R : C;
  constexpr int N2 = n2<SP>(), BNT = bnt<SP>();
  CUtensorMap tAct, tAct2, tW, tS, tF, tOut;
  int st;
  if ((st = make_map(&tAct, act, Kred, L, 64, 128, 128, "activation"))) return st;
  if ((st = make_map(&tAct2, act, Kred, L, 64, N2 ? N2 / 2 : 128, 128, "activation (second MMA)"))) return st;
  if (DX) st = make_map(&tW, w, C, R, 64, 64, 128, "W (dX)");
  else st = make_map(&tW, w, C, Rt, 64, 128, 128, "W (fwd)");
  if (st) return st;
  if (DX) {
    if ((st = make_map(&tS, a, r, R, RP, 32, RP * 2, "a (streamed half)"))) return st;
    if ((st = make_map(&tF, b, C, r, 64, RP, 128, "b (fixed)"))) return st;
  } else {
    if ((st = make_map(&tS, b, C, (uint64_t)r * G, 32, RP, 64, "b (streamed half)"))) return st;
    if ((st = make_map(&tF, a, r, Rt, RP, 128, RP * 2, "a (fixed)"))) return st;
  }
  if (G > 1) st = make_map_3d(&tOut, out, R, L, G, 64, out_rows<SP>(), 128, "grouped output");
  else st = make_map(&tOut, out, Mout, L, 64, out_rows<SP>(), 128, "output");  // [tokens][64 features] SW128
  if (st) return st;
  // 2:4 metadata boxes ([R, C/8] bytes, 128 rows x 16 bytes): a TMA row pitch is a multiple of
  // 16 bytes, so C % 128 == 0; other widths derive the nibbles on chip from W instead
  CUtensorMap tMeta = tW;
  if (SP && meta24 != nullptr) {
    if (C % 128 == 0) {
      if ((st = make_map_u8(&tMeta, meta24, (uint64_t)C / 8, R, 16, 128, "meta24"))) return st;
    } else {
      meta24 = nullptr;
    }
  }
  const bool p2 = alpha_pow2(alpha);
  auto kern = bits ? (p2 ? tc_lors_gemm_kernel<DX, RP, true, SP, false, true> : tc_lors_gemm_kernel<DX, RP, true, SP, false, false>)
                   : (p2 ? tc_lors_gemm_kernel<DX, RP, false, SP, false, true> : tc_lors_gemm_kernel<DX, RP, false, SP, false, false>);
  const size_t smem = smem_bytes<RP, SP>();
  LORS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                "lors_gemm smem attribute");
  const int n_f = (int)ceil_div(Mout, 2 * BM), n_t = (int)ceil_div(L, BNT);
  dim3 grid((unsigned)(2 * n_f), (unsigned)n_t);
  int split = 1;
  float* partials = nullptr;
  unsigned int* counters = nullptr;
  if (persist<SP>()) {  // one CTA pair per co-resident cluster slot, tiles walked in the raster order
    const int mc = persistent_clusters<DX, RP, SP>();
    int units = n_f * n_t;
    const TailSplit ts = plan_tail_split<DX, RP, SP>(L, Rt, C);
    if (ts.split > 1 && ts.clusters == mc && ws != nullptr && ws_bytes >= ts.bytes) {
      split = ts.split;
      counters = (unsigned int*)ws;
      partials = (float*)((char*)ws + ts.counter_bytes);
      units += ts.tail * (split - 1);
      LORS_CUDA_TRY(cudaMemsetAsync(counters, 0, ts.counter_bytes, s), "zero tail-split counters");
    }
    grid = dim3((unsigned)(2 * std::min(units, mc)));
  }
  if (getenv("LORS_VERBOSE")) {  // diagnostics: how many clusters of this kernel fit on the GPU at once
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(threads<SP>());
    cfg.dynamicSmemBytes = smem_bytes<RP, SP>();
    int v = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&v, (void*)kern, &cfg);
    fprintf(stderr, "[lors] tc_lors_gemm<dx=%d,r=%d,sp=%d>: grid %u x %u, max active clusters %d (%s)\n", (int)DX,
            RP, (int)SP, grid.x, grid.y, v, cudaGetErrorString(e));
    (void)cudaGetLastError();
  }
  kern<<<grid, threads<SP>(), smem, s>>>(tAct, tAct2, tW, tS, tF, tOut, tMeta, bias, bits, SP ? meta24 : nullptr,
                                         (int)ceil_div(C, 32), Mout, Kred, n_t, n_f, split, partials, counters,
                                         alpha, L, DX ? Mout : R, G > 1 ? r : 0);
  LORS_CHECK_LAUNCH(DX ? "tc_lors_gemm<dx>" : "tc_lors_gemm<fwd>");
  return LORS_OK;
}

template <bool DX, bool SP = false>
static int lors_gemm(int rp, const bf16* act, const bf16* w, const bf16* a, const bf16* b, const bf16* bias,
                     const uint32_t* bits, bf16* out, int L, int R, int C, int r, float alpha, cudaStream_t s,
                     void* ws, size_t ws_bytes, const uint8_t* meta24 = nullptr, int groups = 1) {
  switch (rp) {
    case 16:
      return launch_lors_gemm<DX, 16, SP>(act, w, a, b, bias, bits, meta24, out, L, R, C, r, alpha, s, ws, ws_bytes,
                                          groups);
    case 32:
      return launch_lors_gemm<DX, 32, SP>(act, w, a, b, bias, bits, meta24, out, L, R, C, r, alpha, s, ws, ws_bytes,
                                          groups);
    default:
      return launch_lors_gemm<DX, 64, SP>(act, w, a, b, bias, bits, meta24, out, L, R, C, r, alpha, s, ws, ws_bytes,
                                          groups);
  }
}

// K6 on the tensor-core path (merged_weight / merge, adapters.py:214-224, 709-727):
// the forward kernel's own prologue -- the same rank-r recompute MMA and the same
// weff_pair -- with each W_eff tile TMA-stored to out [R, C] instead of multiplied,
// so the exported weight is bit-identical to the one the forward and dX GEMMs use.
template <int RP>
static int launch_weff_export(const bf16* w, const bf16* a, const bf16* b, const uint32_t* bits, bf16* out, int R,
                              int C, int r, float alpha, cudaStream_t s) {
  using namespace rg;
  CUtensorMap tW, tS, tF, tOut;
  int st;
  if ((st = make_map(&tW, w, C, R, 64, 128, 128, "W (export)"))) return st;
  if ((st = make_map(&tS, b, C, r, 32, RP, 64, "b (streamed half)"))) return st;
  if ((st = make_map(&tF, a, r, R, RP, 128, RP * 2, "a (fixed)"))) return st;
  if ((st = make_map(&tOut, out, C, R, 64, 128, 128, "W_eff out"))) return st;   // [128 rows][64 k] SW128
  const bool p2 = alpha_pow2(alpha);
  auto kern = bits ? (p2 ? tc_lors_gemm_kernel<false, RP, true, false, true, true> : tc_lors_gemm_kernel<false, RP, true, false, true, false>)
                   : (p2 ? tc_lors_gemm_kernel<false, RP, false, false, true, true> : tc_lors_gemm_kernel<false, RP, false, false, true, false>);
  const size_t smem = smem_bytes<RP, false>();
  LORS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                "weff export smem attribute");
  const int n_f = (int)ceil_div(R, 2 * BM);
  const int mc = persistent_clusters<false, RP, false>();
  dim3 grid((unsigned)(2 * std::min(n_f, mc)));
  // the activation maps are never read in export mode (W's map stands in)
  kern<<<grid, threads<false>(), smem, s>>>(tW, tW, tW, tS, tF, tOut, tW, nullptr, bits, nullptr, (int)ceil_div(C, 32), R,
                                            C, /*n_t=*/1, n_f, /*split=*/1, nullptr, nullptr, alpha, 0, R, 0);
  LORS_CHECK_LAUNCH("tc_lors_gemm<export>");
  return LORS_OK;
}

int tc_effective_weight(const bf16* w, const uint32_t* bits, const bf16* a, const bf16* b, bf16* out, int R, int C,
                        int r, float alpha, cudaStream_t s) {
  if (!tc_shape_ok(R, C, r)) return effective_weight<bf16>(w, bits, a, b, out, R, C, r, alpha, s);  // = the FFMA path's
  switch (pad_rank(r)) {
    case 16: return launch_weff_export<16>(w, a, b, bits, out, R, C, r, alpha, s);
    case 32: return launch_weff_export<32>(w, a, b, bits, out, R, C, r, alpha, s);
    default: return launch_weff_export<64>(w, a, b, bits, out, R, C, r, alpha, s);
  }
}

// workspace of one lors_gemm (the tail split's counters and partials; 0 without a split)
template <bool DX>
static size_t lors_gemm_workspace(int rp, int L, int R, int C) {
  switch (rp) {
    case 16: return plan_tail_split<DX, 16, false>(L, R, C).bytes;
    case 32: return plan_tail_split<DX, 32, false>(L, R, C).bytes;
    default: return plan_tail_split<DX, 64, false>(L, R, C).bytes;
  }
}

// ===========================================================================
// K5: masked-G fused adapter gradient (north_star 3; oracle _sqft_grads,
// adapters.py:303-312): G = (dY^T X) . M is accumulated in TMEM, masked in
// registers and contracted in place -- G never reaches HBM.  On CTA pairs, the G mainloop as
// tcgen05 cta_group::2 MMAs (M = 256 rows of R over the pair, each CTA staging
// its 128 dY columns and half of the 256 X columns: 32 KB per SM per k-step
// instead of 48), and the two small contractions as warp-level mma.sync on
// each CTA's own masked rows:
//   dA[own 128 R x r]   = (G.M)_own [128 x 256 C] . b^T[256 C x r]
//   dB^T[256 C x r]    += (G.M)_own^T [256 C x 128 R] . a[own 128 R x r]
// so no CTA needs its peer's G.M; both partials leave through TMA reduce-adds.
// warps: 0 TMA producer, 1 MMA issuer (leader) / TMA relay (peer), 2..5 mask,
// contract, reduce.
// ===========================================================================
namespace mgp {
constexpr int BK = 64, STAGES = 4, THREADS = 192;
constexpr uint32_t A_BYTES = 128 * BK * 2;      // 16 KB  dY_t [64 tokens][128 R]  (2 MN atoms)
constexpr uint32_t B_BYTES = 128 * BK * 2;      // 16 KB  X_t  [64 tokens][128 C]  (this CTA's half of N)
constexpr uint32_t PIPE = STAGES * (A_BYTES + B_BYTES);   // 128 KB, reused after the mainloop:
constexpr uint32_t GM_OFF = 0, DA_OFF = 65536, DB_OFF = 98304;   // G.M 64 KB, dA 32 KB, dB 64 KB (+32 KB past PIPE)
constexpr uint32_t EXTRA = 32768;
template <int RP>
constexpr uint32_t bt_bytes() { return RP * 256 * 2; }   // b [RP rows][256 C], 4 SW128 atoms of [RP][64]
template <int RP>
constexpr uint32_t at_bytes() { return 128 * RP * 2; }   // a [128 R][RP], swizzle span RP * 2
template <int RP>
constexpr size_t smem_bytes() { return 1024 + PIPE + EXTRA + bt_bytes<RP>() + at_bytes<RP>() + 256; }
}  // namespace mgp

template <int RP, bool BITS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(mgp::THREADS, 1)
    tc_masked_grad_pair_kernel(const __grid_constant__ CUtensorMap tmDY, const __grid_constant__ CUtensorMap tmX,
                               const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmA,
                               const __grid_constant__ CUtensorMap tmDAo, const __grid_constant__ CUtensorMap tmDBo,
                               const bf16* __restrict__ w, const uint32_t* __restrict__ bits, int words_per_row,
                               int L, int R, int C, float alpha, int det, int r_pad) {
  using namespace mgp;
  constexpr uint32_t BT = bt_bytes<RP>(), AT = at_bytes<RP>();
  constexpr uint32_t SWA = RP * 2;              // a tile swizzle span (bytes)
  constexpr int NT = RP / 8;                    // n8 tiles of the contractions
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                            // [STAGES] dY tiles
  uint8_t* sB = sA + STAGES * A_BYTES;           // [STAGES] X half tiles
  uint8_t* sBt = smem + PIPE + EXTRA;            // b tile
  uint8_t* sAt = sBt + BT;                       // a tile (own rows)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sAt + AT);
  uint64_t* full = bars;                         // [STAGES] (leader: own producer + peer relay)
  uint64_t* empty = full + STAGES;               // [STAGES] (leader's commit, multicast)
  uint64_t* gfull = empty + STAGES;              // G accumulated (multicast)
  uint64_t* abfull = gfull + 1;                  // a / b tiles landed (own)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(abfull + 1);

  const int warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int m0 = (int)blockIdx.z * 256 + (int)rank * 128;   // this CTA's R rows
  const int c0 = (int)blockIdx.y * 256;                       // the pair's C columns
  const int nk = (L + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], leader ? 2 : 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(gfull, 1);
    mbar_init(abfull, 1);
    fence_barrier_init();
    tma_prefetch_desc(&tmDY);
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmA);
  }
  if (warp == 1) tmem_alloc_pair<256>(tmem_slot);
  tc_fence_before();
  cluster_sync();                                // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t full_l = mapa_shared(smem_u32(full), 0);

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(abfull, BT + AT);
      for (int q = 0; q < 4; ++q) tma_load_2d(sBt + q * (RP * 128), &tmB, abfull, c0 + 64 * q, 0);
      tma_load_2d(sAt, &tmA, abfull, 0, m0);
      for (int i = 0; i < nk; ++i) {
        const int s = i % STAGES;
        mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], A_BYTES + B_BYTES);
        const int l0 = i * BK;
        uint8_t* a = sA + s * A_BYTES;
        uint8_t* b = sB + s * B_BYTES;
        tma_load_2d(a, &tmDY, &full[s], m0, l0);
        tma_load_2d(a + A_BYTES / 2, &tmDY, &full[s], m0 + 64, l0);
        tma_load_2d(b, &tmX, &full[s], c0 + 128 * (int)rank, l0);
        tma_load_2d(b + B_BYTES / 2, &tmX, &full[s], c0 + 128 * (int)rank + 64, l0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      if (!leader) {
        // relay: this CTA's tiles landed -> one arrival on the leader's barrier
        for (int i = 0; i < nk; ++i) {
          const int s = i % STAGES;
          mbar_wait(&full[s], (i / STAGES) & 1);
          mbar_arrive_cluster(full_l + s * 8);
        }
      } else {
        constexpr uint32_t idesc_g = make_idesc_bf16(256, 256, true, true);
        for (int i = 0; i < nk; ++i) {
          const int s = i % STAGES;
          mbar_wait(&full[s], (i / STAGES) & 1);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + s * A_BYTES), b_base = smem_u32(sB + s * B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            mma_bf16_pair(tmem, make_sdesc(a_base + kk * 2048, A_BYTES / 2, 1024, SW_128),
                          make_sdesc(b_base + kk * 2048, B_BYTES / 2, 1024, SW_128), idesc_g,
                          (i > 0 || kk > 0) ? 1u : 0u);
          mma_commit_pair(&empty[s], 0x3);
        }
        mma_commit_pair(gfull, 0x3);
      }
    }
  } else {
    const int q = warp & 3, ew = warp - 2;       // TMEM lane quarter; epilogue warp 0..3
    const int t = q * 32 + lane;                 // G row (TMEM lane) inside this CTA's tile
    const int gm_row = m0 + t;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    // keep bits of this row's 256 columns, gathered while the mainloop runs
    uint32_t keep[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t keepw = 0;
      const int gc = c0 + 32 * j;
      if (gm_row < R) {
        if (BITS) {
          if (gc < C) {
            keepw = __ldg(bits + (int64_t)gm_row * words_per_row + (gc >> 5));
            if (gc + 32 > C) keepw &= (1u << (C - gc)) - 1u;
          }
        } else {
          const bf16* wr = w + (int64_t)gm_row * C + gc;
#pragma unroll
          for (int u = 0; u < 32; u += 8) {
            if (gc + u + 8 <= C) {
              const uint4 raw = __ldg(reinterpret_cast<const uint4*>(wr + u));
              const uint32_t ww[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const uint32_t nz = nonzero_mask_bf16x2(ww[e]);
                keepw |= ((nz & 1u) | ((nz >> 15) & 2u)) << (u + 2 * e);
              }
            }
          }
        }
      }
      keep[j] = keepw;
    }
    mbar_wait(gfull, 0);
    tc_fence_after();
    // 1. mask G into bf16 G.M: 4 K-major SW128 atoms [128 R][64 C] at GM_OFF
    const uint32_t gmb = smem_u32(smem + GM_OFF);
#pragma unroll
    for (int cb = 0; cb < 256; cb += 32) {
      uint32_t v[32];
      tmem_ld_x32(tmem + lane_addr + cb, v);
      tmem_ld_wait();
      const uint32_t keepw = keep[cb / 32];
      uint32_t pk[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const float g0 = ((keepw >> (2 * e)) & 1u) ? __uint_as_float(v[2 * e]) : 0.0f;
        const float g1 = ((keepw >> (2 * e + 1)) & 1u) ? __uint_as_float(v[2 * e + 1]) : 0.0f;
        pk[e] = pack_bf16x2(g0, g1);
      }
      const uint32_t atom = gmb + (cb >> 6) * 16384 + t * 128;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const uint32_t chunk = ((((cb & 63) >> 3) + cc) ^ (t & 7)) << 4;
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(atom + chunk), "r"(pk[4 * cc]),
                     "r"(pk[4 * cc + 1]), "r"(pk[4 * cc + 2]), "r"(pk[4 * cc + 3])
                     : "memory");
      }
    }
    mbar_wait(abfull, 0);
    named_bar_sync(1, 128);                      // every row of G.M parked
    const int g = lane >> 2, qd = lane & 3;
    const uint32_t bt = smem_u32(sBt), at = smem_u32(sAt);
    // 2. dA rows 32 ew .. +31 (two m16 tiles), K = 256 C
    {
      float acc[2][NT][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[mt][nt][e] = 0.f;
#pragma unroll 4
      for (int ks = 0; ks < 16; ++ks) {
        uint32_t af[2][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const int row = 32 * ew + 16 * mt + (lane & 7) + 8 * ((lane >> 3) & 1);
          const int k = 16 * ks + 8 * (lane >> 4);
          ldsm_x4(gmb + (k >> 6) * 16384 + row * 128 + ((((k & 63) >> 3) ^ (row & 7)) << 4), af[mt]);
        }
#pragma unroll
        for (int np = 0; np < NT / 2; ++np) {
          uint32_t bf[4];
          const int n = 16 * np + (lane & 7) + 8 * (lane >> 4);
          const int k = 16 * ks + 8 * ((lane >> 3) & 1);
          ldsm_x4(bt + (k >> 6) * (RP * 128) + n * 128 + ((((k & 63) >> 3) ^ (n & 7)) << 4), bf);
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            mma_16816(acc[mt][2 * np], af[mt], bf[0], bf[1]);
            mma_16816(acc[mt][2 * np + 1], af[mt], bf[2], bf[3]);
          }
        }
      }
      // stage alpha dA into SW128 boxes [128 rows][32 floats] (box = column / 32)
      uint8_t* st = smem + DA_OFF;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int hr = 0; hr < 2; ++hr) {
            const int row = 32 * ew + 16 * mt + g + 8 * hr, n = 8 * nt + 2 * qd;
            const int chunk = (n & 31) >> 2;
            *reinterpret_cast<float2*>(st + (n >> 5) * 16384 + row * 128 + ((chunk ^ (row & 7)) << 4) + (n & 3) * 4) =
                make_float2(alpha * acc[mt][nt][2 * hr], alpha * acc[mt][nt][2 * hr + 1]);
          }
    }
    // 3. dB^T rows (C) 64 ew .. +63 in two halves of 32, K = 128 own R rows
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      float acc[2][NT][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[mt][nt][e] = 0.f;
#pragma unroll 2
      for (int ks = 0; ks < 8; ++ks) {
        uint32_t af[2][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const int j = lane >> 3;               // matrix: (k 0-7 | 8-15) x (m 0-7 | 8-15)
          const int k = 16 * ks + (lane & 7) + 8 * (j >> 1);
          const int m = 64 * ew + 32 * h + 16 * mt + 8 * (j & 1);
          ldsm_x4_trans(gmb + (m >> 6) * 16384 + k * 128 + ((((m & 63) >> 3) ^ (k & 7)) << 4), af[mt]);
        }
#pragma unroll
        for (int np = 0; np < NT / 2; ++np) {
          uint32_t bf[4];
          const int j = lane >> 3;
          const int k = 16 * ks + (lane & 7) + 8 * (j & 1);
          const int n = 16 * np + 8 * (j >> 1);
          const uint32_t off = (uint32_t)(k * SWA + n * 2);
          ldsm_x4_trans(at + (off ^ (((off >> 7) & (SWA / 16 - 1)) << 4)), bf);
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            mma_16816(acc[mt][2 * np], af[mt], bf[0], bf[1]);
            mma_16816(acc[mt][2 * np + 1], af[mt], bf[2], bf[3]);
          }
        }
      }
      // stage alpha dB^T into [RP rows][128 C] plain boxes per C half (dB is [r, C])
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int hr = 0; hr < 2; ++hr) {
            const int c = 64 * ew + 32 * h + 16 * mt + g + 8 * hr, n = 8 * nt + 2 * qd;
            float* rows = reinterpret_cast<float*>(smem + DB_OFF + (c >> 7) * (RP * 512));
            rows[n * 128 + (c & 127)] = alpha * acc[mt][nt][2 * hr];
            rows[(n + 1) * 128 + (c & 127)] = alpha * acc[mt][nt][2 * hr + 1];
          }
    }
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    if (ew == 0 && lane == 0) {
      if (det) {
        // deterministic: this CTA's partials to their own slabs (dA: slab of the C tile,
        // dB: slab of the 128-row R tile), summed in slab order by slab_sum_kernel
        const int da_row = (int)blockIdx.y * r_pad + m0, db_row = ((int)blockIdx.z * 2 + (int)rank) * RP;
        for (int hf = 0; hf * 32 < RP; ++hf) tma_store_2d(&tmDAo, smem + DA_OFF + hf * 16384, 32 * hf, da_row);
        for (int hc = 0; hc < 2; ++hc) tma_store_2d(&tmDBo, smem + DB_OFF + hc * RP * 512, c0 + 128 * hc, db_row);
      } else {
        for (int hf = 0; hf * 32 < RP; ++hf) tma_reduce_add_2d(&tmDAo, smem + DA_OFF + hf * 16384, 32 * hf, m0);
        for (int hc = 0; hc < 2; ++hc) tma_reduce_add_2d(&tmDBo, smem + DB_OFF + hc * RP * 512, c0 + 128 * hc, 0);
      }
      tma_store_commit();
      tma_store_wait_done();
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) tmem_dealloc_pair<256>(tmem);
}

// out[i] = sum over s in order of part[s * slab + i]  (deterministic slab reduction)
__global__ void slab_sum_kernel(const float* __restrict__ part, int n_slabs, int64_t slab, float* __restrict__ out,
                                int64_t n_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_out) return;
  float acc = 0.f;
  for (int k = 0; k < n_slabs; ++k) acc += part[k * slab + i];
  out[i] = acc;
}

// deterministic masked-G partial slabs: dA [C tiles][R padded to 256][r], dB [128-row R tiles][RP][C]
static size_t masked_grad_det_bytes(int R, int C, int rp) {
  const size_t r_pad = (size_t)ceil_div(R, 256) * 256;
  return (size_t)ceil_div(C, 256) * r_pad * rp * sizeof(float) + 256 +
         (size_t)ceil_div(R, 256) * 2 * rp * (size_t)C * sizeof(float);
}

template <int RP>
static int launch_masked_grad_pair(const bf16* dy, const bf16* x, const bf16* w, const uint32_t* bits, const bf16* a,
                                   const bf16* b, float* da, float* db, int L, int R, int C, int r, float alpha,
                                   cudaStream_t s, float* det_ws = nullptr) {
  using namespace mgp;
  CUtensorMap tDY, tX, tB, tA, tDAo, tDBo;
  int st;
  if ((st = make_map(&tDY, dy, R, L, 64, 64, 128, "dY (MN)"))) return st;
  if ((st = make_map(&tX, x, C, L, 64, 64, 128, "X (MN)"))) return st;
  if ((st = make_map(&tB, b, C, r, 64, RP, 128, "b tile (K-major, K = C)"))) return st;
  if ((st = make_map(&tA, a, r, R, RP, 128, RP * 2, "a tile"))) return st;
  const int n_ct = (int)ceil_div(C, 256), n_rt2 = (int)ceil_div(R, 256) * 2, r_pad = (int)ceil_div(R, 256) * 256;
  float* da_part = det_ws;
  float* db_part = det_ws ? (float*)((char*)det_ws + ((size_t)n_ct * r_pad * r * sizeof(float) + 255) / 256 * 256)
                          : nullptr;
  if (det_ws) {
    if ((st = make_map(&tDAo, da_part, r, (uint64_t)n_ct * r_pad, 32, 128, 128, "dA partial slabs", true))) return st;
    if ((st = make_map(&tDBo, db_part, C, (uint64_t)n_rt2 * RP, 128, RP, 0, "dB partial slabs", true))) return st;
  } else {
    if ((st = make_map(&tDAo, da, r, R, 32, 128, 128, "dA fp32 (masked-G)", true))) return st;
    if ((st = make_map(&tDBo, db, C, r, 128, RP, 0, "dB fp32 (masked-G)", true))) return st;
    LORS_CUDA_TRY(cudaMemsetAsync(da, 0, sizeof(float) * (size_t)R * r, s), "zero dA");
    LORS_CUDA_TRY(cudaMemsetAsync(db, 0, sizeof(float) * (size_t)r * C, s), "zero dB");
  }
  auto kern = bits ? tc_masked_grad_pair_kernel<RP, true> : tc_masked_grad_pair_kernel<RP, false>;
  const size_t smem = smem_bytes<RP>();
  LORS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                "masked_grad_pair smem attribute");
  dim3 grid(2, (unsigned)n_ct, (unsigned)ceil_div(R, 256));
  kern<<<grid, THREADS, smem, s>>>(tDY, tX, tB, tA, tDAo, tDBo, w, bits, (int)ceil_div(C, 32), L, R, C, alpha,
                                   det_ws ? 1 : 0, r_pad);
  LORS_CHECK_LAUNCH("tc_masked_grad_pair");
  if (det_ws) {
    const int64_t na = (int64_t)R * r, nb = (int64_t)r * C;
    slab_sum_kernel<<<(unsigned)ceil_div(na, 256), 256, 0, s>>>(da_part, n_ct, (int64_t)r_pad * r, da, na);
    LORS_CHECK_LAUNCH("slab_sum dA");
    slab_sum_kernel<<<(unsigned)ceil_div(nb, 256), 256, 0, s>>>(db_part, n_rt2, (int64_t)RP * C, db, nb);
    LORS_CHECK_LAUNCH("slab_sum dB");
  }
  return LORS_OK;
}

static int masked_grad_tc(int rp, const bf16* dy, const bf16* x, const bf16* w, const uint32_t* bits, const bf16* a,
                          const bf16* b, float* da, float* db, int L, int R, int C, int r, float alpha,
                          cudaStream_t s, float* det_ws) {
  switch (rp) {
    case 16: return launch_masked_grad_pair<16>(dy, x, w, bits, a, b, da, db, L, R, C, r, alpha, s, det_ws);
    case 32: return launch_masked_grad_pair<32>(dy, x, w, bits, a, b, da, db, L, R, C, r, alpha, s, det_ws);
    default: return launch_masked_grad_pair<64>(dy, x, w, bits, a, b, da, db, L, R, C, r, alpha, s, det_ws);
  }
}

// ===========================================================================
// dispatch
// ===========================================================================
bool tc_shape_ok(int64_t R, int64_t C, int64_t r) {
  return R % 8 == 0 && C % 8 == 0 && r % 8 == 0 && r <= 64;
}

// the forward's tail-split workspace (0 when the walk has no tail to split)
size_t tc_fwd_workspace(const lors_fwd_args* a) {
  if (a->dtype != LORS_DTYPE_BF16 || (a->flags & (LORS_FLAG_SPARSE24 | LORS_FLAG_NO_TAIL_SPLIT)) || a->L <= 0 ||
      !tc_shape_ok(a->R, a->C, a->r))
    return 0;
  return lors_gemm_workspace<false>((int)pad_rank(a->r), (int)a->L, (int)a->R, (int)a->C);
}
static size_t dx_workspace(const lors_bwd_args* a) {
  if (a->dtype != LORS_DTYPE_BF16 || (a->flags & (LORS_FLAG_NO_DX | LORS_FLAG_NO_TAIL_SPLIT)) || a->L <= 0 ||
      !tc_shape_ok(a->R, a->C, a->r))
    return 0;
  return lors_gemm_workspace<true>((int)pad_rank(a->r), (int)a->L, (int)a->R, (int)a->C);
}
static size_t rank_slot(const lors_bwd_args* a) {
  return ((size_t)a->L * (size_t)a->r * sizeof(float) + 255) / 256 * 256;
}
// the region after the capi's two bf16 P / Q slots: P / Q's fp32 split-K accumulators, or
// (LORS_FLAG_DETERMINISTIC) the partial slabs of the ordered reductions
static size_t rank_r_region(const lors_bwd_args* a) {
  const size_t slot = rank_slot(a);
  if (!(a->flags & LORS_FLAG_DETERMINISTIC) || a->dtype != LORS_DTYPE_BF16 || a->L <= 0 ||
      !tc_shape_ok(a->R, a->C, a->r))
    return 2 * slot;
  const int L = (int)a->L, R = (int)a->R, C = (int)a->C, rp = (int)pad_rank((int)a->r);
  size_t need = 0;
  if (a->grad_mode == LORS_GRAD_MASKED) {
    need = masked_grad_det_bytes(R, C, rp);
  } else {
    for (size_t v : {skinny_partial_bytes(L, C, rp), skinny_partial_bytes(L, R, rp), skinny_partial_bytes(R, L, rp),
                     skinny_partial_bytes(C, L, rp)})
      need = std::max(need, v);
  }
  return (need + 255) / 256 * 256;
}
// DX_ONLY: the dX GEMM's tail split alone; otherwise, beyond the capi's two bf16
// P / Q slots: the rank-r region, then the dX tail split
size_t tc_bwd_workspace(const lors_bwd_args* a) {
  if (a->flags & LORS_FLAG_DX_ONLY) return dx_workspace(a);
  return rank_r_region(a) + dx_workspace(a);
}

int tc_fwd(const lors_fwd_args* A, cudaStream_t s) {
  const int L = (int)A->L, R = (int)A->R, C = (int)A->C, r = (int)A->r;
  const uint32_t* bits = A->mask_mode == LORS_MASK_BITS ? A->mask_bits : nullptr;
  const bf16 *x = (const bf16*)A->x, *w = (const bf16*)A->w, *a = (const bf16*)A->a, *b = (const bf16*)A->b;
  int st;
  if (!tc_shape_ok(R, C, r)) {  // FFMA kernels for shapes TMA cannot address
    st = simt_lors_gemm<bf16>(false, x, w, bits, a, b, (const bf16*)A->bias, (bf16*)A->y, L, R, C, r, A->alpha, s);
    if (st) return st;
    if (A->flags & LORS_FLAG_EMIT_P)
      st = simt_strided_gemm<bf16, bf16, bf16>(x, C, 1, b, C, 1, (bf16*)A->p, r, 1, L, r, C, 1.0f, false, s);
    return st;
  }
  const int rp = (int)pad_rank(r);
  if (A->flags & LORS_FLAG_SPARSE24) {
    if (C % 64 != 0) {
      set_error("2:4 sparse forward needs C % 64 == 0");
      return LORS_ERR_SHAPE;
    }
    st = lors_gemm<false, true>(rp, x, w, a, b, (const bf16*)A->bias, bits, (bf16*)A->y, L, R, C, r, A->alpha, s,
                                nullptr, 0, A->meta24);
  } else {
    const bool split = !(A->flags & LORS_FLAG_NO_TAIL_SPLIT);
    st = lors_gemm<false>(rp, x, w, a, b, (const bf16*)A->bias, bits, (bf16*)A->y, L, R, C, r, A->alpha, s,
                          split ? A->workspace : nullptr, split ? A->workspace_bytes : 0);
  }
  if (st) return st;
  if (A->flags & LORS_FLAG_EMIT_P)  // P = X_t b^T: A = X_t K-major, B = b [r, C] K-major
    st = skinny<false, false, 0>(rp, x, b, A->p, L, r, C, r, 1.0f, false, s);
  return st;
}

// Grouped forward: G projections of one input X as ONE persistent launch over their G * R / 256
// pair tiles (the tiles of all projections share the rounds, instead of each projection's
// partial last round).  Same per-tile arithmetic as tc_fwd, so every Y_g is bit-identical to
// its own lors_fwd.  Shapes: tc_fwd_group_ok.
bool tc_fwd_group_ok(const lors_fwd_args* A, int groups) {
  return groups >= 1 && A->dtype == LORS_DTYPE_BF16 && A->mask_mode == LORS_MASK_FROM_W && A->bias == nullptr &&
         !(A->flags & (LORS_FLAG_SPARSE24 | LORS_FLAG_EMIT_P)) && tc_shape_ok(A->R, A->C, A->r) &&
         A->R % 256 == 0 && pad_rank((int)A->r) == A->r;
}
size_t tc_fwd_group_workspace(const lors_fwd_args* A, int groups) {
  if (A->L <= 0 || !tc_fwd_group_ok(A, groups) || (A->flags & LORS_FLAG_NO_TAIL_SPLIT)) return 0;
  return lors_gemm_workspace<false>((int)A->r, (int)A->L, (int)(A->R * groups), (int)A->C);
}
int tc_fwd_group(const lors_fwd_args* A, int groups, cudaStream_t s) {
  const int L = (int)A->L, R = (int)A->R, C = (int)A->C, r = (int)A->r;
  const bool split = !(A->flags & LORS_FLAG_NO_TAIL_SPLIT);
  return lors_gemm<false>(r, (const bf16*)A->x, (const bf16*)A->w, (const bf16*)A->a, (const bf16*)A->b, nullptr,
                          nullptr, (bf16*)A->y, L, R, C, r, A->alpha, s, split ? A->workspace : nullptr,
                          split ? A->workspace_bytes : 0, nullptr, groups);
}

int tc_bwd(const lors_bwd_args* A, cudaStream_t s) {
  const int L = (int)A->L, R = (int)A->R, C = (int)A->C, r = (int)A->r;
  const uint32_t* bits = A->mask_mode == LORS_MASK_BITS ? A->mask_bits : nullptr;
  const bf16 *x = (const bf16*)A->x, *w = (const bf16*)A->w, *a = (const bf16*)A->a, *b = (const bf16*)A->b,
             *dy = (const bf16*)A->dy;
  const bool tc = tc_shape_ok(R, C, r);
  const bool det = (A->flags & LORS_FLAG_DETERMINISTIC) != 0;
  const int rp = (int)pad_rank(r);
  int st;
  if (!(A->flags & LORS_FLAG_NO_DX)) {
    // the dX tail split's workspace: all of it (DX_ONLY) or after the P / Q slots and the rank-r region
    const size_t off = (A->flags & LORS_FLAG_DX_ONLY) ? 0 : 2 * rank_slot(A) + rank_r_region(A);
    const size_t dxw = dx_workspace(A);
    void* ws = dxw && A->workspace && A->workspace_bytes >= off + dxw ? (char*)A->workspace + off : nullptr;
    st = tc ? lors_gemm<true>(rp, dy, w, a, b, nullptr, bits, (bf16*)A->dx, L, R, C, r, A->alpha, s, ws, dxw)
            : simt_lors_gemm<bf16>(true, dy, w, bits, a, b, nullptr, (bf16*)A->dx, L, R, C, r, A->alpha, s);
    if (st) return st;
  }
  if (A->flags & LORS_FLAG_DX_ONLY) return LORS_OK;
  if (A->grad_mode == LORS_GRAD_STE) {
    const size_t slot = ((size_t)L * r * sizeof(float) + 255) / 256 * 256;
    bf16* P = (bf16*)A->p;
    bf16* Q = (bf16*)((char*)A->workspace + slot);
    if (tc && det) {
      // deterministic: every split-K product writes per-split partials that one kernel
      // sums in split order (P / Q rounded to bf16 there); adapters.py:396-399 order
      float* part = (float*)((char*)A->workspace + 2 * slot);
      if (P == nullptr) {  // P = X_t b^T
        P = (bf16*)A->workspace;
        if ((st = skinny<false, false, 0>(rp, x, b, P, L, r, C, r, 1.0f, true, s, nullptr, false, part))) return st;
      }
      if ((st = skinny<false, true, 0>(rp, dy, a, Q, L, r, R, r, 1.0f, true, s, nullptr, false, part))) return st;
      if ((st = skinny<true, true, 1>(rp, dy, P, A->da, R, r, L, r, A->alpha, true, s, nullptr, false, part)))
        return st;
      if ((st = skinny<true, true, 2>(rp, x, Q, A->db, C, r, L, C, A->alpha, true, s, nullptr, false, part)))
        return st;
    } else if (tc) {
      // P = X_t b^T and Q = dY_t a are split over their reductions (C, R) into fp32
      // accumulators so that L / 128 token tiles still fill the SMs, then rounded to bf16
      float* P32 = (float*)((char*)A->workspace + 2 * slot);
      float* Q32 = (float*)((char*)A->workspace + 3 * slot);
      const bool need_p = P == nullptr;
      const bool zeroed = (A->flags & LORS_FLAG_ZEROED) != 0;   // caller-zeroed dA and dB
      LORS_CUDA_TRY(cudaMemsetAsync(need_p ? (void*)P32 : (void*)Q32, 0, (need_p ? 2 : 1) * slot, s),
                    "zero rank-r accumulators");
      if (need_p) {  // P = X_t b^T
        P = (bf16*)A->workspace;
        if ((st = skinny<false, false, 0>(rp, x, b, P, L, r, C, r, 1.0f, true, s, P32))) return st;
      }
      static const bool fused_q_da = getenv("LORS_NO_QDA_PASS") == nullptr;
      if (fused_q_da && q_da_fits(rp, R)) {
        // P rounded first; then Q and dA from one pass over dY (K4b), Q rounded; dB
        if (!zeroed) LORS_CUDA_TRY(cudaMemsetAsync(A->da, 0, sizeof(float) * (size_t)R * r, s), "zero dA");
        if (need_p) {
          const int64_t na4 = (int64_t)L * r / 4;
          f32_to_bf16_pair_kernel<<<(unsigned)ceil_div(na4, 256), 256, 0, s>>>((const float4*)P32, P, na4, nullptr,
                                                                               nullptr, 0);
          LORS_CHECK_LAUNCH("P fp32 -> bf16");
        }
        if ((st = q_da(rp, dy, a, P, Q32, A->da, L, R, r, A->alpha, s))) return st;
        const int64_t nb4 = (int64_t)L * r / 4;
        f32_to_bf16_pair_kernel<<<(unsigned)ceil_div(nb4, 256), 256, 0, s>>>(nullptr, nullptr, 0,
                                                                             (const float4*)Q32, Q, nb4);
        LORS_CHECK_LAUNCH("Q fp32 -> bf16");
        if ((st = skinny<true, true, 2>(rp, x, Q, A->db, C, r, L, C, A->alpha, true, s, nullptr, zeroed))) return st;
        goto rank_r_done;
      }
      // Q = dY_t a: A = dY_t K-major [L, R], B = a [R, r] MN-major
      if ((st = skinny<false, true, 0>(rp, dy, a, Q, L, r, R, r, 1.0f, true, s, Q32))) return st;
      {
        const int64_t na4 = need_p ? (int64_t)L * r / 4 : 0, nb4 = (int64_t)L * r / 4;
        f32_to_bf16_pair_kernel<<<(unsigned)ceil_div(na4 + nb4, 256), 256, 0, s>>>(
            (const float4*)P32, P, na4, (const float4*)Q32, Q, nb4);
        LORS_CHECK_LAUNCH("rank-r fp32 -> bf16");
      }
      // dA = alpha dY_t^T P: A = dY_t as MN-major [L, R] (m = R), B = P [L, r] MN-major
      if ((st = skinny<true, true, 1>(rp, dy, P, A->da, R, r, L, r, A->alpha, true, s))) return st;
      // dB^T = alpha X_t^T Q: A = X_t MN-major (m = C), B = Q MN-major; stored transposed into dB [r, C]
      if ((st = skinny<true, true, 2>(rp, x, Q, A->db, C, r, L, C, A->alpha, true, s))) return st;
    rank_r_done:;
    } else {
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
    }
  } else {
    float* det_ws = det ? (float*)((char*)A->workspace + 2 * rank_slot(A)) : nullptr;
    st = tc ? masked_grad_tc(rp, dy, x, w, bits, a, b, A->da, A->db, L, R, C, r, A->alpha, s, det_ws)
            : simt_masked_grad<bf16>(dy, x, w, bits, a, b, A->da, A->db, L, R, C, r, A->alpha, s);
    if (st) return st;
  }
  if (A->dbias) {
    st = colsum<bf16>(dy, A->dbias, L, R, s);
    if (st) return st;
  }
  if (A->flags & LORS_FLAG_FAULT_DA_SIGN) return negate_f32(A->da, (int64_t)R * r, s);
  return LORS_OK;
}


// ===========================================================================
// K8: the fp32 parity mode's forward / dX on the tensor cores, 3xTF32:
//   out[t, m] = sum_k act[t, k] * Weff(m, k)
//   (FWD: act = X_t, Weff(m, k) = W_eff[m, k]; DX: act = dY_t, Weff(m, k) = W_eff[k, m])
// Each fp32 operand is split x = hi + lo (hi: the top 19 bits, what a TF32 MMA reads; lo = x - hi,
// exact), and D = A_hi B_hi + A_hi B_lo + A_lo B_hi in fp32 (TMEM) -- rel-L2 ~1e-6, inside the
// fp32 bar (1e-4) that plain TF32 misses.  W_eff is built by the FFMA kernels'
// weff_value (same p = sum_j fixed_j * streamed_j order), so the effective weight is the same
// fp32 value; only the GEMM's summation differs.  One CTA per [128 tokens x 128 features]
// tile, BK = 32 (one 128-byte SW128 row of fp32), two stages:
//   warp 8: TMA (activation tile, W tile, the streamed factor slice) into stage s
//   warps 0-7: split the activation tile in place (hi) + lo copy; W_eff of the W tile, split,
//              written K-major into two B tiles
//   warp 9: 12 MMAs per k-step (4 x K8, three products), M = N = 128, kind::tf32
//   warps 0-3: epilogue, TMEM -> registers -> out (+bias)
// ===========================================================================
namespace t3 {
// One CTA: 128 output features x 256 tokens; the W_eff tile of a k-step (built once) feeds all 256.
// D[feature][token] in TMEM (256 columns); A = W_eff (M = 128), B = activations (N = 256).
// TW transform warps (latency hiding: the split and the W_eff build are short dependent chains), then the
// TMA warp and the MMA warp; APT threads per activation row
constexpr int BF = 128, BT = 256, BK = 32, NSTAGE = 2, TW = 16, THREADS = 32 * (TW + 2);
constexpr int APT = TW * 32 / 256;
constexpr uint32_t WTILE = 128 * 128, ATILE = 256 * 128;   // [128][32] / [256][32] fp32, bytes
template <int RP>
constexpr uint32_t fac_bytes() { return 32 * RP * 4; }     // streamed factor slice, fp32
// stage: activation (raw -> hi in place), activation lo, W (raw -> W_eff hi in place), W_eff lo, factor
template <int RP>
constexpr uint32_t stage_bytes() { return 2 * ATILE + 2 * WTILE + fac_bytes<RP>(); }
template <int RP>
constexpr size_t smem_bytes() { return 1024 + NSTAGE * stage_bytes<RP>() + 256; }
__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t M, uint32_t N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
}  // namespace t3

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

template <bool DX, int RP>
__global__ void __launch_bounds__(t3::THREADS, 1)
    tf32x3_lors_kernel(const __grid_constant__ CUtensorMap tmAct, const __grid_constant__ CUtensorMap tmW,
                       const __grid_constant__ CUtensorMap tmS, const float* __restrict__ a,
                       const float* __restrict__ b, const uint32_t* __restrict__ bits,
                       const float* __restrict__ bias, float* __restrict__ out, int L, int R, int C, int r,
                       float alpha) {
  using namespace t3;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NSTAGE * stage_bytes<RP>());
  uint64_t* xf = full + NSTAGE;
  uint64_t* empty = xf + NSTAGE;
  uint64_t* accf = empty + NSTAGE;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);
  const int warp = warp_id(), lane = lane_id();
  const int M = DX ? C : R, K = DX ? R : C;
  const int m0 = blockIdx.x * BF, t0 = blockIdx.y * BT;
  const int nk = (K + BK - 1) / BK;
  const int64_t words = (C + 31) / 32;
  auto act_t = [&](int s) { return smem + s * stage_bytes<RP>(); };
  auto alo_t = [&](int s) { return smem + s * stage_bytes<RP>() + ATILE; };
  auto w_t = [&](int s) { return smem + s * stage_bytes<RP>() + 2 * ATILE; };
  auto wlo_t = [&](int s) { return smem + s * stage_bytes<RP>() + 2 * ATILE + WTILE; };
  auto fac_t = [&](int s) { return smem + s * stage_bytes<RP>() + 2 * ATILE + 2 * WTILE; };
  if (warp == TW && lane == 0) {
    for (int i = 0; i < NSTAGE; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&xf[i], TW);
      mbar_init(&empty[i], 1);
    }
    mbar_init(accf, 1);
    fence_barrier_init();
  }
  if (warp == TW + 1) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == TW) {
    if (lane == 0) {
      for (int i = 0; i < nk; ++i) {
        const int s = i % NSTAGE;
        mbar_wait(&empty[s], ((i / NSTAGE) & 1) ^ 1);
        const int k0 = i * BK;
        mbar_arrive_expect_tx(&full[s], ATILE + WTILE + fac_bytes<RP>());
        tma_load_2d(act_t(s), &tmAct, &full[s], k0, t0);                        // tokens t0 .. t0+127
        tma_load_2d(act_t(s) + ATILE / 2, &tmAct, &full[s], k0, t0 + 128);     // tokens t0+128 .. +255
        if (DX) tma_load_2d(w_t(s), &tmW, &full[s], m0, k0);                    // [32 k][128 m] plain
        else tma_load_2d(w_t(s), &tmW, &full[s], k0, m0);                       // [128 m][32 k] SW128
        if (DX) tma_load_2d(fac_t(s), &tmS, &full[s], 0, k0);                   // a [32 k][RP]
        else tma_load_2d(fac_t(s), &tmS, &full[s], k0, 0);                      // b [RP][32 k]
      }
    }
  } else if (warp == TW + 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(128, 256);
      for (int i = 0; i < nk; ++i) {
        const int s = i % NSTAGE;
        mbar_wait(&xf[s], (i / NSTAGE) & 1);
        tc_fence_after();
        const uint64_t wh = make_sdesc(smem_u32(w_t(s)), 16, 1024, SW_128);
        const uint64_t wl = make_sdesc(smem_u32(wlo_t(s)), 16, 1024, SW_128);
        const uint64_t ah = make_sdesc(smem_u32(act_t(s)), 16, 1024, SW_128);
        const uint64_t al = make_sdesc(smem_u32(alo_t(s)), 16, 1024, SW_128);
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {   // K = 8 tf32 = 32 bytes of the 128-byte row
          mma_tf32(tmem, wh + kk * 2, ah + kk * 2, idesc, (i > 0 || kk > 0) ? 1u : 0u);
          mma_tf32(tmem, wh + kk * 2, al + kk * 2, idesc, 1u);
          mma_tf32(tmem, wl + kk * 2, ah + kk * 2, idesc, 1u);
        }
        mma_commit(&empty[s]);
      }
      mma_commit(accf);
    }
  } else {
    // ---------------------------------------------------------------- transform warps 0 .. TW-1
    const int tid = threadIdx.x;            // 0 .. 32 TW - 1
    // W_eff: RPT rows (row0, row0 + 128 / RPT) x KQ k a thread; a warp shares its k group, so the factor
    // slice reads are broadcasts (two rows a thread halve them; r <= 16 keeps both rows' factors in registers)
    constexpr int RPT = RP <= 16 ? 2 : 1, RSTEP = 128 / RPT, KQ = BK * RSTEP / (TW * 32);
    const int row0 = tid % RSTEP, half = tid / RSTEP;
    float fix[RPT][RP];                     // fixed factor of each row: FWD a[m][j], DX b[j][m]
#pragma unroll
    for (int rr = 0; rr < RPT; ++rr) {
      const int gm = m0 + row0 + rr * RSTEP;
#pragma unroll
      for (int j = 0; j < RP; ++j)
        fix[rr][j] = (j < r && gm < M) ? (DX ? b[(int64_t)j * C + gm] : a[(int64_t)gm * r + j]) : 0.f;
    }
    // packed-mask words of a step (FWD one a row, DX one a row and k), fetched a step ahead
    constexpr int NWB = RPT * (DX ? KQ : 1);
    auto fetch_bits = [&](const int k0n, uint32_t (&dst)[NWB]) {
#pragma unroll
      for (int rr = 0; rr < RPT; ++rr) {
        const int gm = m0 + row0 + rr * RSTEP;
#pragma unroll
        for (int e = 0; e < (DX ? KQ : 1); ++e) {
          const int gk = k0n + half * KQ + e;
          dst[rr * (DX ? KQ : 1) + e] =
              (gm < M && gk < K) ? __ldg(bits + (int64_t)(DX ? gk : gm) * words + ((DX ? gm : gk) >> 5)) : 0u;
        }
      }
    };
    uint32_t mwn[NWB] = {};
    if (bits != nullptr) fetch_bits(0, mwn);
    for (int i = 0; i < nk; ++i) {
      const int s = i % NSTAGE;
      const int k0 = i * BK;
      mbar_wait(&full[s], (i / NSTAGE) & 1);
      uint32_t mwd[NWB];
#pragma unroll
      for (int e = 0; e < NWB; ++e) mwd[e] = mwn[e];
      if (bits != nullptr) fetch_bits(k0 + BK, mwn);
      // 1. activation row tid / APT (256 tokens): hi in place, lo beside it
      {
        const int ar = tid / APT, ac = (tid % APT) * (8 / APT);
        const uint32_t arow = smem_u32(act_t(s)) + ar * 128, lrow = smem_u32(alo_t(s)) + ar * 128;
#pragma unroll
        for (int c = ac; c < ac + 8 / APT; ++c) {
          const uint32_t off = (uint32_t)((c ^ (ar & 7)) << 4);
          uint32_t v[4];
          lds128(arow + off, v);
          float h[4], l[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            h[e] = tf32_hi(__uint_as_float(v[e]));
            l[e] = __uint_as_float(v[e]) - h[e];
          }
          // (hi stays as the raw value: kind::tf32 reads only the top 19 bits of each fp32 operand)
          asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(lrow + off), "f"(l[0]), "f"(l[1]), "f"(l[2]),
                       "f"(l[3]) : "memory");
        }
      }
      // 2. W_eff(m = row0 + RSTEP rr, k = k0 + KQ half + e)
      float wv[RPT][KQ];
#pragma unroll
      for (int rr = 0; rr < RPT; ++rr) {
        const int row = row0 + rr * RSTEP;
        if (DX) {
          const float* wr = reinterpret_cast<const float*>(w_t(s));   // [32 k][128 m]
#pragma unroll
          for (int e = 0; e < KQ; ++e) wv[rr][e] = wr[(half * KQ + e) * 128 + row];
        } else {
          const uint32_t wrow = smem_u32(w_t(s)) + row * 128;
#pragma unroll
          for (int c = 0; c < KQ / 4; ++c) {
            uint32_t v[4];
            lds128(wrow + (uint32_t)(((half * (KQ / 4) + c) ^ (row & 7)) << 4), v);
#pragma unroll
            for (int e = 0; e < 4; ++e) wv[rr][4 * c + e] = __uint_as_float(v[e]);
          }
        }
      }
      float pv[RPT][KQ];
      const uint32_t fbase = smem_u32(fac_t(s));
#pragma unroll
      for (int rr = 0; rr < RPT; ++rr)
#pragma unroll
        for (int e = 0; e < KQ; ++e) pv[rr][e] = 0.f;
      if (DX) {   // a[k][j] ([32][RP]): row k's factors as float4, the chain over j in order
#pragma unroll
        for (int e = 0; e < KQ; ++e) {
#pragma unroll
          for (int j4 = 0; j4 < RP / 4; ++j4) {
            uint32_t f[4];
            lds128(fbase + (uint32_t)(((half * KQ + e) * RP + 4 * j4) * 4), f);   // warp-uniform: a broadcast
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (4 * j4 + u < r) {
#pragma unroll
                for (int rr = 0; rr < RPT; ++rr)
                  pv[rr][e] = fmaf(fix[rr][4 * j4 + u], __uint_as_float(f[u]), pv[rr][e]);
              }
          }
        }
      } else {    // b[j][k] ([RP][32]): KQ consecutive k of row j
#pragma unroll
        for (int j = 0; j < RP; ++j) {
          if (j < r) {
#pragma unroll
            for (int c = 0; c < KQ / 4; ++c) {
              uint32_t f[4];
              lds128(fbase + (uint32_t)((j * BK + half * KQ + 4 * c) * 4), f);   // warp-uniform: a broadcast
#pragma unroll
              for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int rr = 0; rr < RPT; ++rr)
                  pv[rr][4 * c + u] = fmaf(fix[rr][j], __uint_as_float(f[u]), pv[rr][4 * c + u]);
            }
          }
        }
      }
      float hv[RPT][KQ], lv[RPT][KQ];
#pragma unroll
      for (int rr = 0; rr < RPT; ++rr) {
        const int gm = m0 + row0 + rr * RSTEP;
#pragma unroll
        for (int e = 0; e < KQ; ++e) {
          const int gk = k0 + half * KQ + e;
          float v = 0.f;
          if (gm < M && gk < K) {
            const int wcol = DX ? gm : gk;
            const bool keep = bits != nullptr
                                  ? ((mwd[rr * (DX ? KQ : 1) + (DX ? e : 0)] >> (wcol & 31)) & 1u) != 0u
                                  : wv[rr][e] != 0.0f;
            v = weff_value<float>(keep, wv[rr][e], pv[rr][e], alpha);
          }
          hv[rr][e] = tf32_hi(v);
          lv[rr][e] = v - hv[rr][e];
        }
      }
      // (dX: the W tile's [k][m] layout is rewritten as [m][k], so every thread reads first)
      if (DX) named_bar_sync(1, TW * 32);
#pragma unroll
      for (int rr = 0; rr < RPT; ++rr) {
        const int row = row0 + rr * RSTEP;
        const uint32_t hrow = smem_u32(w_t(s)) + row * 128, lrow = smem_u32(wlo_t(s)) + row * 128;
#pragma unroll
        for (int c = 0; c < KQ / 4; ++c) {
          const uint32_t off = (uint32_t)(((half * (KQ / 4) + c) ^ (row & 7)) << 4);
          asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(hrow + off), "f"(hv[rr][4 * c]),
                       "f"(hv[rr][4 * c + 1]), "f"(hv[rr][4 * c + 2]), "f"(hv[rr][4 * c + 3]) : "memory");
          asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(lrow + off), "f"(lv[rr][4 * c]),
                       "f"(lv[rr][4 * c + 1]), "f"(lv[rr][4 * c + 2]), "f"(lv[rr][4 * c + 3]) : "memory");
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&xf[s]);
    }
    // ---------------------------------------------------------------- epilogue (warps 0-7: TMEM lanes = features,
    // warp / 4 picks the token half)
    if (warp < 8) {
      mbar_wait(accf, 0);
      tc_fence_after();
      const int m = m0 + (warp & 3) * 32 + lane;
      const float bv = (!DX && bias != nullptr && m < M) ? bias[m] : 0.f;
#pragma unroll 1
      for (int c0 = (warp >> 2) * (BT / 2); c0 < (warp >> 2) * (BT / 2) + BT / 2; c0 += 32) {
        uint32_t v[32];
        tmem_ld_x32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)c0, v);
        tmem_ld_wait();
        if (m < M) {
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const int t = t0 + c0 + q;
            if (t < L) out[(int64_t)t * M + m] = __uint_as_float(v[q]) + bv;   // a warp: 32 consecutive m
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == TW + 1) tmem_dealloc<256>(tmem);
}

template <bool DX, int RP>
static int launch_tf32x3(const float* act, const float* w, const float* a, const float* b, const uint32_t* bits,
                         const float* bias, float* out, int L, int R, int C, int r, float alpha, cudaStream_t s) {
  using namespace t3;
  const int M = DX ? C : R, K = DX ? R : C;
  CUtensorMap tAct, tW, tS;
  int st;
  if ((st = make_map(&tAct, act, K, L, 32, 128, 128, "tf32 activation", true))) return st;
  if (DX) st = make_map(&tW, w, C, R, 128, 32, 0, "tf32 W (dX)", true);     // [32 k rows][128 m], plain
  else st = make_map(&tW, w, C, R, 32, 128, 128, "tf32 W", true);           // [128 m][32 k], SW128
  if (st) return st;
  if (DX) st = make_map(&tS, a, r, R, RP, 32, 0, "tf32 a slice", true);     // a [32 k][RP]
  else st = make_map(&tS, b, C, r, 32, RP, 0, "tf32 b slice", true);        // b [RP][32 k]
  if (st) return st;
  auto kern = tf32x3_lors_kernel<DX, RP>;
  const size_t smem = smem_bytes<RP>();
  LORS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                "tf32x3 smem attribute");
  dim3 grid((unsigned)ceil_div(M, BF), (unsigned)ceil_div(L, BT));
  kern<<<grid, THREADS, smem, s>>>(tAct, tW, tS, a, b, bits, bias, out, L, R, C, r, alpha);
  LORS_CHECK_LAUNCH(DX ? "tf32x3_lors<dx>" : "tf32x3_lors<fwd>");
  (void)K;
  return LORS_OK;
}

// fp32 forward / dX on the tensor cores when the shapes allow 16-byte TMA rows (R, C, r multiples of 4,
// r <= 32); returns LORS_ERR_SHAPE otherwise (the caller runs the FFMA kernels)
int tf32x3_lors_gemm(bool dx, const float* act, const float* w, const float* a, const float* b, const uint32_t* bits,
                     const float* bias, float* out, int L, int R, int C, int r, float alpha, cudaStream_t s) {
  if (R % 4 || C % 4 || r % 4 || r > 32 || r < 1 || L < 1) return LORS_ERR_SHAPE;
  if (r <= 16)
    return dx ? launch_tf32x3<true, 16>(act, w, a, b, bits, bias, out, L, R, C, r, alpha, s)
              : launch_tf32x3<false, 16>(act, w, a, b, bits, bias, out, L, R, C, r, alpha, s);
  return dx ? launch_tf32x3<true, 32>(act, w, a, b, bits, bias, out, L, R, C, r, alpha, s)
            : launch_tf32x3<false, 32>(act, w, a, b, bits, bias, out, L, R, C, r, alpha, s);
}

}  // namespace lors
