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
//   K4 tc_skinny            the rank-r products P = X b^T, Q = dY a,
//        dA = alpha dY^T P, dB = alpha Q^T X (adapters.py:396-399), N = r.
//
// Shapes that the TMA path cannot address (rows not 16-byte multiples, or
// r > 64) run the FFMA kernels of lors_simt.cu instead.
#include <cuda.h>

#include <algorithm>
#include <cstring>

#include "lors_simt.cuh"
#include "lors_tc.cuh"
#include "ptx_sm100.cuh"

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
                    uint32_t box_outer, uint32_t swizzle_bytes, const char* what) {
  PFN_encodeTiled_t fn = encode_fn();
  if (fn == nullptr) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return LORS_ERR_CUDA;
  }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * sizeof(bf16)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, to_swizzle(swizzle_bytes), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error(std::string("cuTensorMapEncodeTiled failed for ") + what + " (CUresult " + std::to_string((int)r) +
              ")");
    return LORS_ERR_CUDA;
  }
  return LORS_OK;
}

static inline uint32_t pad_rank(int r) { return r <= 16 ? 16 : r <= 32 ? 32 : 64; }

// ===========================================================================
// K4: skinny GEMM  D[M, BN] = sum_k A[m, k] B[n, k]   (M tile 128, BN = padded r)
//   A_MN / B_MN: operand stored MN-major (m resp. n contiguous) instead of K-major.
//   OUT 0: bf16 out[m*ldo + n]; 1: fp32 alpha*out[m*ldo + n]; 2: fp32 alpha*out[n*ldo + m]
//   (1/2 accumulate atomically when the grid splits K).
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
                     int M, int N, int K, int k_per_split, int ldo, float alpha, int atomic_out) {
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
        if (OUT == 0) {
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
              if (atomic_out) atomicAdd(dst, val);
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
template <int BN, bool A_MN, bool B_MN, int OUT>
static int launch_skinny(const bf16* A, const bf16* B, void* out, int M, int N, int K, int ldo, float alpha,
                         bool allow_split, cudaStream_t s) {
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
  int split = 1;
  if (allow_split && OUT != 0) split = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(148, mt), kblocks / 4));
  const int kps = (int)ceil_div(kblocks, split) * sk::BK;
  split = (int)ceil_div(K, kps);
  if (split > 1) {
    const size_t elems = OUT == 2 ? (size_t)N * ldo : (size_t)M * ldo;
    LORS_CUDA_TRY(cudaMemsetAsync(out, 0, elems * sizeof(float), s), "zero split-K output");
  }
  auto kern = tc_skinny_kernel<BN, A_MN, B_MN, OUT>;
  const size_t smem = sk::smem_bytes<BN>();
  LORS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                "skinny smem attribute");
  kern<<<dim3(mt, split), sk::THREADS, smem, s>>>(tA, tB, out, M, N, K, kps, ldo, alpha, split > 1 ? 1 : 0);
  LORS_CHECK_LAUNCH("tc_skinny");
  return LORS_OK;
}

// dispatch on the padded rank
template <bool A_MN, bool B_MN, int OUT>
static int skinny(int rp, const bf16* A, const bf16* B, void* out, int M, int N, int K, int ldo, float alpha,
                  bool allow_split, cudaStream_t s) {
  switch (rp) {
    case 16: return launch_skinny<16, A_MN, B_MN, OUT>(A, B, out, M, N, K, ldo, alpha, allow_split, s);
    case 32: return launch_skinny<32, A_MN, B_MN, OUT>(A, B, out, M, N, K, ldo, alpha, allow_split, s);
    default: return launch_skinny<64, A_MN, B_MN, OUT>(A, B, out, M, N, K, ldo, alpha, allow_split, s);
  }
}

// ===========================================================================
// K1 / K3: GEMM with W_eff rebuilt in the prologue.
//
//   out[l, m] = sum_k act[l, k] * Weff'(m, k)
//   FWD (DX=false): act = X_t [L, C], m over R, k over C, Weff'(m,k) = Weff[m,k]
//   DX  (DX=true) : act = dY_t [L, R], m over C, k over R, Weff'(m,k) = Weff[k,m]
//
// CTA tile: 128 output features (TMEM lanes) x 256 tokens (TMEM columns),
// k-step 64.  Per k-step:
//   TMA   : W tile, act tile [256 x 64] (SW128), streamed adapter factor
//   MMA   : recompute D_re[128 x 64] = F . S^T (K = r) into TMEM (2 buffers)
//   xform : 8 warps read D_re (tcgen05.ld), add W, select on the mask, round
//           to bf16, store the K-major SW128 W_eff tile (2 buffers)
//   MMA   : D[128 x 256] += W_eff . act^T (4 x K16)
// The recompute of step i is issued before the main MMA of step i-1, so the
// transform of step i overlaps the tensor-core work of step i-1.
// warps 0-7: transform + epilogue, warp 8: TMA producer, warp 9: MMA issuer.
// ===========================================================================
namespace rg {
constexpr int BM = 128, BN = 256, BK = 64, THREADS = 320, XFORM_THREADS = 256;
constexpr uint32_t ACT_BYTES = BN * BK * 2;   // 32 KB
constexpr uint32_t W_BYTES = BM * BK * 2;     // 16 KB
constexpr uint32_t WEFF_BYTES = BM * BK * 2;  // 16 KB
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t RE_COL = 256;              // recompute buffers at TMEM cols 256 / 320
template <int RP>
constexpr int stages() { return 3; }
template <int RP>
constexpr uint32_t sf_bytes() { return 64 * RP * 2; }   // streamed factor tile (64 k x RP)
template <int RP>
constexpr uint32_t ff_bytes() { return 128 * RP * 2; }  // fixed factor tile (128 m x RP)
template <int RP>
constexpr uint32_t stage_bytes() { return W_BYTES + ACT_BYTES + sf_bytes<RP>(); }
template <int RP>
constexpr size_t smem_bytes() {
  return 1024 + stages<RP>() * stage_bytes<RP>() + 2 * WEFF_BYTES + ff_bytes<RP>() + 256;
}
}  // namespace rg

template <bool DX, int RP>
__global__ void __launch_bounds__(rg::THREADS, 1)
    tc_lors_gemm_kernel(const __grid_constant__ CUtensorMap tmAct, const __grid_constant__ CUtensorMap tmW,
                        const __grid_constant__ CUtensorMap tmS, const __grid_constant__ CUtensorMap tmF,
                        const __grid_constant__ CUtensorMap tmOut, const bf16* __restrict__ bias,
                        const uint32_t* __restrict__ bits, int words_per_row, int Mout, int Kred, float alpha) {
  using namespace rg;
  constexpr int S = stages<RP>();
  constexpr uint32_t SF = sf_bytes<RP>(), FF = ff_bytes<RP>(), STG = stage_bytes<RP>();
  constexpr uint32_t SWR = RP * 2;  // swizzle span of the K-major rank-r tiles
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // stage s: [W | act | streamed factor]
  uint8_t* stage0 = smem;
  uint8_t* weff = smem + S * STG;           // 2 buffers
  uint8_t* ffac = weff + 2 * WEFF_BYTES;    // fixed factor
  uint64_t* bars = reinterpret_cast<uint64_t*>(ffac + FF);
  uint64_t* full = bars;                    // [S]   TMA -> MMA / xform
  uint64_t* empty = full + S;               // [S]   main MMA -> TMA
  uint64_t* refull = empty + S;             // [2]   recompute MMA -> xform
  uint64_t* reempty = refull + 2;           // [2]   xform -> MMA
  uint64_t* wready = reempty + 2;           // [2]   xform -> main MMA
  uint64_t* wempty = wready + 2;            // [2]   main MMA -> xform
  uint64_t* ffull = wempty + 2;             // fixed factor landed
  uint64_t* accf = ffull + 1;               // accumulator complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);

  const int warp = warp_id(), lane = lane_id();
  const int m0 = blockIdx.x * BM;
  const int l0 = blockIdx.y * BN;
  const int nk = (Kred + BK - 1) / BK;

  if (warp == 8 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&refull[b], 1);
      mbar_init(&reempty[b], 8);
      mbar_init(&wready[b], 8);
      mbar_init(&wempty[b], 1);
    }
    mbar_init(ffull, 1);
    mbar_init(accf, 1);
    fence_barrier_init();
    tma_prefetch_desc(&tmAct);
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmS);
    tma_prefetch_desc(&tmF);
    tma_prefetch_desc(&tmOut);
  }
  if (warp == 9) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      mbar_arrive_expect_tx(ffull, FF);
      if (DX) {  // b [r, C] as MN-major A of the recompute: two 64-wide atoms
        tma_load_2d(ffac, &tmF, ffull, m0, 0);
        tma_load_2d(ffac + FF / 2, &tmF, ffull, m0 + 64, 0);
      } else {   // a [R, r] K-major
        tma_load_2d(ffac, &tmF, ffull, 0, m0);
      }
      for (int i = 0; i < nk; ++i) {
        const int s = i % S;
        const uint32_t ph = (i / S) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], STG);
        uint8_t* st = stage0 + s * STG;
        const int k0 = i * BK;
        if (DX) tma_load_2d(st, &tmW, &full[s], m0, k0);   // W[k0:k0+64, m0:m0+128], no swizzle
        else tma_load_2d(st, &tmW, &full[s], k0, m0);      // W[m0:m0+128, k0:k0+64], SW128
        tma_load_2d(st + W_BYTES, &tmAct, &full[s], k0, l0);
        if (DX) tma_load_2d(st + W_BYTES + ACT_BYTES, &tmS, &full[s], 0, k0);  // a[k0:k0+64, :] K-major
        else tma_load_2d(st + W_BYTES + ACT_BYTES, &tmS, &full[s], k0, 0);     // b[:, k0:k0+64] MN-major
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_re = make_idesc_bf16(128, 64, DX, !DX);
      constexpr uint32_t idesc_main = make_idesc_bf16(128, 256, false, false);
      mbar_wait(ffull, 0);
      const uint32_t ff_base = smem_u32(ffac);
      for (int i = 0; i <= nk; ++i) {
        if (i < nk) {
          const int s = i % S;
          const int rb = i & 1;
          mbar_wait(&full[s], (i / S) & 1);
          mbar_wait(&reempty[rb], ((i >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t sf_base = smem_u32(stage0 + s * STG + W_BYTES + ACT_BYTES);
#pragma unroll
          for (int kk = 0; kk < RP / 16; ++kk) {
            uint64_t ad, bd;
            if (DX) {
              ad = make_sdesc(ff_base + kk * 2048, FF / 2, 1024, SW_128);            // b^T, MN-major
              bd = make_sdesc(sf_base + kk * 32, 16, 8 * SWR, sw_layout(SWR));       // a rows, K-major
            } else {
              ad = make_sdesc(ff_base + kk * 32, 16, 8 * SWR, sw_layout(SWR));       // a rows, K-major
              bd = make_sdesc(sf_base + kk * 2048, 0, 1024, SW_128);                 // b cols, MN-major
            }
            mma_bf16(tmem + RE_COL + rb * 64, ad, bd, idesc_re, kk > 0 ? 1u : 0u);
          }
          mma_commit(&refull[rb]);
        }
        if (i >= 1) {
          const int j = i - 1;
          const int s = j % S;
          const int wb = j & 1;
          mbar_wait(&wready[wb], (j >> 1) & 1);
          tc_fence_after();
          const uint32_t a_base = smem_u32(weff + wb * WEFF_BYTES);
          const uint32_t b_base = smem_u32(stage0 + s * STG + W_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            mma_bf16(tmem, make_sdesc(a_base + kk * 32, 16, 1024, SW_128), make_sdesc(b_base + kk * 32, 16, 1024, SW_128),
                     idesc_main, (j > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&empty[s]);
          mma_commit(&wempty[wb]);
        }
      }
      mma_commit(accf);
    }
  } else {
    // ------------------------------------------------------------ transform warps 0..7
    const int q = warp & 3;        // TMEM lane quarter
    const int h = warp >> 2;       // column half of the 64-wide k-step
    const int t = q * 32 + lane;   // feature row inside the tile (TMEM lane)
    const int gm = m0 + t;         // global output feature
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    for (int i = 0; i < nk; ++i) {
      const int s = i % S;
      const int rb = i & 1;
      // 1. rank-r product of this k-step, 32 columns for this thread's row
      mbar_wait(&refull[rb], (i >> 1) & 1);
      tc_fence_after();
      uint32_t p[32];
      tmem_ld_x32(tmem + lane_addr + RE_COL + rb * 64 + h * 32, p);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&reempty[rb]);
      // 2. W values (TMA landed) and the destination buffer free
      mbar_wait(&full[s], (i / S) & 1);
      mbar_wait(&wempty[rb], ((i >> 1) & 1) ^ 1);
      const uint8_t* wt = stage0 + s * STG;
      uint8_t* dst = weff + rb * WEFF_BYTES + t * 128;
      const int kbase = i * BK + h * 32;
      uint32_t mword = 0xFFFFFFFFu;
      if (bits != nullptr) {
        if (!DX) {
          mword = (gm < Mout) ? __ldg(bits + (int64_t)gm * words_per_row + (kbase >> 5)) : 0u;
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {  // 4 chunks of 8 k-values
        float wv[8];
        if (!DX) {
          const uint4 raw = *reinterpret_cast<const uint4*>(wt + t * 128 + (((h * 4 + c) ^ (t & 7)) << 4));
          const bf16* e = reinterpret_cast<const bf16*>(&raw);
#pragma unroll
          for (int u = 0; u < 8; ++u) wv[u] = __bfloat162float(e[u]);
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u)
            wv[u] = __bfloat162float(*reinterpret_cast<const bf16*>(wt + (h * 32 + c * 8 + u) * 256 + t * 2));
        }
        uint32_t pk[4];
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
          float o[2];
#pragma unroll
          for (int e2 = 0; e2 < 2; ++e2) {
            const int kk = c * 8 + u + e2;  // 0..31 within this thread's half
            bool keep;
            if (bits == nullptr) {
              keep = wv[u + e2] != 0.0f;
            } else if (!DX) {
              keep = (mword >> kk) & 1u;
            } else {
              const int64_t krow = kbase + kk;
              keep = (gm < Mout && krow < Kred)
                         ? ((__ldg(bits + krow * words_per_row + (gm >> 5)) >> (gm & 31)) & 1u)
                         : false;
            }
            o[e2] = keep ? fmaf(alpha, __uint_as_float(p[kk]), wv[u + e2]) : 0.0f;
          }
          pk[u / 2] = pack_bf16x2(o[0], o[1]);
        }
        *reinterpret_cast<uint4*>(dst + (((h * 4 + c) ^ (t & 7)) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&wready[rb]);
    }
    // ------------------------------------------------------------ epilogue
    mbar_wait(accf, 0);
    tc_fence_after();
    // stage [256 tokens][128 features] bf16 (256 B rows) in the drained pipeline buffers
    uint8_t* stg = smem;
    float bv = 0.f;
    if (!DX && bias != nullptr && gm < Mout) bv = __bfloat162float(bias[gm]);
#pragma unroll 1
    for (int c0 = 0; c0 < 128; c0 += 32) {
      const int col = h * 128 + c0;  // token offset inside the tile
      uint32_t v[32];
      tmem_ld_x32(tmem + lane_addr + col, v);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        *reinterpret_cast<bf16*>(stg + (col + j) * 256 + t * 2) = __float2bfloat16_rn(__uint_as_float(v[j]) + bv);
      }
    }
    fence_proxy_async_smem();
    named_bar_sync(1, XFORM_THREADS);
    if (warp == 0 && lane == 0) {
      tma_store_2d(&tmOut, stg, m0, l0);
      tma_store_commit();
      tma_store_wait_all();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc<TMEM_COLS>(tmem);
}

template <bool DX, int RP>
static int launch_lors_gemm(const bf16* act, const bf16* w, const bf16* a, const bf16* b, const bf16* bias,
                            const uint32_t* bits, bf16* out, int L, int R, int C, int r, float alpha,
                            cudaStream_t s) {
  using namespace rg;
  const int Mout = DX ? C : R, Kred = DX ? R : C;
  CUtensorMap tAct, tW, tS, tF, tOut;
  int st;
  if ((st = make_map(&tAct, act, Kred, L, 64, BN, 128, "activation"))) return st;
  if (DX) st = make_map(&tW, w, C, R, 128, 64, 0, "W (dX)");
  else st = make_map(&tW, w, C, R, 64, 128, 128, "W (fwd)");
  if (st) return st;
  if (DX) {
    if ((st = make_map(&tS, a, r, R, RP, 64, RP * 2, "a (streamed)"))) return st;
    if ((st = make_map(&tF, b, C, r, 64, RP, 128, "b (fixed)"))) return st;
  } else {
    if ((st = make_map(&tS, b, C, r, 64, RP, 128, "b (streamed)"))) return st;
    if ((st = make_map(&tF, a, r, R, RP, 128, RP * 2, "a (fixed)"))) return st;
  }
  if ((st = make_map(&tOut, out, Mout, L, 128, BN, 0, "output"))) return st;
  auto kern = tc_lors_gemm_kernel<DX, RP>;
  const size_t smem = smem_bytes<RP>();
  LORS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                "lors_gemm smem attribute");
  dim3 grid((unsigned)ceil_div(Mout, BM), (unsigned)ceil_div(L, BN));
  kern<<<grid, THREADS, smem, s>>>(tAct, tW, tS, tF, tOut, bias, bits, (int)ceil_div(C, 32), Mout, Kred, alpha);
  LORS_CHECK_LAUNCH(DX ? "tc_lors_gemm<dx>" : "tc_lors_gemm<fwd>");
  return LORS_OK;
}

template <bool DX>
static int lors_gemm(int rp, const bf16* act, const bf16* w, const bf16* a, const bf16* b, const bf16* bias,
                     const uint32_t* bits, bf16* out, int L, int R, int C, int r, float alpha, cudaStream_t s) {
  switch (rp) {
    case 16: return launch_lors_gemm<DX, 16>(act, w, a, b, bias, bits, out, L, R, C, r, alpha, s);
    case 32: return launch_lors_gemm<DX, 32>(act, w, a, b, bias, bits, out, L, R, C, r, alpha, s);
    default: return launch_lors_gemm<DX, 64>(act, w, a, b, bias, bits, out, L, R, C, r, alpha, s);
  }
}

// ===========================================================================
// dispatch
// ===========================================================================
bool tc_shape_ok(int64_t R, int64_t C, int64_t r) {
  return R % 8 == 0 && C % 8 == 0 && r % 8 == 0 && r <= 64;
}

size_t tc_fwd_workspace(const lors_fwd_args*) { return 0; }
size_t tc_bwd_workspace(const lors_bwd_args*) { return 0; }

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
  st = lors_gemm<false>(rp, x, w, a, b, (const bf16*)A->bias, bits, (bf16*)A->y, L, R, C, r, A->alpha, s);
  if (st) return st;
  if (A->flags & LORS_FLAG_EMIT_P)  // P = X_t b^T: A = X_t K-major, B = b [r, C] K-major
    st = skinny<false, false, 0>(rp, x, b, A->p, L, r, C, r, 1.0f, false, s);
  return st;
}

int tc_bwd(const lors_bwd_args* A, cudaStream_t s) {
  const int L = (int)A->L, R = (int)A->R, C = (int)A->C, r = (int)A->r;
  const uint32_t* bits = A->mask_mode == LORS_MASK_BITS ? A->mask_bits : nullptr;
  const bf16 *x = (const bf16*)A->x, *w = (const bf16*)A->w, *a = (const bf16*)A->a, *b = (const bf16*)A->b,
             *dy = (const bf16*)A->dy;
  const bool tc = tc_shape_ok(R, C, r);
  const int rp = (int)pad_rank(r);
  int st;
  if (!(A->flags & LORS_FLAG_NO_DX)) {
    st = tc ? lors_gemm<true>(rp, dy, w, a, b, nullptr, bits, (bf16*)A->dx, L, R, C, r, A->alpha, s)
            : simt_lors_gemm<bf16>(true, dy, w, bits, a, b, nullptr, (bf16*)A->dx, L, R, C, r, A->alpha, s);
    if (st) return st;
  }
  if (A->grad_mode == LORS_GRAD_STE) {
    const size_t slot = ((size_t)L * r * sizeof(float) + 255) / 256 * 256;
    bf16* P = (bf16*)A->p;
    bf16* Q = (bf16*)((char*)A->workspace + slot);
    if (tc) {
      if (P == nullptr) {  // P = X_t b^T
        P = (bf16*)A->workspace;
        if ((st = skinny<false, false, 0>(rp, x, b, P, L, r, C, r, 1.0f, false, s))) return st;
      }
      // Q = dY_t a: A = dY_t K-major [L, R], B = a [R, r] MN-major
      if ((st = skinny<false, true, 0>(rp, dy, a, Q, L, r, R, r, 1.0f, false, s))) return st;
      // dA = alpha dY_t^T P: A = dY_t as MN-major [L, R] (m = R), B = P [L, r] MN-major
      if ((st = skinny<true, true, 1>(rp, dy, P, A->da, R, r, L, r, A->alpha, true, s))) return st;
      // dB^T = alpha X_t^T Q: A = X_t MN-major (m = C), B = Q MN-major; stored transposed into dB [r, C]
      if ((st = skinny<true, true, 2>(rp, x, Q, A->db, C, r, L, C, A->alpha, true, s))) return st;
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
