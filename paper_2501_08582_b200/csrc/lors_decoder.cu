// Decoder-side helpers (include/lors_decoder.h): fused RoPE + head transpose.
// Memory-bound elementwise work: one thread per 8 consecutive elements of a head's
// first half and their partners in the second half (16-byte loads and stores), for
// four heads at once when H % 4 == 0.
#include <type_traits>
#include "../../include/lors_decoder.h"
#include "lors_common.cuh"

#include <cmath>

namespace lors {

__device__ __forceinline__ void unpack8(const uint4 v, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 v;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return v;
}

// One thread: 8 + 8 elements (both halves) of HPT consecutive heads at one (b, s) -- the
// cos / sin rows are loaded once for the HPT heads and all x loads are issued before any
// arithmetic.  IDX: the index type of the thread -> (b, s, head group, c) decomposition,
// 32-bit whenever the thread count allows (64-bit division made the kernel issue-bound).
template <int LAYOUT, int HPT, typename IDX>
__global__ void rope_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y,
                            const __nv_bfloat16* __restrict__ cs, const __nv_bfloat16* __restrict__ sn, IDX B,
                            IDX S, IDX H, int hd, float sgn) {
  const int half = hd / 2, per_head = half / 8;
  const IDX HG = H / HPT;
  const IDX idx = (IDX)blockIdx.x * (IDX)blockDim.x + (IDX)threadIdx.x;
  const IDX total = B * S * HG * (IDX)per_head;
  if (idx >= total) return;
  const int c = (int)(idx % (IDX)per_head) * 8;
  IDX rest = idx / (IDX)per_head;
  // LAYOUT 0 / 2 walk the input [B, S, H] order, LAYOUT 1 the input [B, H, S] order
  IDX b, s, hg;
  if (LAYOUT != 1) {
    hg = rest % HG; rest /= HG; s = rest % S; b = rest / S;
  } else {
    s = rest % S; rest /= S; hg = rest % HG; b = rest / HG;
  }
  uint4 xa[HPT], xb[HPT];
  int64_t outo[HPT];
#pragma unroll
  for (int k = 0; k < HPT; ++k) {
    const IDX h = hg * HPT + k;
    const int64_t bsh = (((int64_t)b * S + s) * H + h) * hd;   // [B, S, H, hd]
    const int64_t bhs = (((int64_t)b * H + h) * S + s) * hd;   // [B, H, S, hd]
    const int64_t in = LAYOUT == 1 ? bhs : bsh;
    outo[k] = LAYOUT == 0 ? bhs : bsh;                         // 2: [B, S, H, hd] in place order
    xa[k] = *reinterpret_cast<const uint4*>(x + in + c);
    xb[k] = *reinterpret_cast<const uint4*>(x + in + half + c);
  }
  float c1[8], c2[8], s1[8], s2[8];
  const int64_t sr = (int64_t)s * hd;
  unpack8(__ldg(reinterpret_cast<const uint4*>(cs + sr + c)), c1);
  unpack8(__ldg(reinterpret_cast<const uint4*>(cs + sr + half + c)), c2);
  unpack8(__ldg(reinterpret_cast<const uint4*>(sn + sr + c)), s1);
  unpack8(__ldg(reinterpret_cast<const uint4*>(sn + sr + half + c)), s2);
#pragma unroll
  for (int k = 0; k < HPT; ++k) {
    float x1[8], x2[8], o1[8], o2[8];
    unpack8(xa[k], x1);
    unpack8(xb[k], x2);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      // rotate_half(x) = (-x2, x1)
      o1[i] = fmaf(x1[i], c1[i], -sgn * x2[i] * s1[i]);
      o2[i] = fmaf(x2[i], c2[i], sgn * x1[i] * s2[i]);
    }
    *reinterpret_cast<uint4*>(y + outo[k] + c) = pack8(o1);
    *reinterpret_cast<uint4*>(y + outo[k] + half + c) = pack8(o2);
  }
}

__global__ void swiglu_kernel(const uint4* __restrict__ g, const uint4* __restrict__ u, uint4* __restrict__ h,
                              int64_t n8) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n8) return;
  float gf[8], uf[8], o[8];
  unpack8(g[i], gf);
  unpack8(u[i], uf);
#pragma unroll
  for (int k = 0; k < 8; ++k) o[k] = gf[k] / (1.0f + __expf(-gf[k])) * uf[k];
  h[i] = pack8(o);
}

// out = bf16(a + b (+ c)), the sum in fp32 (the grouped projections' input gradient: one pass
// over the two or three dX instead of one bf16 add per extra projection)
__global__ void add3_kernel(const uint4* __restrict__ a, const uint4* __restrict__ b, const uint4* __restrict__ c,
                            uint4* __restrict__ out, int64_t n8) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n8) return;
  float af[8], bf[8], cf[8];
  unpack8(a[i], af);
  unpack8(b[i], bf);
  if (c != nullptr) {
    unpack8(c[i], cf);
#pragma unroll
    for (int k = 0; k < 8; ++k) af[k] = af[k] + bf[k] + cf[k];
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) af[k] += bf[k];
  }
  out[i] = pack8(af);
}

__global__ void swiglu_bwd_kernel(const uint4* __restrict__ dh, const uint4* __restrict__ g,
                                  const uint4* __restrict__ u, uint4* __restrict__ dg, uint4* __restrict__ du,
                                  int64_t n8) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n8) return;
  float d[8], gf[8], uf[8], og[8], ou[8];
  unpack8(dh[i], d);
  unpack8(g[i], gf);
  unpack8(u[i], uf);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float s = 1.0f / (1.0f + __expf(-gf[k]));
    const float silu = gf[k] * s;
    og[k] = d[k] * uf[k] * (s * (1.0f + gf[k] * (1.0f - s)));
    ou[k] = d[k] * silu;
  }
  dg[i] = pack8(og);
  du[i] = pack8(ou);
}

__global__ void adamw_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                             float* __restrict__ v, __nv_bfloat16* __restrict__ shadow, int64_t n, float decay,
                             float b1, float b2, float step_size, float inv_sqrt_bc2, float eps) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float gi = g[i];
  const float mi = fmaf(b1, m[i], (1.0f - b1) * gi);
  const float vi = fmaf(b2, v[i], (1.0f - b2) * gi * gi);
  const float pi = p[i] * decay - step_size * mi / (sqrtf(vi) * inv_sqrt_bc2 + eps);
  m[i] = mi;
  v[i] = vi;
  p[i] = pi;
  if (shadow != nullptr) shadow[i] = __float2bfloat16_rn(pi);
}

// AdamW with the step counter on the device (a CUDA-graph replay reuses the launch, so the
// bias correction cannot be a host argument): counter[0] = updates taken, counter[1] = scratch.
// One thread advances the count and computes the two bias-correction scalars in double, as
// lors_adamw does on the host; the elementwise update (adamw_kernel's arithmetic) reads them.
__global__ void adamw_advance_kernel(unsigned long long* counter, float lr, float b1, float b2) {
  const unsigned long long t = counter[0] + 1ull;
  counter[0] = t;
  const double bc1 = 1.0 - pow((double)b1, (double)t);
  const double bc2 = 1.0 - pow((double)b2, (double)t);
  float* sc = reinterpret_cast<float*>(&counter[1]);
  sc[0] = (float)((double)lr / bc1);
  sc[1] = (float)(1.0 / sqrt(bc2));
}

__global__ void adamw_dstep_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                                   float* __restrict__ v, __nv_bfloat16* __restrict__ shadow, int64_t n, float decay,
                                   float b1, float b2, float eps, const unsigned long long* __restrict__ counter) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float* sc = reinterpret_cast<const float*>(&counter[1]);
  const float step_size = sc[0], inv_sqrt_bc2 = sc[1];
  const float gi = g[i];
  const float mi = fmaf(b1, m[i], (1.0f - b1) * gi);
  const float vi = fmaf(b2, v[i], (1.0f - b2) * gi * gi);
  const float pi = p[i] * decay - step_size * mi / (sqrtf(vi) * inv_sqrt_bc2 + eps);
  m[i] = mi;
  v[i] = vi;
  p[i] = pi;
  if (shadow != nullptr) shadow[i] = __float2bfloat16_rn(pi);
}

// Peer-memory AdamW over one shard: 4 elements per thread (16-byte peer loads and stores).
// The rank's own master copy is read through params[rank] (all copies are identical).
__global__ void adamw_p2p_kernel(const float* const* __restrict__ grads, float* const* __restrict__ params,
                                 __nv_bfloat16* const* __restrict__ shadows, float* __restrict__ m,
                                 float* __restrict__ v, int64_t lo, int64_t shard4, int rank, int world, float decay,
                                 float b1, float b2, float step_size, float inv_sqrt_bc2, float eps, float inv_world) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // float4 index inside the shard
  if (q >= shard4) return;
  const int64_t e = lo + 4 * q;                                         // element index in the flat buffer
  float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int p = 0; p < world; ++p) {                                     // reduce over the ranks (NVLink loads)
    const float4 x = *reinterpret_cast<const float4*>(grads[p] + e);
    g.x += x.x; g.y += x.y; g.z += x.z; g.w += x.w;
  }
  const float4 p0 = *reinterpret_cast<const float4*>(params[rank] + e);
  float4 mm = reinterpret_cast<float4*>(m)[q], vv = reinterpret_cast<float4*>(v)[q];
  float gi[4] = {g.x * inv_world, g.y * inv_world, g.z * inv_world, g.w * inv_world};
  float pi[4] = {p0.x, p0.y, p0.z, p0.w}, mi[4] = {mm.x, mm.y, mm.z, mm.w}, vi[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    mi[k] = fmaf(b1, mi[k], (1.0f - b1) * gi[k]);
    vi[k] = fmaf(b2, vi[k], (1.0f - b2) * gi[k] * gi[k]);
    pi[k] = pi[k] * decay - step_size * mi[k] / (sqrtf(vi[k]) * inv_sqrt_bc2 + eps);
  }
  reinterpret_cast<float4*>(m)[q] = make_float4(mi[0], mi[1], mi[2], mi[3]);
  reinterpret_cast<float4*>(v)[q] = make_float4(vi[0], vi[1], vi[2], vi[3]);
  const float4 pn = make_float4(pi[0], pi[1], pi[2], pi[3]);
  __nv_bfloat162 s01 = __floats2bfloat162_rn(pi[0], pi[1]), s23 = __floats2bfloat162_rn(pi[2], pi[3]);
  uint2 sb;
  sb.x = *reinterpret_cast<uint32_t*>(&s01);
  sb.y = *reinterpret_cast<uint32_t*>(&s23);
  for (int p = 0; p < world; ++p) {                                     // all-gather (NVLink stores)
    *reinterpret_cast<float4*>(params[p] + e) = pn;
    if (shadows != nullptr) *reinterpret_cast<uint2*>(shadows[p] + e) = sb;
  }
}

}  // namespace lors

extern "C" int lors_adamw_p2p(const void* grads, const void* params, const void* shadows, float* m_shard,
                              float* v_shard, int64_t n, int32_t rank, int32_t world, float lr, float beta1,
                              float beta2, float eps, float weight_decay, int64_t step, void* stream) {
  using namespace lors;
  if (!grads || !params || !m_shard || !v_shard) {
    set_error("lors_adamw_p2p: null pointer");
    return LORS_ERR_ARGUMENT;
  }
  if (world < 1 || world > 64 || rank < 0 || rank >= world || n < 0 || n % (4 * (int64_t)world) != 0) {
    set_error("lors_adamw_p2p: need 1 <= world <= 64, 0 <= rank < world, n a multiple of 4 * world");
    return LORS_ERR_ARGUMENT;
  }
  if (step < 1 || !(lr >= 0.0f) || !(beta1 >= 0.0f && beta1 < 1.0f) || !(beta2 >= 0.0f && beta2 < 1.0f)) {
    set_error("lors_adamw_p2p: invalid hyper-parameters");
    return LORS_ERR_ARGUMENT;
  }
  const int64_t shard = n / world, shard4 = shard / 4;
  if (shard4 == 0) return LORS_OK;
  const double bc1 = 1.0 - std::pow((double)beta1, (double)step);
  const double bc2 = 1.0 - std::pow((double)beta2, (double)step);
  adamw_p2p_kernel<<<(unsigned)ceil_div(shard4, 256), 256, 0, (cudaStream_t)stream>>>(
      (const float* const*)grads, (float* const*)params, (__nv_bfloat16* const*)shadows, m_shard, v_shard,
      (int64_t)rank * shard, shard4, rank, world, 1.0f - lr * weight_decay, beta1, beta2, (float)(lr / bc1),
      (float)(1.0 / std::sqrt(bc2)), eps, 1.0f / (float)world);
  LORS_CHECK_LAUNCH("adamw_p2p");
  return LORS_OK;
}

extern "C" int lors_adamw_dstep(float* p, const float* g, float* m, float* v, void* shadow, int64_t n, float lr,
                                float beta1, float beta2, float eps, float weight_decay, int64_t* counter,
                                void* stream) {
  using namespace lors;
  if (!p || !g || !m || !v || !counter) {
    set_error("lors_adamw_dstep: null pointer");
    return LORS_ERR_ARGUMENT;
  }
  if (n < 0 || !(lr >= 0.0f) || !(beta1 >= 0.0f && beta1 < 1.0f) || !(beta2 >= 0.0f && beta2 < 1.0f)) {
    set_error("lors_adamw_dstep: invalid hyper-parameters (n >= 0, lr >= 0, 0 <= beta < 1)");
    return LORS_ERR_ARGUMENT;
  }
  if (n == 0) return LORS_OK;
  auto* cnt = reinterpret_cast<unsigned long long*>(counter);
  adamw_advance_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(cnt, lr, beta1, beta2);
  LORS_CHECK_LAUNCH("adamw_advance");
  adamw_dstep_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(
      p, g, m, v, (__nv_bfloat16*)shadow, n, 1.0f - lr * weight_decay, beta1, beta2, eps, cnt);
  LORS_CHECK_LAUNCH("adamw_dstep");
  return LORS_OK;
}

extern "C" int lors_adamw(float* p, const float* g, float* m, float* v, void* shadow, int64_t n, float lr,
                          float beta1, float beta2, float eps, float weight_decay, int64_t step, void* stream) {
  using namespace lors;
  if (!p || !g || !m || !v) {
    set_error("lors_adamw: null pointer");
    return LORS_ERR_ARGUMENT;
  }
  if (n < 0 || step < 1 || !(lr >= 0.0f) || !(beta1 >= 0.0f && beta1 < 1.0f) || !(beta2 >= 0.0f && beta2 < 1.0f)) {
    set_error("lors_adamw: invalid hyper-parameters (n >= 0, step >= 1, lr >= 0, 0 <= beta < 1)");
    return LORS_ERR_ARGUMENT;
  }
  if (n == 0) return LORS_OK;
  const double bc1 = 1.0 - std::pow((double)beta1, (double)step);
  const double bc2 = 1.0 - std::pow((double)beta2, (double)step);
  adamw_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(
      p, g, m, v, (__nv_bfloat16*)shadow, n, 1.0f - lr * weight_decay, beta1, beta2, (float)(lr / bc1),
      (float)(1.0 / std::sqrt(bc2)), eps);
  LORS_CHECK_LAUNCH("adamw");
  return LORS_OK;
}

// ---------------------------------------------------------------------------
// residual add + RMSNorm: one CTA of 256 threads per row, each thread NV 16-byte
// vectors of the row held in registers between the two passes
// ---------------------------------------------------------------------------
namespace lors {
namespace {
constexpr int NORM_THREADS = 256;

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();                       // red[] reusable
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < NORM_THREADS / 32; ++i) t += red[i];
  return t;
}
}  // namespace

template <int NV, bool ADD>
__global__ void __launch_bounds__(NORM_THREADS) add_rmsnorm_kernel(const uint4* __restrict__ h, const uint4* __restrict__ o,
                                                                   const uint4* __restrict__ gamma,
                                                                   uint4* __restrict__ hn, uint4* __restrict__ x,
                                                                   float* __restrict__ rstd, int d8, float eps) {
  __shared__ float red[NORM_THREADS / 32];
  const int64_t base = (int64_t)blockIdx.x * d8;
  float f[NV][8];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int v = threadIdx.x + k * NORM_THREADS;
    if (v < d8) {
      unpack8(h[base + v], f[k]);
      if (ADD) {
        float g[8];
        unpack8(o[base + v], g);
#pragma unroll
        for (int e = 0; e < 8; ++e) f[k][e] += g[e];
        const uint4 r = pack8(f[k]);     // the residual stream is bf16: round, then normalise that
        if (hn) hn[base + v] = r;
        unpack8(r, f[k]);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) ss += f[k][e] * f[k][e];
    }
  }
  const float rs = rsqrtf(block_sum(ss, red) / (float)(d8 * 8) + eps);
  if (threadIdx.x == 0) rstd[blockIdx.x] = rs;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int v = threadIdx.x + k * NORM_THREADS;
    if (v < d8) {
      float g[8];
      unpack8(gamma[v], g);
#pragma unroll
      for (int e = 0; e < 8; ++e) f[k][e] = f[k][e] * rs * g[e];
      x[base + v] = pack8(f[k]);
    }
  }
}

template <int NV>
__global__ void __launch_bounds__(NORM_THREADS) add_rmsnorm_bwd_kernel(const uint4* __restrict__ dhn,
                                                                       const uint4* __restrict__ dx,
                                                                       const uint4* __restrict__ hn,
                                                                       const uint4* __restrict__ gamma,
                                                                       const float* __restrict__ rstd,
                                                                       uint4* __restrict__ dh, int d8) {
  __shared__ float red[NORM_THREADS / 32];
  const int64_t base = (int64_t)blockIdx.x * d8;
  float dg[NV][8], hv[NV][8];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int v = threadIdx.x + k * NORM_THREADS;
    if (v < d8) {
      float g[8];
      unpack8(dx[base + v], dg[k]);
      unpack8(gamma[v], g);
      unpack8(hn[base + v], hv[k]);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        dg[k][e] *= g[e];
        s += dg[k][e] * hv[k][e];
      }
    }
  }
  const float r = rstd[blockIdx.x];
  const float c = r * r * r * block_sum(s, red) / (float)(d8 * 8);
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int v = threadIdx.x + k * NORM_THREADS;
    if (v < d8) {
      float out[8];
      if (dhn) unpack8(dhn[base + v], out);
      else {
#pragma unroll
        for (int e = 0; e < 8; ++e) out[e] = 0.f;
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) out[e] += r * dg[k][e] - c * hv[k][e];
      dh[base + v] = pack8(out);
    }
  }
}
}  // namespace lors

// ---------------------------------------------------------------------------
// cross-entropy: one CTA of 256 threads per row, 16-byte vectors, online max / sum
// ---------------------------------------------------------------------------
namespace lors {
namespace {
constexpr int CE_THREADS = 256;
}  // namespace

__global__ void __launch_bounds__(CE_THREADS) ce_fwd_kernel(const uint4* __restrict__ logits,
                                                            const int64_t* __restrict__ targets,
                                                            float* __restrict__ loss_rows, float* __restrict__ lse,
                                                            int v8) {
  __shared__ float sm[CE_THREADS / 32], ss[CE_THREADS / 32];
  const int64_t base = (int64_t)blockIdx.x * v8;
  float m = -INFINITY, sum = 0.f;
  for (int v = threadIdx.x; v < v8; v += CE_THREADS) {
    float f[8];
    unpack8(logits[base + v], f);
    float lm = f[0];
#pragma unroll
    for (int e = 1; e < 8; ++e) lm = fmaxf(lm, f[e]);
    if (lm > m) {
      sum *= __expf(m - lm);
      m = lm;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) sum += __expf(f[e] - m);
  }
  // combine (max, sum) pairs: warp, then block
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, sum, o);
    const float nm = fmaxf(m, om);
    sum = (m == -INFINITY ? 0.f : sum * __expf(m - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
    m = nm;
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sm[w] = m;
    ss[w] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = sm[0];
    for (int i = 1; i < CE_THREADS / 32; ++i) M = fmaxf(M, sm[i]);
    float S = 0.f;
    for (int i = 0; i < CE_THREADS / 32; ++i) S += ss[i] * __expf(sm[i] - M);
    const float L = M + __logf(S);
    const int64_t t = targets[blockIdx.x];
    const __nv_bfloat16* row = reinterpret_cast<const __nv_bfloat16*>(logits + base);
    lse[blockIdx.x] = L;
    loss_rows[blockIdx.x] = L - __bfloat162float(row[t]);
  }
}

__global__ void __launch_bounds__(CE_THREADS) ce_bwd_kernel(const uint4* logits, const int64_t* __restrict__ targets,
                                                            const float* __restrict__ lse,
                                                            const float* __restrict__ grad_out, uint4* dlogits,
                                                            int v8, float inv_n) {
  const int64_t base = (int64_t)blockIdx.x * v8;
  const float L = lse[blockIdx.x], g = grad_out[0] * inv_n;
  const int64_t t = targets[blockIdx.x];
  for (int v = threadIdx.x; v < v8; v += CE_THREADS) {
    float f[8];
    unpack8(logits[base + v], f);
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = (__expf(f[e] - L) - ((int64_t)v * 8 + e == t ? 1.f : 0.f)) * g;
    dlogits[base + v] = pack8(f);
  }
}
}  // namespace lors

extern "C" int lors_cross_entropy(const void* logits, const int64_t* targets, float* loss_rows, float* lse,
                                  int64_t N, int64_t V, void* stream) {
  using namespace lors;
  if (!logits || !targets || !loss_rows || !lse) {
    set_error("lors_cross_entropy: null pointer");
    return LORS_ERR_ARGUMENT;
  }
  if (N < 0 || V <= 0 || V % 8 != 0 || N > INT32_MAX || V / 8 > INT32_MAX) {
    set_error("lors_cross_entropy: need V % 8 == 0");
    return LORS_ERR_SHAPE;
  }
  if (N == 0) return LORS_OK;
  ce_fwd_kernel<<<(unsigned)N, CE_THREADS, 0, (cudaStream_t)stream>>>((const uint4*)logits, targets, loss_rows, lse,
                                                                      (int)(V / 8));
  LORS_CHECK_LAUNCH("cross_entropy");
  return LORS_OK;
}

extern "C" int lors_cross_entropy_bwd(const void* logits, const int64_t* targets, const float* lse,
                                      const float* grad_out, void* dlogits, int64_t N, int64_t V, void* stream) {
  using namespace lors;
  if (!logits || !targets || !lse || !grad_out || !dlogits) {
    set_error("lors_cross_entropy_bwd: null pointer");
    return LORS_ERR_ARGUMENT;
  }
  if (N < 0 || V <= 0 || V % 8 != 0 || N > INT32_MAX || V / 8 > INT32_MAX) {
    set_error("lors_cross_entropy_bwd: need V % 8 == 0");
    return LORS_ERR_SHAPE;
  }
  if (N == 0) return LORS_OK;
  ce_bwd_kernel<<<(unsigned)N, CE_THREADS, 0, (cudaStream_t)stream>>>((const uint4*)logits, targets, lse, grad_out,
                                                                      (uint4*)dlogits, (int)(V / 8), 1.0f / (float)N);
  LORS_CHECK_LAUNCH("cross_entropy_bwd");
  return LORS_OK;
}

extern "C" int lors_add_rmsnorm(const void* h, const void* o, const void* gamma, void* hn, void* x, float* rstd,
                                int64_t rows, int64_t D, float eps, void* stream) {
  using namespace lors;
  if (!h || !gamma || !x || !rstd || (o && !hn)) {
    set_error("lors_add_rmsnorm: null pointer");
    return LORS_ERR_ARGUMENT;
  }
  if (rows < 0 || D <= 0 || D % 8 != 0 || D > 8192 || rows > INT32_MAX) {
    set_error("lors_add_rmsnorm: need D % 8 == 0, 0 < D <= 8192");
    return LORS_ERR_SHAPE;
  }
  if (rows == 0) return LORS_OK;
  const int d8 = (int)(D / 8);
  const int nv = (d8 + NORM_THREADS - 1) / NORM_THREADS;
  cudaStream_t s = (cudaStream_t)stream;
  auto go = [&](auto kern) {
    kern<<<(unsigned)rows, NORM_THREADS, 0, s>>>((const uint4*)h, (const uint4*)o, (const uint4*)gamma, (uint4*)hn,
                                                 (uint4*)x, rstd, d8, eps);
  };
  if (o) {
    if (nv <= 1) go(add_rmsnorm_kernel<1, true>);
    else if (nv <= 2) go(add_rmsnorm_kernel<2, true>);
    else go(add_rmsnorm_kernel<4, true>);
  } else {
    if (nv <= 1) go(add_rmsnorm_kernel<1, false>);
    else if (nv <= 2) go(add_rmsnorm_kernel<2, false>);
    else go(add_rmsnorm_kernel<4, false>);
  }
  LORS_CHECK_LAUNCH("add_rmsnorm");
  return LORS_OK;
}

extern "C" int lors_add_rmsnorm_bwd(const void* dhn, const void* dx, const void* hn, const void* gamma,
                                    const float* rstd, void* dh, int64_t rows, int64_t D, void* stream) {
  using namespace lors;
  if (!dx || !hn || !gamma || !rstd || !dh) {
    set_error("lors_add_rmsnorm_bwd: null pointer");
    return LORS_ERR_ARGUMENT;
  }
  if (rows < 0 || D <= 0 || D % 8 != 0 || D > 8192 || rows > INT32_MAX) {
    set_error("lors_add_rmsnorm_bwd: need D % 8 == 0, 0 < D <= 8192");
    return LORS_ERR_SHAPE;
  }
  if (rows == 0) return LORS_OK;
  const int d8 = (int)(D / 8);
  const int nv = (d8 + NORM_THREADS - 1) / NORM_THREADS;
  cudaStream_t s = (cudaStream_t)stream;
  auto go = [&](auto kern) {
    kern<<<(unsigned)rows, NORM_THREADS, 0, s>>>((const uint4*)dhn, (const uint4*)dx, (const uint4*)hn,
                                                 (const uint4*)gamma, rstd, (uint4*)dh, d8);
  };
  if (nv <= 1) go(add_rmsnorm_bwd_kernel<1>);
  else if (nv <= 2) go(add_rmsnorm_bwd_kernel<2>);
  else go(add_rmsnorm_bwd_kernel<4>);
  LORS_CHECK_LAUNCH("add_rmsnorm_bwd");
  return LORS_OK;
}

extern "C" int lors_add3(const void* a, const void* b, const void* c, void* out, int64_t n, void* stream) {
  using namespace lors;
  if (!a || !b || !out) {
    set_error("lors_add3: null pointer");
    return LORS_ERR_ARGUMENT;
  }
  if (n < 0 || n % 8 != 0) {
    set_error("lors_add3: element count must be a non-negative multiple of 8");
    return LORS_ERR_SHAPE;
  }
  if (n == 0) return LORS_OK;
  const int64_t n8 = n / 8;
  add3_kernel<<<(unsigned)ceil_div(n8, 256), 256, 0, (cudaStream_t)stream>>>(
      (const uint4*)a, (const uint4*)b, (const uint4*)c, (uint4*)out, n8);
  LORS_CHECK_LAUNCH("add3");
  return LORS_OK;
}

extern "C" int lors_swiglu(const void* g, const void* u, void* h, int64_t n, void* stream) {
  using namespace lors;
  if (!g || !u || !h) {
    set_error("lors_swiglu: null pointer");
    return LORS_ERR_ARGUMENT;
  }
  if (n < 0 || n % 8 != 0) {
    set_error("lors_swiglu: element count must be a non-negative multiple of 8");
    return LORS_ERR_SHAPE;
  }
  if (n == 0) return LORS_OK;
  const int64_t n8 = n / 8;
  swiglu_kernel<<<(unsigned)ceil_div(n8, 256), 256, 0, (cudaStream_t)stream>>>((const uint4*)g, (const uint4*)u,
                                                                              (uint4*)h, n8);
  LORS_CHECK_LAUNCH("swiglu");
  return LORS_OK;
}

extern "C" int lors_swiglu_bwd(const void* dh, const void* g, const void* u, void* dg, void* du, int64_t n,
                               void* stream) {
  using namespace lors;
  if (!dh || !g || !u || !dg || !du) {
    set_error("lors_swiglu_bwd: null pointer");
    return LORS_ERR_ARGUMENT;
  }
  if (n < 0 || n % 8 != 0) {
    set_error("lors_swiglu_bwd: element count must be a non-negative multiple of 8");
    return LORS_ERR_SHAPE;
  }
  if (n == 0) return LORS_OK;
  const int64_t n8 = n / 8;
  swiglu_bwd_kernel<<<(unsigned)ceil_div(n8, 256), 256, 0, (cudaStream_t)stream>>>(
      (const uint4*)dh, (const uint4*)g, (const uint4*)u, (uint4*)dg, (uint4*)du, n8);
  LORS_CHECK_LAUNCH("swiglu_bwd");
  return LORS_OK;
}

extern "C" int lors_rope(const void* x, void* y, const void* cos_t, const void* sin_t, int64_t B, int64_t S,
                         int64_t H, int64_t hd, int32_t layout, int32_t inverse, void* stream) {
  using namespace lors;
  if (!x || !y || !cos_t || !sin_t) {
    set_error("lors_rope: null pointer");
    return LORS_ERR_ARGUMENT;
  }
  if (B < 0 || S < 0 || H < 0 || hd <= 0 || hd % 16 != 0) {
    set_error("lors_rope: head dim must be a positive multiple of 16 (two 8-element halves)");
    return LORS_ERR_SHAPE;
  }
  if (layout != 0 && layout != 1 && layout != 2) {
    set_error("lors_rope: layout must be 0 ([B,S,H,hd] -> [B,H,S,hd]), 1 (the reverse) or 2 (no transpose)");
    return LORS_ERR_ARGUMENT;
  }
  const int hpt = H % 4 == 0 ? 4 : 1;
  const int64_t total = B * S * (H / hpt) * (hd / 16);
  if (total == 0) return LORS_OK;
  const cudaStream_t s = (cudaStream_t)stream;
  const unsigned grid = (unsigned)ceil_div(total, 256);
  const float sgn = inverse ? -1.0f : 1.0f;
  auto xp = (const __nv_bfloat16*)x;
  auto yp = (__nv_bfloat16*)y;
  auto cp = (const __nv_bfloat16*)cos_t;
  auto sp = (const __nv_bfloat16*)sin_t;
  auto launch = [&](auto layout_c, auto hpt_c, auto idx_zero) {
    using IDX = decltype(idx_zero);
    rope_kernel<decltype(layout_c)::value, decltype(hpt_c)::value, IDX><<<grid, 256, 0, s>>>(
        xp, yp, cp, sp, (IDX)B, (IDX)S, (IDX)H, (int)hd, sgn);
  };
  auto by_layout = [&](auto hpt_c, auto idx_zero) {
    if (layout == 0) launch(std::integral_constant<int, 0>(), hpt_c, idx_zero);
    else if (layout == 1) launch(std::integral_constant<int, 1>(), hpt_c, idx_zero);
    else launch(std::integral_constant<int, 2>(), hpt_c, idx_zero);
  };
  auto by_hpt = [&](auto idx_zero) {
    if (hpt == 4) by_layout(std::integral_constant<int, 4>(), idx_zero);
    else by_layout(std::integral_constant<int, 1>(), idx_zero);
  };
  if (total < ((int64_t)1 << 31)) by_hpt(uint32_t(0));
  else by_hpt(int64_t(0));
  LORS_CHECK_LAUNCH("rope");
  return LORS_OK;
}
