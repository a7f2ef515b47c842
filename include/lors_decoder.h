/* Decoder-side helpers of the B200 LoRS library (not the drop-in boundary of
 * the LoRS path -- that is lors_b200.h).  They serve the LLaMA-shaped decoder
 * that benchmarks the path at BASELINE configs 3-5.  Same status
 * codes and error string (lors_last_error) as lors_b200.h.
 */
#ifndef LORS_DECODER_H_
#define LORS_DECODER_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Rotary position embedding (rotate-half convention), bf16, optionally fused with
 * a head transpose:
 *   layout 0:  x [B, S, H, hd] -> y [B, H, S, hd]   (forward: projection output -> attention input)
 *   layout 1:  x [B, H, S, hd] -> y [B, S, H, hd]   (backward: attention grad -> projection grad)
 *   layout 2:  x [B, S, H, hd] -> y [B, S, H, hd]   (no transpose: attention reads strided heads)
 * y = x * cos + rotate_half(x) * (inverse ? -sin : sin), cos / sin [S, hd] (bf16), computed in fp32 and
 * rounded once.  hd must be a multiple of 8 (16-byte accesses). */
int lors_rope(const void* x, void* y, const void* cos_t, const void* sin_t, int64_t B, int64_t S, int64_t H,
              int64_t hd, int32_t layout, int32_t inverse, void* stream);

/* SwiGLU of the decoder MLP, bf16, n elements (n % 8 == 0, 16-byte aligned):
 *   forward  h = silu(g) * u
 *   backward dg = dh * u * silu'(g),  du = dh * silu(g)     (silu'(g) = s (1 + g (1 - s)), s = sigmoid(g))
 * computed in fp32 and rounded once per output. */
int lors_swiglu(const void* g, const void* u, void* h, int64_t n, void* stream);
int lors_swiglu_bwd(const void* dh, const void* g, const void* u, void* dg, void* du, int64_t n, void* stream);

/* out = a + b (+ c when c != NULL), bf16, n elements (n % 8 == 0, 16-byte aligned), summed in fp32 and
 * rounded once; out may alias a.  The input gradient of projections sharing one input (q/k/v, gate/up). */
int lors_add3(const void* a, const void* b, const void* c, void* out, int64_t n, void* stream);

/* Residual add fused with the RMSNorm that follows it (pre-norm decoder), bf16 rows of D elements
 * (D % 8 == 0, D <= 8192), gamma [D] bf16, fp32 arithmetic:
 *   forward   hn = bf16(h + o)            (o may be NULL: hn = h and `hn` may be NULL)
 *             rstd = 1 / sqrt(mean(hn^2) + eps)   (fp32 [rows], saved for the backward)
 *             x = bf16(hn rstd gamma)
 *   backward  dh = bf16(dhn + rstd (dx gamma) - hn rstd^3 sum(dx gamma hn) / D)   (dhn may be NULL)
 *             -- the gradient of both h and o; the residual path's gradient and the norm's meet in
 *             one rounding, without a separate add kernel. */
int lors_add_rmsnorm(const void* h, const void* o, const void* gamma, void* hn, void* x, float* rstd,
                     int64_t rows, int64_t D, float eps, void* stream);
int lors_add_rmsnorm_bwd(const void* dhn, const void* dx, const void* hn, const void* gamma, const float* rstd,
                         void* dh, int64_t rows, int64_t D, void* stream);

/* Next-token cross-entropy over bf16 logits [N, V] (V % 8 == 0) with int64 targets [N], fp32 arithmetic:
 *   forward   lse = logsumexp(logits[n, :]) (one online max / sum pass), loss_rows[n] = lse[n] - logits[n, t_n]
 *   backward  dlogits[n, j] = bf16((exp(logits[n, j] - lse[n]) - [j == t_n]) * grad_out[0] / N)
 * grad_out is a device fp32 scalar (the gradient of the mean loss, read on the device: no host sync);
 * dlogits may alias logits (the backward then overwrites them in place). */
int lors_cross_entropy(const void* logits, const int64_t* targets, float* loss_rows, float* lse, int64_t N,
                       int64_t V, void* stream);
int lors_cross_entropy_bwd(const void* logits, const int64_t* targets, const float* lse, const float* grad_out,
                           void* dlogits, int64_t N, int64_t V, void* stream);

/* Fused AdamW over the flat fp32 adapter masters (torch.optim.AdamW semantics, decoupled weight decay,
 * bias-corrected moments), one launch for every adapter of the model; also refreshes the bf16 compute
 * copies (`shadow`, may be NULL) the LoRS kernels read, so no per-call casts remain:
 *   p *= 1 - lr wd;  m = b1 m + (1 - b1) g;  v = b2 v + (1 - b2) g^2;
 *   p -= lr / (1 - b1^t) * m / (sqrt(v) / sqrt(1 - b2^t) + eps);  shadow = bf16(p) */
int lors_adamw(float* p, const float* g, float* m, float* v, void* shadow, int64_t n, float lr, float beta1,
               float beta2, float eps, float weight_decay, int64_t step, void* stream);

/* lors_adamw with the step count on the device, for CUDA-graph capture (trainer.Trainer(cuda_graph=True)):
 * counter = int64[2] in device memory, zero-initialised; counter[0] = updates taken so far.  The call applies
 * update t = counter[0] + 1 (bias corrections computed on the device from t, in double as lors_adamw does on
 * the host, by a one-thread launch ahead of the elementwise one) and leaves counter[0] = t; counter[1] is
 * scratch (the two corrections). */
int lors_adamw_dstep(float* p, const float* g, float* m, float* v, void* shadow, int64_t n, float lr, float beta1,
                     float beta2, float eps, float weight_decay, int64_t* counter, void* stream);

/* Fused gradient collective + AdamW over NVLink peer memory: every rank owns the shard
 * [rank n / world, (rank + 1) n / world) of the flat adapter buffers (n a multiple of 4 * world).  For each
 * element of its shard it sums the gradient over all ranks' gradient buffers (peer loads), divides by world,
 * applies the AdamW update of lors_adamw to its master copy with its optimizer-state shard (m, v hold n /
 * world elements), and stores the new value -- and its bf16 compute copy -- into every rank's parameter
 * (and shadow) buffer (peer stores).  `grads`, `params`, `shadows` are device arrays of `world` peer
 * pointers (symmetric-memory buffer_ptrs_dev); the caller brackets the call with symmetric-memory barriers.
 * One reduce-scatter, one optimizer step and one all-gather in a single kernel. */
int lors_adamw_p2p(const void* grads, const void* params, const void* shadows, float* m_shard, float* v_shard,
                   int64_t n, int32_t rank, int32_t world, float lr, float beta1, float beta2, float eps,
                   float weight_decay, int64_t step, void* stream);

#ifdef __cplusplus
}
#endif
#endif
