/*
 * lors_b200.h -- C ABI of the B200-native LoRS masked-LoRA linear layer.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/pkg/src/lors/adapters.py):
 *
 *   lors_fwd               replaces  lors_forward            adapters.py:359-373
 *                          (and sqft_gc_forward, bitwise the same function,
 *                           adapters.py:330-334)
 *   lors_bwd               replaces  lors_backward           adapters.py:376-406
 *                          grad_mode = LORS_GRAD_MASKED replaces
 *                          sqft_gc_backward / _sqft_grads    adapters.py:303-312,337-352
 *   lors_effective_weight  replaces  merged_weight / merge   adapters.py:214-224,709-727
 *   lors_pack_mask         replaces  mask_matrix (M = W != 0) adapters.py:209-211,
 *                                    SparseWeight.mask_bool  prune.py:61-62
 *   lors_compress_24       2:4 values+metadata for the sparse-tensor-core forward;
 *                          validity rule of two_four_valid   prune.py:72-77
 *   lors_grad_outer        dW = dY^T X (optionally (.)M), the per-layer probe gradient
 *                          of init_gradient_svd              initialization.py:209-211
 *
 * Layout is the torch one (row-major, tokens are ROWS):
 *   X_t [L, C], W [R, C], a [R, r], b [r, C], Y_t [L, R], dY_t [L, R], dX_t [L, C].
 * The reference orientation (X is C x L) is the transpose; the Python wrapper
 * translates views without copies.
 *
 * Conventions: memory is owned by the caller, the
 * library never allocates device memory; all work is stream-ordered on the
 * given cudaStream_t with no host synchronisation; no global mutable state
 * except a per-device capability cache and a thread-local error string, so
 * calls are reentrant across streams and threads.  Pointers must be 16-byte
 * aligned.  The bf16 path runs tcgen05/TMA/TMEM kernels and requires sm_100;
 * the fp32 path runs FFMA kernels (fp32 parity mode).
 */
#ifndef LORS_B200_H_
#define LORS_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LORS_ABI_VERSION 1

/* Status codes; the Python wrapper maps them to the reference's error
 * vocabulary (errors.py): 1 -> ShapeError, 2 -> ArgumentError,
 * 3/4 -> RuntimeError. */
typedef enum {
  LORS_OK = 0,
  LORS_ERR_SHAPE = 1,
  LORS_ERR_ARGUMENT = 2,
  LORS_ERR_DEVICE = 3, /* not an sm_100 device */
  LORS_ERR_CUDA = 4    /* launch / CUDA runtime error */
} lors_status_t;

typedef enum { LORS_DTYPE_F32 = 0, LORS_DTYPE_BF16 = 1 } lors_dtype_t;

/* Where the mask M comes from.  FROM_W derives M = (W != 0) in registers from
 * the staged W tile (the reference semantics, 0 extra bytes).  BITS reads a
 * packed mask [R, ceil(C/32)] uint32 (bit j of word k = column 32k+j). */
typedef enum { LORS_MASK_FROM_W = 0, LORS_MASK_BITS = 1 } lors_mask_mode_t;

/* Adapter-gradient semantics.  STE = the reference `lors`
 * (no mask on dA/dB); MASKED = sqft_gc's G = (dY^T X) (.) M contraction. */
typedef enum { LORS_GRAD_STE = 0, LORS_GRAD_MASKED = 1 } lors_grad_mode_t;

#define LORS_FLAG_EMIT_P (1u << 0)   /* forward also writes P = X_t b^T [L, r] */
#define LORS_FLAG_SPARSE24 (1u << 1) /* forward on 2:4 sparse tensor cores: each
                                        masked W_eff tile is compressed on chip
                                        (W must be 2:4 along C; bf16; C % 64 == 0) */
#define LORS_FLAG_NO_DX (1u << 2)    /* backward skips dX (first layer)        */
#define LORS_FLAG_DX_ONLY (1u << 3)  /* backward computes dX only (da, db,     */
                                     /* dbias may be NULL; workspace only for   */
                                     /* the dX GEMM's tail split) -- the caller */
                                     /* runs the rank-r part separately, e.g.   */
                                     /* on a second stream, with NO_DX          */
#define LORS_FLAG_ZEROED (1u << 4)   /* backward: dA and dB are zero on entry   */
                                     /* (one fill of a joint buffer by the      */
                                     /* caller replaces the library's two       */
                                     /* zeroing launches); ignored elsewhere    */
#define LORS_FLAG_DETERMINISTIC (1u << 5) /* backward: dA / dB (and P, Q) through split
                                        partials summed in a fixed order -- no
                                        atomics or TMA reduce-adds -- so they are
                                        bitwise reproducible run to run (the
                                        reference replays training bitwise,
                                        test_train.py:169-178); needs the larger
                                        workspace lors_bwd_workspace reports */
#define LORS_FLAG_NO_TAIL_SPLIT (1u << 6) /* forward / dX GEMMs: walk every tile whole,
                                        without the tail split along K (the split
                                        fills the last round's idle SMs: faster for
                                        a GEMM timed alone, 0.3-0.8% slower in a
                                        sustained, power-capped training step, where
                                        idle SMs leave their power to the busy ones);
                                        its workspace is then not needed */
#define LORS_FLAG_FAULT_DA_SIGN (1u << 30) /* negative control: flip dA sign,
                                              mirrors FAULT_INJECTION
                                              "lors_backward_sign_flip"
                                              adapters.py:57-60,400-401 */

typedef struct lors_fwd_args {
  int64_t L, R, C, r;
  int32_t dtype;     /* lors_dtype_t: x, w, a, b, bias, y, p share it  */
  int32_t mask_mode; /* lors_mask_mode_t                               */
  uint32_t flags;
  float alpha;       /* > 0, reference default 2.0 (adapters.py:69)    */
  const void* x;     /* [L, C]                                         */
  const void* w;     /* [R, C] frozen pruned weight                    */
  const uint32_t* mask_bits; /* [R, ceil(C/32)] when mask_mode == BITS */
  const void* w24;   /* reserved (pre-compressed 2:4 values), unused   */
  const uint8_t* meta24; /* SPARSE24 only, optional: [R, C/8] index     */
                     /* nibbles of W from lors_compress_24 (built once; */
                     /* NULL = derived on chip from every W tile)       */
  const void* a;     /* [R, r]                                         */
  const void* b;     /* [r, C]                                         */
  const void* bias;  /* [R] or NULL                                    */
  void* y;           /* [L, R] out                                     */
  void* p;           /* [L, r] out when LORS_FLAG_EMIT_P               */
  void* workspace;
  size_t workspace_bytes;
} lors_fwd_args;

typedef struct lors_bwd_args {
  int64_t L, R, C, r;
  int32_t dtype;
  int32_t mask_mode;
  int32_t grad_mode; /* lors_grad_mode_t                                */
  uint32_t flags;
  float alpha;
  const void* x;     /* [L, C] saved input (the only saved activation)  */
  const void* w;     /* [R, C]                                          */
  const uint32_t* mask_bits;
  const void* a;     /* [R, r] adapter as it is at backward time (b2)   */
  const void* b;     /* [r, C]                                          */
  const void* dy;    /* [L, R]                                          */
  const void* p;     /* [L, r] saved P = X_t b^T, or NULL (recomputed)  */
  void* dx;          /* [L, C] out (dtype), skipped with FLAG_NO_DX     */
  float* da;         /* [R, r] out, fp32                                */
  float* db;         /* [r, C] out, fp32                                */
  float* dbias;      /* [R] out fp32, or NULL                           */
  void* workspace;
  size_t workspace_bytes;
} lors_bwd_args;

/* Forward: Y_t = X_t . W_eff^T (+ bias), W_eff = select(M, W + alpha a b, +0)
 * built tile by tile on chip and never written to HBM. */
int lors_fwd(const lors_fwd_args* args, void* stream);
/* Bytes of device workspace lors_fwd can use (0 = none): fp32 partials and
 * counters of the persistent walk's tail split along K.  A call given less
 * (or NULL) runs without the split; results differ only in fp32 summation order.
 * A workspace (forward or backward) belongs to one call at a time: calls that
 * may run concurrently (different streams) need separate workspaces. */
size_t lors_fwd_workspace(const lors_fwd_args* args);

/* Grouped forward (beyond the reference's per-layer call, which a host loops over
 * its projections, adapters.py:359-373): `groups` projections of the same input x
 * -- q / k / v, gate / up -- as ONE persistent tensor-core launch.  args describes
 * one projection (R rows each) and points at consecutive storage for all of them:
 * w [groups * R, C], a [groups * R, r], b [groups * r, C], y [groups][L][R].
 * Needs bf16, mask_mode FROM_W, no bias, no SPARSE24 / EMIT_P, R % 256 == 0,
 * C % 8 == 0 and r in {16, 32, 64} (LORS_ERR_ARGUMENT otherwise).  Each y[g] is
 * bit-identical to lors_fwd of projection g. */
int lors_fwd_group(const lors_fwd_args* args, int32_t groups, void* stream);
size_t lors_fwd_group_workspace(const lors_fwd_args* args, int32_t groups);

/* Backward: dX_t = dY_t . W_eff (recomputed tiles); STE: dA = alpha dY^T P,
 * dB = alpha Q^T X (P = X b^T, Q = dY a); MASKED: G = (dY^T X) (.) M never
 * materialised, dA = alpha G b^T, dB = alpha a^T G; dbias = sum_L dY. */
int lors_bwd(const lors_bwd_args* args, void* stream);
size_t lors_bwd_workspace(const lors_bwd_args* args);

/* W_eff (or merge() result) into out [R, C] in `dtype`: select(M, W + alpha a b, +0)
 * with one fp32 fma per element and one rounding to `dtype`.  bf16 on tensor-core
 * shapes runs the forward GEMM's own prologue (the same rank-r recompute MMA and
 * the same weff_pair) with each tile TMA-stored instead of multiplied, so the
 * result is bit-identical to the W_eff the forward and dX GEMMs consume
 * (tests/test_weff_identity.py); fp32 and other shapes run the FFMA kernels'
 * shared weff_value.  +0.0 bit pattern wherever M = 0. */
int lors_effective_weight(int64_t R, int64_t C, int64_t r, int32_t dtype,
                          int32_t mask_mode, float alpha, const void* w,
                          const uint32_t* mask_bits, const void* a,
                          const void* b, void* out, void* stream);

/* Packed mask bits [R, ceil(C/32)] uint32 from W != 0. */
int lors_pack_mask(int64_t R, int64_t C, int32_t dtype, const void* w,
                   uint32_t* bits, void* stream);

/* 2:4 compression: values [R, C/2] (dtype) and metadata [R, C/8] bytes, one
 * byte per 2 groups: group g's nibble = idx0 | idx1 << 2 (idx0 < idx1, the
 * kept positions inside the group).  *invalid (device int, may be NULL) is
 * set to 1 when a group holds more than 2 nonzeros (prune.py:72-77). */
int lors_compress_24(int64_t R, int64_t C, int32_t dtype, const void* w,
                     void* values, uint8_t* meta, int32_t* invalid,
                     void* stream);

/* dW [R, C] fp32 = dY_t^T X_t, optionally (.) M (initialization.py:209-211). */
int lors_grad_outer(int64_t L, int64_t R, int64_t C, int32_t dtype,
                    int32_t masked, const void* dy, const void* x,
                    const void* w, float* dw, void* stream);

/* Thread-local message for the last non-OK status of this thread. */
const char* lors_last_error(void);
int lors_abi_version(void);
/* LORS_OK when the current device is sm_100, else LORS_ERR_DEVICE. */
int lors_device_check(void);
/* Number of kernels this thread launched through the library (counter the
 * bench uses for its gpu_launches claim); reset with lors_reset_launch_count. */
uint64_t lors_launch_count(void);
void lors_reset_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* LORS_B200_H_ */
