"""torch.autograd.Function / nn.Module form of the LoRS linear.

Mirrors the paper's PyTorch listing `forward_lors` / `backward_lors`
(/root/reference/PAPER.md:481-510): `lora_A` is the reference `a` [out, r],
`lora_B` is `b` [r, in]; backward returns
(grad_x, None, grad_bias, grad_A, grad_B, None).  Differences by design:
the merged weight is never materialised (the native kernels rebuild W_eff
tiles on chip), and only X is saved for backward (the paper listing saves
x, weight, lora_A, lora_B; the reference package saves X only,
adapters.py:372).
"""

from __future__ import annotations

import contextlib
import math
import os
from dataclasses import dataclass
from typing import Optional

import torch
from torch import nn

from . import ops
from .errors import ArgumentError, ShapeError


@dataclass
class LoRSParams:
    alpha: float = 2.0            # scaling_factor (adapters.py:69)
    grad_mode: str = "ste"        # "ste" = lors (adapters.py:376-406); "masked" = sqft_gc (:303-312)
    mask_bits: Optional[torch.Tensor] = None
    save_p: bool = False          # keep P = X b^T (rL elements, dense-LoRA footprint)
    fault_da_sign: bool = False   # negative control (adapters.py:57-60)
    sparse24: bool = False        # forward on 2:4 sparse tensor cores (north_star 4)
    meta24: Optional[torch.Tensor] = None  # kept-position metadata of the frozen 2:4 weight
    check_finite: bool = False    # raise NumericError on NaN / inf outputs (one host sync per call)


def compute_copy(t: torch.Tensor, dt: torch.dtype) -> torch.Tensor:
    """`t` (an fp32 adapter master) in the compute dtype, contiguous.  When the
    fused optimizer (trainer.FlatAdamW) maintains a compute copy next to the
    master and the master is unchanged since (same version counter), that copy
    is returned instead of casting."""
    sh = getattr(t, "_lors_shadow", None)
    if sh is not None and sh.dtype == dt and getattr(t, "_lors_shadow_version", None) == t._version:
        return sh
    src = t.detach()
    return src if src.dtype == dt and src.is_contiguous() else src.to(dt).contiguous()


def grad_slots(lora_A, lora_B):
    """(dA, dB) destinations inside the optimizer's flat fp32 gradient buffer (trainer.FlatAdamW sets
    `_lors_grad_base` = (buffer, offset) on each adapter and keeps the buffer zeroed between steps), or
    (None, None).  Used only while both adapters hold no gradient: the views become .grad as they are
    (fresh view objects, so autograd takes them without a copy), which saves the per-layer fp32
    gradient buffers, their zero fills and the optimizer's concatenation."""
    ga, gb = getattr(lora_A, "_lors_grad_base", None), getattr(lora_B, "_lors_grad_base", None)
    if ga is None or gb is None or lora_A.grad is not None or lora_B.grad is not None:
        return None, None
    (buf_a, off_a), (buf_b, off_b) = ga, gb
    return (buf_a[off_a:off_a + lora_A.numel()].view(lora_A.shape),
            buf_b[off_b:off_b + lora_B.numel()].view(lora_B.shape))


class LoRSFunction(torch.autograd.Function):
    """y = x (W + alpha a b . M)^T + bias over x [..., in]."""

    @staticmethod
    def forward(ctx, x, weight, bias, lora_A, lora_B, params: LoRSParams):
        out_f, in_f = weight.shape
        if x.shape[-1] != in_f:
            raise ShapeError(f"layer expects {in_f} input features, got {x.shape[-1]}")
        dt = weight.dtype
        shape = x.shape
        x2 = x.reshape(-1, in_f)
        if x2.dtype != dt:
            x2 = x2.to(dt)
        x2 = x2.contiguous()
        a = compute_copy(lora_A, dt)
        b = compute_copy(lora_B, dt)
        bias_c = None if bias is None else bias.detach().to(dt).contiguous()
        y, p = ops.lors_fwd(x2, weight, a, b, params.alpha, bias_c, params.mask_bits, emit_p=params.save_p,
                            sparse24=params.sparse24, meta24=params.meta24 if params.sparse24 else None)
        if params.check_finite:
            ops.require_finite("LoRS forward output", y)
        if params.save_p:
            ctx.save_for_backward(x2, p)
        else:
            ctx.save_for_backward(x2)
        # adapter read at backward time (reference b2, adapters.py:387-394)
        ctx.lors = (weight, lora_A, lora_B, None if bias is None else bias.dtype, params, shape, x.dtype)
        return y.view(*shape[:-1], out_f)

    @staticmethod
    def backward(ctx, grad_y):
        weight, lora_A, lora_B, bias_dtype, params, x_shape, x_dtype = ctx.lors
        has_bias = bias_dtype is not None
        saved = ctx.saved_tensors
        x2 = saved[0]
        p = saved[1] if len(saved) > 1 else None
        out_f, in_f = weight.shape
        dt = weight.dtype
        dy = grad_y.reshape(-1, out_f)
        if dy.dtype != dt:
            dy = dy.to(dt)
        dy = dy.contiguous()
        # adapter read at backward time (a fresh compute-dtype copy: holding the
        # forward's copies until the backward would cost r(R + C) elements per layer
        # of peak memory, above the dense-LoRA bar)
        a = compute_copy(lora_A, dt)
        b = compute_copy(lora_B, dt)
        need_dx = ctx.needs_input_grad[0]
        da_out, db_out = grad_slots(lora_A, lora_B) if ctx.needs_input_grad[3] and ctx.needs_input_grad[4] \
            else (None, None)
        dx, da, db, dbias = ops.lors_bwd(x2, weight, a, b, dy, params.alpha, p=p, mask_bits=params.mask_bits,
                                         grad_mode=params.grad_mode, need_dx=need_dx, with_bias=has_bias,
                                         fault_da_sign=params.fault_da_sign, da_out=da_out, db_out=db_out)
        del da_out, db_out
        if params.check_finite:
            ops.require_finite("LoRS backward gradients", dx, da, db, dbias)
        grad_x = dx.view(x_shape).to(x_dtype) if need_dx else None
        grad_bias = dbias.to(bias_dtype) if has_bias and ctx.needs_input_grad[2] else None
        grad_a = da.to(lora_A.dtype) if ctx.needs_input_grad[3] else None
        grad_b = db.to(lora_B.dtype) if ctx.needs_input_grad[4] else None
        return grad_x, None, grad_bias, grad_a, grad_b, None


class LoRSGroupFunction(torch.autograd.Function):
    """Several LoRS projections of one input (q / k / v, gate / up) as one autograd
    node.  Forward: the GEMMs run on concurrent high-priority streams, so the CTA
    pairs a GEMM leaves idle in its last, partial round start the next GEMM's tiles
    (a persistent kernel's pairs exit as their static tile lists end, lowest pair
    index = most tiles first).  Backward: the dX GEMMs run the same way, the
    rank-r products of every projection on a normal-priority stream, and the
    input gradient is their sum (one add per extra projection, in projection order).
    Per projection the arithmetic is LoRSFunction's (lors_forward / lors_backward,
    adapters.py:359-406)."""

    @staticmethod
    def forward(ctx, x, params_list, *tensors):
        n = len(params_list)
        weights, biases, As, Bs = tensors[0::4], tensors[1::4], tensors[2::4], tensors[3::4]
        in_f = weights[0].shape[1]
        dt = weights[0].dtype
        if x.shape[-1] != in_f:
            raise ShapeError(f"layer expects {in_f} input features, got {x.shape[-1]}")
        shape = x.shape
        x2 = x.reshape(-1, in_f)
        if x2.dtype != dt:
            x2 = x2.to(dt)
        x2 = x2.contiguous()
        dev = x2.device
        # every main-stream producer (casts, compute copies) is enqueued before the fork
        ab = [(compute_copy(As[i], dt), compute_copy(Bs[i], dt)) for i in range(n)]
        bc = [None if biases[i] is None else biases[i].detach().to(dt).contiguous() for i in range(n)]
        main = torch.cuda.current_stream(dev)
        w_cat = packed_weights(weights, biases, As, params_list)
        keep, outs, streams = [], [], ()
        if w_cat is not None:
            # one persistent launch over every projection's tiles (lors_fwd_group), on the main
            # stream; outputs bit-identical to the per-projection launches
            a_cat = torch.cat([ab[i][0] for i in range(n)])
            b_cat = torch.cat([ab[i][1] for i in range(n)])
            y = ops.lors_fwd_group(x2, w_cat, a_cat, b_cat, n, params_list[0].alpha)
            outs = [y[i].view(*shape[:-1], weights[i].shape[0]) for i in range(n)]
        else:
            streams, _ = ops.group_streams(dev, n)
            streams = streams[:n]
            fork = torch.cuda.Event()
            fork.record(main)
            for i, prm in enumerate(params_list):
                streams[i].wait_event(fork)
                y, _ = ops.lors_fwd(x2, weights[i], ab[i][0], ab[i][1], prm.alpha, bc[i], prm.mask_bits,
                                    sparse24=prm.sparse24, meta24=prm.meta24 if prm.sparse24 else None,
                                    launch_stream=streams[i], keep=keep)
                outs.append(y.view(*shape[:-1], weights[i].shape[0]))
        for st in streams:
            ev = torch.cuda.Event()
            ev.record(st)
            main.wait_event(ev)
        # keep / ab / bc were allocated on the main stream and are released after the
        # joins are enqueued there, so no later main-stream reuse can overtake the GEMMs
        ctx.save_for_backward(x2)
        if any(prm.check_finite for prm in params_list):
            ops.require_finite("LoRS forward outputs", *outs)
        ctx.lors = (weights, As, Bs, tuple(None if b is None else b.dtype for b in biases), params_list, shape,
                    x.dtype)
        return tuple(outs)

    @staticmethod
    def backward(ctx, *grads):
        weights, As, Bs, bias_dtypes, params_list, x_shape, x_dtype = ctx.lors
        has_bias = tuple(d is not None for d in bias_dtypes)
        (x2,) = ctx.saved_tensors
        n = len(params_list)
        dt = weights[0].dtype
        dev = x2.device
        dys = []
        for i, g in enumerate(grads):
            dy = g.reshape(-1, weights[i].shape[0])
            dys.append((dy if dy.dtype == dt else dy.to(dt)).contiguous())
        ab = [(compute_copy(As[i], dt), compute_copy(Bs[i], dt)) for i in range(n)]   # read at backward time
        need_dx = ctx.needs_input_grad[0]
        main = torch.cuda.current_stream(dev)
        # rank-r products of each projection on their own normal-priority stream (LORS_GROUP_SIDE=1:
        # one shared stream), so the small HBM-bound kernels of different projections overlap
        n_side = 1 if os.environ.get("LORS_GROUP_SIDE", "n") == "1" else n
        streams, sides = ops.group_streams(dev, n, n_side)
        sides = sides if isinstance(sides, list) else [sides]
        fork = torch.cuda.Event()
        fork.record(main)
        for sd in sides:
            sd.wait_event(fork)
        dxs, res, keep = [], [], []
        for i, prm in enumerate(params_list):
            if need_dx:
                streams[i].wait_event(fork)
                dx, _, _, _, ws = ops._lors_bwd_call(x2, weights[i], ab[i][0], ab[i][1], dys[i], prm.alpha, None,
                                                     prm.mask_bits, prm.grad_mode, True, False, False,
                                                     dx_only=True, launch_stream=streams[i])
                dxs.append(dx)
                keep.append(ws)
            k = 2 + 4 * i
            da_out, db_out = grad_slots(As[i], Bs[i]) if ctx.needs_input_grad[k + 2] and ctx.needs_input_grad[k + 3] \
                else (None, None)
            _, da, db, dbias, ws = ops._lors_bwd_call(x2, weights[i], ab[i][0], ab[i][1], dys[i], prm.alpha, None,
                                                      prm.mask_bits, prm.grad_mode, False, has_bias[i],
                                                      prm.fault_da_sign, launch_stream=sides[i % len(sides)],
                                                      deterministic=ops.deterministic_default(),
                                                      da_out=da_out, db_out=db_out)
            del da_out, db_out
            res.append((da, db, dbias))
            keep.append(ws)
        for st in (streams if need_dx else []) + sides:
            ev = torch.cuda.Event()
            ev.record(st)
            main.wait_event(ev)
        grad_x = None
        if need_dx:
            if len(dxs) > 1 and dxs[0].dtype == torch.bfloat16 and dxs[0].numel() % 8 == 0:
                dx = ops.sum_into(dxs)            # one fp32 pass over the projections' dX
            else:
                dx = dxs[0]
                for d in dxs[1:]:
                    dx.add_(d)
            grad_x = dx.view(x_shape).to(x_dtype)
        if any(prm.check_finite for prm in params_list):
            ops.require_finite("LoRS backward gradients", grad_x, *[t for r3 in res for t in r3])
        out = [grad_x, None]
        for i in range(n):
            da, db, dbias = res[i]
            k = 2 + 4 * i
            out += [None,
                    dbias.to(bias_dtypes[i]) if has_bias[i] and ctx.needs_input_grad[k + 1] else None,
                    da.to(As[i].dtype) if ctx.needs_input_grad[k + 2] else None,
                    db.to(Bs[i].dtype) if ctx.needs_input_grad[k + 3] else None]
        return tuple(out)


_GROUPING = [True]


@contextlib.contextmanager
def no_grouping():
    """Run every projection as its own LoRSLinear call (init_gradient_svd's probe needs each
    layer's forward hook to fire)."""
    prev = _GROUPING[0]
    _GROUPING[0] = False
    try:
        yield
    finally:
        _GROUPING[0] = prev


def packed_weights(weights, biases, As, params_list) -> Optional[torch.Tensor]:
    """[G R, C] storage holding `weights` back to back (pack_group_weights) when the projections
    can run as one grouped launch (lors_fwd_group: bf16, masks from W, no bias / 2:4, equal alpha,
    R % 256 == 0, r in {16, 32, 64}), else None."""
    if os.environ.get("LORS_GROUP_FWD", "1") == "0":
        return None
    w0 = weights[0]
    base = w0._base
    n = len(weights)
    R, C = w0.shape
    r = As[0].shape[1]
    if (base is None or w0.dtype != torch.bfloat16 or R % 256 or r not in (16, 32, 64) or C % 8
            or tuple(base.shape) != (n * R, C) or not base.is_contiguous()):
        return None
    for i, (w, bias, a, prm) in enumerate(zip(weights, biases, As, params_list)):
        if (w._base is not base or tuple(w.shape) != (R, C) or w.data_ptr() != base.data_ptr() + i * R * C * 2
                or bias is not None or a.shape[1] != r or prm.mask_bits is not None or prm.sparse24
                or prm.alpha != params_list[0].alpha):
            return None
    return base


def pack_group_weights(layers) -> bool:
    """Move the frozen weights of `layers` (projections of one input with equal shapes) into one
    [G R, C] buffer, each layer's `weight` becoming its row slice, so LoRSGroupFunction can run
    them as one grouped launch.  Values, shapes and state_dict names are unchanged."""
    ws = [m.weight for m in layers]
    if len(ws) < 2 or any(tuple(w.shape) != tuple(ws[0].shape) or w.dtype != ws[0].dtype or w.device != ws[0].device
                          for w in ws):
        return False
    buf = torch.cat(ws)
    R = ws[0].shape[0]
    for i, m in enumerate(layers):
        m._buffers["weight"] = buf[i * R:(i + 1) * R]
    return True


def groupable(layers) -> bool:
    """Whether `layers` can run as one LoRSGroupFunction node: LoRSLinear projections
    of the same input on a CUDA device in bf16 (the tensor-core path), without the
    options that change the saved set (save_p)."""
    if len(layers) < 2 or not _GROUPING[0] or os.environ.get("LORS_GROUP", "1") == "0":
        return False
    w0 = getattr(layers[0], "weight", None)
    return all(isinstance(m, LoRSLinear) and m.weight.is_cuda and m.weight.dtype == torch.bfloat16
               and m.weight.shape[1] == w0.shape[1] and not m.save_p for m in layers)


def lors_group(layers, x: torch.Tensor):
    """Outputs of several LoRS projections of the same `x` (see LoRSGroupFunction)."""
    tensors = []
    for m in layers:
        tensors += [m.weight, m.bias, m.a, m.b]
    return LoRSGroupFunction.apply(x, tuple(m.params() for m in layers), *tensors)


class LoRSLinear(nn.Module):
    """Sparsity-preserving LoRA linear: frozen pruned `weight`, trainable `a`, `b`.

    Constructor follows the reference contract (make_layer / AdaptedLayer,
    adapters.py:114-176): `weight` (the pruned base; zeros are the mask),
    `rank` (zero-initialised a and b, as make_layer) or explicit `a`/`b`,
    `alpha=2.0`, `bias=None`, `name`.  state_dict: `weight` (frozen buffer),
    `a`, `b` (fp32 master parameters), `bias`, and `mask` (packed bits) when
    mask_mode == "bits".  The compute dtype is weight.dtype (float32 = FFMA
    parity mode, bfloat16 = tcgen05 mode).
    """

    def __init__(self, weight: torch.Tensor, rank: Optional[int] = None, a: Optional[torch.Tensor] = None,
                 b: Optional[torch.Tensor] = None, alpha: float = 2.0, bias: Optional[torch.Tensor] = None,
                 name: str = "", grad_mode: str = "ste", mask_mode: str = "from_w", save_p: bool = False,
                 param_dtype: torch.dtype = torch.float32, sparse24: bool = False, check_finite: bool = False):
        super().__init__()
        if weight.dim() != 2:
            raise ShapeError("weight must be 2-D [out, in]")
        R, C = weight.shape
        if (a is None) != (b is None):
            raise ArgumentError("give both a and b, or neither")
        if a is None:
            if rank is None:
                raise ArgumentError("need rank or a/b")
            a = torch.zeros(R, rank, dtype=param_dtype, device=weight.device)
            b = torch.zeros(rank, C, dtype=param_dtype, device=weight.device)
        if a.shape[1] != b.shape[0]:
            raise ShapeError(f"adapter rank mismatch: a is {a.shape[0]}x{a.shape[1]}, b is {b.shape[0]}x{b.shape[1]}")
        r = a.shape[1]
        if r < 1 or r > min(R, C):
            raise ArgumentError(f"rank {r} must satisfy 1 <= r <= min({R}, {C})")
        if a.shape[0] != R:
            raise ShapeError(f"adapter a has {a.shape[0]} rows, base has {R}")
        if b.shape[1] != C:
            raise ShapeError(f"adapter b has {b.shape[1]} cols, base has {C}")
        if not alpha > 0:
            raise ArgumentError(f"alpha must be positive, got {alpha}")
        if grad_mode not in ("ste", "masked"):
            raise ArgumentError(f"grad_mode must be 'ste' or 'masked', got {grad_mode!r}")
        if mask_mode not in ("from_w", "bits"):
            raise ArgumentError(f"mask_mode must be 'from_w' or 'bits', got {mask_mode!r}")
        w = weight.detach()
        w = torch.where(w == 0, torch.zeros_like(w), w).contiguous()  # -0.0 -> +0.0 (prune.py:47)
        if sparse24:
            from .prune import two_four_valid
            if w.dtype != torch.bfloat16 or C % 64 or not two_four_valid(w):
                raise ArgumentError("sparse24 needs a bf16 weight that is 2:4 along the input axis, in % 64 == 0")
        self.sparse24 = sparse24
        self.register_buffer("weight", w)
        # 2:4 index nibbles of the frozen weight ([R, C/8] u8, 1/16 of W's bytes),
        # built once here (lors_compress_24) and read by the sparse forward
        self.register_buffer("meta24", ops.compress_24(w)[1] if sparse24 else None, persistent=False)
        self.a = nn.Parameter(a.detach().clone())
        self.b = nn.Parameter(b.detach().clone())
        self.bias = None if bias is None else nn.Parameter(bias.detach().clone().reshape(R))
        if mask_mode == "bits":
            self.register_buffer("mask", ops.pack_mask(w))
        else:
            self.mask = None
        self.alpha = float(alpha)
        self.name = name
        self.grad_mode = grad_mode
        self.save_p = save_p
        self.fault_da_sign = False
        self.check_finite = check_finite   # NumericError on NaN / inf (matrix.py:53-54), one host sync per call

    @property
    def in_features(self) -> int:
        return self.weight.shape[1]

    @property
    def out_features(self) -> int:
        return self.weight.shape[0]

    @property
    def rank(self) -> int:
        return self.a.shape[1]

    def params(self) -> LoRSParams:
        return LoRSParams(alpha=self.alpha, grad_mode=self.grad_mode, mask_bits=self.mask,
                          save_p=self.save_p, fault_da_sign=self.fault_da_sign, sparse24=self.sparse24,
                          meta24=self.meta24, check_finite=self.check_finite)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return LoRSFunction.apply(x, self.weight, self.bias, self.a, self.b, self.params())

    @torch.no_grad()
    def effective_weight(self) -> torch.Tensor:
        """W_eff through the kernels' prologue function (bit-exact +0 where M = 0)."""
        dt = self.weight.dtype
        return ops.effective_weight(self.weight, self.a.to(dt).contiguous(), self.b.to(dt).contiguous(),
                                    self.alpha, self.mask)

    @torch.no_grad()
    def merge(self) -> torch.Tensor:
        """merge() (adapters.py:709-727): the finalised sparse weight."""
        return self.effective_weight()

    def extra_repr(self) -> str:
        return (f"in={self.in_features}, out={self.out_features}, r={self.rank}, alpha={self.alpha}, "
                f"grad_mode={self.grad_mode}, dtype={self.weight.dtype}")

    @staticmethod
    def init_normal(a_std: float, b_std: float, R: int, C: int, r: int, generator=None, device="cuda"):
        """BASELINE config-1 init in reference names: b ~ N(0, b_std^2) (north_star A),
        a ~ N(0, a_std^2) (north_star B); SURVEY C2."""
        a = torch.randn(R, r, generator=generator, device=device) * a_std
        b = torch.randn(r, C, generator=generator, device=device) * b_std
        return a, b


def default_b_std(r: int) -> float:
    return 1.0 / math.sqrt(r)
