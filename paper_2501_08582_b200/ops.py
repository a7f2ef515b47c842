"""Torch-tensor wrappers over the C ABI (torch layout: tokens are rows).

PyTorch is plumbing here: it owns device memory and the current stream; the
work happens in the native library.  Every function validates shapes with
the reference's messages (adapters.py:227-238) and raises ShapeError /
ArgumentError; nothing falls back to torch math.
"""

from __future__ import annotations

import ctypes as ct
import os
from typing import Optional

import torch

from . import _native as N
from .errors import ArgumentError, NumericError, ShapeError

_DTYPES = {torch.float32: N.DTYPE_F32, torch.bfloat16: N.DTYPE_BF16}


def dtype_code(dt: torch.dtype) -> int:
    if dt not in _DTYPES:
        raise ArgumentError(f"unsupported dtype {dt}; expected float32 or bfloat16")
    return _DTYPES[dt]


def _p(t: Optional[torch.Tensor]):
    return None if t is None else ct.c_void_p(t.data_ptr())


def _stream() -> ct.c_void_p:
    return ct.c_void_p(torch.cuda.current_stream().cuda_stream)


def _need(t: torch.Tensor, name: str, shape, dtype=None):
    if tuple(t.shape) != tuple(shape):
        raise ShapeError(f"{name} must be {'x'.join(map(str, shape))}, got {'x'.join(map(str, t.shape))}")
    if dtype is not None and t.dtype != dtype:
        raise ArgumentError(f"{name} has dtype {t.dtype}, expected {dtype}")
    if not t.is_cuda:
        raise ArgumentError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if not t.is_contiguous():
        raise ArgumentError(f"{name} must be contiguous")


def _check_layer(x_t, w, a, b):
    if w.dim() != 2 or a.dim() != 2 or b.dim() != 2 or x_t.dim() != 2:
        raise ShapeError("x_t, w, a, b must be 2-D")
    R, C = w.shape
    if a.shape[1] != b.shape[0]:
        raise ShapeError(f"adapter rank mismatch: a is {a.shape[0]}x{a.shape[1]}, b is {b.shape[0]}x{b.shape[1]}")
    if a.shape[0] != R:
        raise ShapeError(f"adapter a has {a.shape[0]} rows, base has {R}")
    if b.shape[1] != C:
        raise ShapeError(f"adapter b has {b.shape[1]} cols, base has {C}")
    if x_t.shape[1] != C:
        raise ShapeError(f"layer expects {C} input rows, got {x_t.shape[1]}x{x_t.shape[0]}")
    return x_t.shape[0], R, C, a.shape[1]


def require_finite(what: str, *tensors: Optional[torch.Tensor]) -> None:
    """Raise NumericError when any given tensor holds NaN or +-inf -- the reference checks
    every matrix result (matrix.py:44-45, 53-54).  One device reduction and one host read."""
    ts = [t for t in tensors if t is not None and t.numel()]
    if not ts:
        return
    ok = torch.stack([torch.isfinite(t).all() for t in ts]).all()
    if not bool(ok):
        raise NumericError(f"non-finite values in {what}")


def lors_fwd(x_t: torch.Tensor, w: torch.Tensor, a: torch.Tensor, b: torch.Tensor, alpha: float = 2.0,
             bias: Optional[torch.Tensor] = None, mask_bits: Optional[torch.Tensor] = None,
             emit_p: bool = False, sparse24: bool = False, meta24: Optional[torch.Tensor] = None,
             launch_stream=None, keep: Optional[list] = None):
    """Y_t [L, R] = X_t . W_eff^T (+ bias); optionally P = X_t b^T [L, r].

    Outputs and workspace come from the current stream's pool; `launch_stream`
    (default: the current stream) runs the kernels, in which case the caller must
    make the current stream wait for it before the outputs are used or freed and
    keep the workspace (appended to `keep`) alive until then.

    sparse24=True runs the forward on 2:4 sparse tensor cores: the kernel
    compresses each masked W_eff tile on chip (W must satisfy 2:4 along C,
    prune.py:72-77; bf16 only).  `meta24` ([R, C/8] uint8, the metadata of
    `compress_24(w)`, computed once per frozen weight) lets the kernel read the
    kept positions instead of deriving them from every W tile."""
    L, R, C, r = _check_layer(x_t, w, a, b)
    dt = w.dtype
    code = dtype_code(dt)
    for t, nm, sh in ((x_t, "x", (L, C)), (w, "w", (R, C)), (a, "a", (R, r)), (b, "b", (r, C))):
        _need(t, nm, sh, dt)
    if bias is not None:
        _need(bias, "bias", (R,), dt)
    if meta24 is not None:
        if not sparse24:
            raise ArgumentError("meta24 is only used by the 2:4 sparse forward (sparse24=True)")
        _need(meta24, "meta24", (R, C // 8), torch.uint8)
    y = torch.empty((L, R), dtype=dt, device=w.device)
    p = torch.empty((L, r), dtype=dt, device=w.device) if emit_p else None
    args = N.FwdArgs()
    args.L, args.R, args.C, args.r = L, R, C, r
    args.dtype = code
    args.mask_mode = N.MASK_BITS if mask_bits is not None else N.MASK_FROM_W
    args.flags = (N.FLAG_EMIT_P if emit_p else 0) | (N.FLAG_SPARSE24 if sparse24 else 0) | _split_flag()
    args.alpha = float(alpha)
    args.x, args.w, args.a, args.b = _p(x_t), _p(w), _p(a), _p(b)
    args.mask_bits = _p(mask_bits)
    args.meta24 = _p(meta24)
    args.bias, args.y, args.p = _p(bias), _p(y), _p(p)
    lib = N.load()
    ws_bytes = lib.lors_fwd_workspace(ct.byref(args))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=w.device) if ws_bytes else None
    args.workspace, args.workspace_bytes = _p(ws), ws_bytes
    if keep is not None and ws is not None:
        keep.append(ws)
    st = _stream() if launch_stream is None else ct.c_void_p(launch_stream.cuda_stream)
    N.check(lib.lors_fwd(ct.byref(args), st))
    return y, p


def lors_fwd_group(x_t: torch.Tensor, w: torch.Tensor, a: torch.Tensor, b: torch.Tensor, groups: int,
                   alpha: float = 2.0, launch_stream=None, keep: Optional[list] = None) -> torch.Tensor:
    """Y [G, L, R] of G projections of the same X_t in one launch (lors_fwd_group): w [G R, C],
    a [G R, r], b [G r, C] hold the projections consecutively (bf16, masks from W, no bias).
    Y[g] is bit-identical to lors_fwd(x_t, w[g R:(g+1) R], a[g R:(g+1) R], b[g r:(g+1) r])."""
    G = int(groups)
    if G < 1 or w.dim() != 2 or w.shape[0] % G or b.shape[0] % G:
        raise ShapeError(f"w {tuple(w.shape)} / b {tuple(b.shape)} do not split into {groups} projections")
    R, C, r = w.shape[0] // G, w.shape[1], b.shape[0] // G
    L = x_t.shape[0]
    dt = w.dtype
    for t, nm, sh in ((x_t, "x", (L, C)), (w, "w", (G * R, C)), (a, "a", (G * R, r)), (b, "b", (G * r, C))):
        _need(t, nm, sh, dt)
    y = torch.empty((G, L, R), dtype=dt, device=w.device)
    args = N.FwdArgs()
    args.L, args.R, args.C, args.r = L, R, C, r
    args.dtype = dtype_code(dt)
    args.mask_mode = N.MASK_FROM_W
    args.flags = _split_flag()
    args.alpha = float(alpha)
    args.x, args.w, args.a, args.b, args.y = _p(x_t), _p(w), _p(a), _p(b), _p(y)
    lib = N.load()
    ws_bytes = lib.lors_fwd_group_workspace(ct.byref(args), G)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=w.device) if ws_bytes else None
    args.workspace, args.workspace_bytes = _p(ws), ws_bytes
    if keep is not None and ws is not None:
        keep.append(ws)
    st = _stream() if launch_stream is None else ct.c_void_p(launch_stream.cuda_stream)
    N.check(lib.lors_fwd_group(ct.byref(args), G, st))
    return y


_GROUP_STREAMS = {}


def group_streams(dev: torch.device, n: int, n_side: int = 1):
    """n high-priority streams (one per concurrent LoRS GEMM) and `n_side` normal-priority
    streams for the rank-r products (a list when n_side > 1), created once per device."""
    pool = _GROUP_STREAMS.get(dev.index)
    if pool is None or len(pool[0]) < n or len(pool[1]) < n_side:
        lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
        pool = ([torch.cuda.Stream(device=dev, priority=hi) for _ in range(max(n, 3))],
                [torch.cuda.Stream(device=dev) for _ in range(max(n_side, 3))])
        _GROUP_STREAMS[dev.index] = pool
    return pool[0][:n], (pool[1][:n_side] if n_side > 1 else pool[1][0])


_SIDE_STREAMS = {}


def _side_stream(dev: torch.device):
    """(high-priority stream for dX, normal stream for the rank-r part, fork event,
    two join events) for `dev`, created once and reused.  The priority makes the
    persistent dX kernel's CTAs win the SMs when both are ready; the rank-r
    kernels fill whatever it leaves idle."""
    s = _SIDE_STREAMS.get(dev.index)
    if s is None:
        lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
        s = (torch.cuda.Stream(device=dev, priority=hi), torch.cuda.Stream(device=dev),
             torch.cuda.Event(), torch.cuda.Event(), torch.cuda.Event())
        _SIDE_STREAMS[dev.index] = s
    return s


_TAIL_SPLIT = [True]


def set_tail_split(enabled: bool) -> bool:
    """Process-wide: whether the forward / dX GEMMs split their last round's tiles along K
    (LORS_FLAG_NO_TAIL_SPLIT when off).  The split helps a GEMM timed alone; a sustained,
    power-capped training step runs 0.3-0.8% faster without it (trainer.Trainer turns it off
    during its steps).  Returns the previous setting."""
    prev = _TAIL_SPLIT[0]
    _TAIL_SPLIT[0] = bool(enabled)
    return prev


def _split_flag() -> int:
    return 0 if _TAIL_SPLIT[0] else N.FLAG_NO_TAIL_SPLIT


def deterministic_default() -> bool:
    """Default of lors_bwd's `deterministic` (LORS_DETERMINISTIC=1 turns it on process-wide)."""
    return os.environ.get("LORS_DETERMINISTIC", "0") == "1"


def lors_bwd(x_t: torch.Tensor, w: torch.Tensor, a: torch.Tensor, b: torch.Tensor, dy_t: torch.Tensor,
             alpha: float = 2.0, p: Optional[torch.Tensor] = None, mask_bits: Optional[torch.Tensor] = None,
             grad_mode: str = "ste", need_dx: bool = True, with_bias: bool = False,
             fault_da_sign: bool = False, overlap: Optional[bool] = None, deterministic: Optional[bool] = None,
             da_out: Optional[torch.Tensor] = None, db_out: Optional[torch.Tensor] = None):
    """(dX_t [L, C] | None, dA [R, r] fp32, dB [r, C] fp32, dbias [R] fp32 | None).

    deterministic=True (LORS_FLAG_DETERMINISTIC): the adapter gradients' split-K
    partials are summed in a fixed order instead of by atomics / TMA reduce-adds,
    so dA and dB are bitwise reproducible run to run (default: LORS_DETERMINISTIC).

    overlap=True (bf16 tensor-core shapes): the dX GEMM is enqueued on the
    current stream and the rank-r products (P, Q, dA, dB) on a side stream, two
    C-ABI calls (LORS_FLAG_DX_ONLY / LORS_FLAG_NO_DX); the HBM-bound rank-r
    kernels then fill the SMs the persistent dX kernel leaves idle in its last
    round.  The current stream waits for both before returning."""
    if overlap is None:
        overlap = os.environ.get("LORS_BWD_OVERLAP", "1") != "0"
    if deterministic is None:
        deterministic = deterministic_default()
    R_, C_ = w.shape
    r_ = a.shape[1] if a.dim() == 2 else 0
    if (overlap and need_dx and w.is_cuda and w.dtype == torch.bfloat16 and R_ % 8 == 0 and C_ % 8 == 0
            and r_ % 8 == 0 and 0 < r_ <= 64 and x_t.dim() == 2 and x_t.shape[0] > 0):
        dev = w.device
        main = torch.cuda.current_stream(dev)
        hi, side, fork, join_hi, join = _side_stream(dev)
        fork.record(main)
        hi.wait_event(fork)
        side.wait_event(fork)
        # (the dX call's workspace -- tail-split partials -- is held until the joins below)
        dx, _, _, _, ws_dx = _lors_bwd_call(x_t, w, a, b, dy_t, alpha, p, mask_bits, grad_mode, True, False,
                                            fault_da_sign, dx_only=True, launch_stream=hi)
        # Every buffer comes from the current stream's pool, and the current stream
        # waits for both side streams before this call returns, so any later reuse
        # of these blocks is ordered after the side work: no record_stream (whose
        # deferred frees made the caching allocator grow with cudaMalloc stalls).
        _, da, db, dbias, ws = _lors_bwd_call(x_t, w, a, b, dy_t, alpha, p, mask_bits, grad_mode, False, with_bias,
                                              fault_da_sign, launch_stream=side, deterministic=deterministic,
                                              da_out=da_out, db_out=db_out)
        join_hi.record(hi)
        join.record(side)
        main.wait_event(join_hi)
        main.wait_event(join)
        return dx, da, db, dbias
    return _lors_bwd_call(x_t, w, a, b, dy_t, alpha, p, mask_bits, grad_mode, need_dx, with_bias,
                          fault_da_sign, deterministic=deterministic, da_out=da_out, db_out=db_out)[:4]


def _lors_bwd_call(x_t, w, a, b, dy_t, alpha, p, mask_bits, grad_mode, need_dx, with_bias, fault_da_sign,
                   dx_only: bool = False, launch_stream=None, deterministic: bool = False,
                   da_out: Optional[torch.Tensor] = None, db_out: Optional[torch.Tensor] = None):
    """One lors_bwd C-ABI call: outputs and workspace allocated on the current
    stream, the kernels launched on `launch_stream` (default: the current stream).
    da_out / db_out: zero-filled fp32 [R, r] / [r, C] destinations (views into an
    optimizer's flat gradient buffer) used by the tensor-core STE path instead of a
    fresh zeroed buffer.  Returns (dx, da, db, dbias, workspace)."""
    L, R, C, r = _check_layer(x_t, w, a, b)
    dt = w.dtype
    code = dtype_code(dt)
    if tuple(dy_t.shape) != (L, R):
        raise ShapeError(f"gradient must be {R}x{L}, got {dy_t.shape[1]}x{dy_t.shape[0]}")
    for t, nm, sh in ((x_t, "x", (L, C)), (w, "w", (R, C)), (a, "a", (R, r)), (b, "b", (r, C)),
                      (dy_t, "dy", (L, R))):
        _need(t, nm, sh, dt)
    if p is not None:
        _need(p, "p", (L, r), dt)
    if grad_mode not in ("ste", "masked"):
        raise ArgumentError(f"grad_mode must be 'ste' or 'masked', got {grad_mode!r}")
    dev = w.device
    dx = torch.empty((L, C), dtype=dt, device=dev) if need_dx else None
    # tensor-core STE path: dA and dB carved out of one zero-filled buffer -- one fill
    # kernel instead of the library's two memsets (the buffer is what the grads keep)
    zeroed = (not dx_only and dt == torch.bfloat16 and grad_mode == "ste" and L > 0 and R % 8 == 0
              and C % 8 == 0 and r % 8 == 0 and r <= 64)
    if zeroed:
        da_b, db_b = (R * r * 4 + 255) // 256 * 256, (r * C * 4 + 255) // 256 * 256
    da = None if dx_only or zeroed else torch.empty((R, r), dtype=torch.float32, device=dev)
    db = None if dx_only or zeroed else torch.empty((r, C), dtype=torch.float32, device=dev)
    dbias = torch.empty((R,), dtype=torch.float32, device=dev) if with_bias and not dx_only else None
    args = N.BwdArgs()
    args.L, args.R, args.C, args.r = L, R, C, r
    args.dtype = code
    args.mask_mode = N.MASK_BITS if mask_bits is not None else N.MASK_FROM_W
    args.grad_mode = N.GRAD_STE if grad_mode == "ste" else N.GRAD_MASKED
    args.flags = ((0 if need_dx else N.FLAG_NO_DX) | (N.FLAG_DX_ONLY if dx_only else 0)
                  | (N.FLAG_FAULT_DA_SIGN if fault_da_sign and not dx_only else 0)
                  | (N.FLAG_DETERMINISTIC if deterministic and not dx_only else 0) | _split_flag())
    args.alpha = float(alpha)
    args.x, args.w, args.mask_bits, args.a, args.b = _p(x_t), _p(w), _p(mask_bits), _p(a), _p(b)
    lib = N.load()
    ws_bytes = lib.lors_bwd_workspace(ct.byref(args))
    if zeroed:
        if (da_out is not None and db_out is not None and tuple(da_out.shape) == (R, r)
                and tuple(db_out.shape) == (r, C) and da_out.dtype == torch.float32
                and db_out.dtype == torch.float32 and da_out.is_contiguous() and db_out.is_contiguous()):
            da, db = da_out, db_out          # zero-filled by their owner (trainer.FlatAdamW.zero_grad)
        else:
            buf = torch.zeros(da_b + db_b, dtype=torch.uint8, device=dev)
            da = buf[:R * r * 4].view(torch.float32).view(R, r)
            db = buf[da_b:da_b + r * C * 4].view(torch.float32).view(r, C)
        args.flags |= N.FLAG_ZEROED
        if launch_stream is not None:
            # the fill ran on the current stream, after the caller's fork: order it
            # before the kernels on the launch stream
            filled = torch.cuda.Event()
            filled.record(torch.cuda.current_stream(dev))
            launch_stream.wait_event(filled)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev) if ws_bytes else None
    args.dy, args.p, args.dx, args.da, args.db, args.dbias = _p(dy_t), _p(p), _p(dx), _p(da), _p(db), _p(dbias)
    args.workspace, args.workspace_bytes = _p(ws), ws_bytes
    st = _stream() if launch_stream is None else ct.c_void_p(launch_stream.cuda_stream)
    N.check(lib.lors_bwd(ct.byref(args), st))
    return dx, da, db, dbias, ws


def effective_weight(w: torch.Tensor, a: torch.Tensor, b: torch.Tensor, alpha: float = 2.0,
                     mask_bits: Optional[torch.Tensor] = None) -> torch.Tensor:
    """W_eff = select(M, W + alpha a b, +0) [R, C] (merged_weight, adapters.py:214-224)."""
    R, C = w.shape
    r = a.shape[1]
    _check_layer(torch.empty((0, C), device="meta"), w, a, b)
    for t, nm, sh in ((w, "w", (R, C)), (a, "a", (R, r)), (b, "b", (r, C))):
        _need(t, nm, sh, w.dtype)
    out = torch.empty_like(w)
    N.check(N.load().lors_effective_weight(R, C, r, dtype_code(w.dtype),
                                           N.MASK_BITS if mask_bits is not None else N.MASK_FROM_W,
                                           float(alpha), _p(w), _p(mask_bits), _p(a), _p(b), _p(out),
                                           _stream()))
    return out


def pack_mask(w: torch.Tensor) -> torch.Tensor:
    """Packed mask [R, ceil(C/32)] (int32 storage of uint32 words), bit j of
    word k = (W[:, 32k+j] != 0)."""
    R, C = w.shape
    _need(w, "w", (R, C))
    bits = torch.empty((R, (C + 31) // 32), dtype=torch.int32, device=w.device)
    N.check(N.load().lors_pack_mask(R, C, dtype_code(w.dtype), _p(w), _p(bits), _stream()))
    return bits


def compress_24(w: torch.Tensor):
    """(values [R, C/2], meta [R, C/8] uint8, valid) for a 2:4 pruned W."""
    R, C = w.shape
    _need(w, "w", (R, C))
    vals = torch.empty((R, C // 2), dtype=w.dtype, device=w.device)
    meta = torch.empty((R, C // 8), dtype=torch.uint8, device=w.device)
    flag = torch.zeros((1,), dtype=torch.int32, device=w.device)
    N.check(N.load().lors_compress_24(R, C, dtype_code(w.dtype), _p(w), _p(vals), _p(meta), _p(flag),
                                      _stream()))
    return vals, meta, flag


def grad_outer(dy_t: torch.Tensor, x_t: torch.Tensor, w: Optional[torch.Tensor] = None,
               masked: bool = False) -> torch.Tensor:
    """dW [R, C] fp32 = dY_t^T X_t, optionally (.) (W != 0) (initialization.py:209-211)."""
    L, R = dy_t.shape
    C = x_t.shape[1]
    _need(dy_t, "dy", (L, R))
    _need(x_t, "x", (L, C), dy_t.dtype)
    if masked:
        if w is None:
            raise ArgumentError("masked grad_outer needs w")
        _need(w, "w", (R, C), dy_t.dtype)
    dw = torch.empty((R, C), dtype=torch.float32, device=dy_t.device)
    N.check(N.load().lors_grad_outer(L, R, C, dtype_code(dy_t.dtype), int(masked), _p(dy_t), _p(x_t),
                                     _p(w), _p(dw), _stream()))
    return dw


def rope(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor, layout: int = 0, inverse: bool = False):
    """Fused RoPE (rotate-half) + head transpose, bf16 (include/lors_decoder.h).
    layout 0: x [B, S, H, hd] -> [B, H, S, hd]; layout 1: x [B, H, S, hd] -> [B, S, H, hd];
    layout 2: x [B, S, H, hd] -> [B, S, H, hd] (no transpose).
    inverse=True rotates by -theta (the backward)."""
    if x.dtype != torch.bfloat16 or cos.dtype != torch.bfloat16 or sin.dtype != torch.bfloat16:
        raise ArgumentError("rope: bf16 tensors expected")
    if x.dim() != 4:
        raise ShapeError(f"rope: x must be 4-D, got {tuple(x.shape)}")
    x = x.contiguous()
    if layout == 0:
        B, S, H, hd = x.shape
        y = torch.empty((B, H, S, hd), dtype=x.dtype, device=x.device)
    elif layout == 2:
        B, S, H, hd = x.shape
        y = torch.empty_like(x)
    else:
        B, H, S, hd = x.shape
        y = torch.empty((B, S, H, hd), dtype=x.dtype, device=x.device)
    if cos.shape[0] < S or cos.shape[1] != hd or sin.shape != cos.shape:
        raise ShapeError(f"rope: tables {tuple(cos.shape)} do not cover [S={S}, hd={hd}]")
    cos, sin = cos.contiguous(), sin.contiguous()
    N.check(N.load().lors_rope(_p(x), _p(y), _p(cos), _p(sin), B, S, H, hd, layout, int(inverse), _stream()))
    return y


def sum_into(tensors) -> torch.Tensor:
    """tensors[0] <- the sum of 2+ same-shape bf16 tensors, three at a time in fp32 (lors_add3);
    returns tensors[0]."""
    out = tensors[0]
    if any(t.shape != out.shape or t.dtype != torch.bfloat16 or not t.is_contiguous() for t in tensors) \
            or out.numel() % 8:
        raise ShapeError("sum_into: contiguous bf16 tensors of one shape, a multiple of 8 elements")
    rest = list(tensors[1:])
    while rest:
        b = rest.pop(0)
        c = rest.pop(0) if rest else None
        N.check(N.load().lors_add3(_p(out), _p(b), None if c is None else _p(c), _p(out), out.numel(), _stream()))
    return out


def swiglu(g: torch.Tensor, u: torch.Tensor) -> torch.Tensor:
    """h = silu(g) * u, bf16, one kernel (include/lors_decoder.h)."""
    if g.shape != u.shape or g.dtype != torch.bfloat16 or u.dtype != torch.bfloat16:
        raise ShapeError("swiglu: g and u must be bf16 tensors of one shape")
    g, u = g.contiguous(), u.contiguous()
    h = torch.empty_like(g)
    N.check(N.load().lors_swiglu(_p(g), _p(u), _p(h), g.numel(), _stream()))
    return h


def add_rmsnorm(h: torch.Tensor, o: Optional[torch.Tensor], gamma: torch.Tensor, eps: float):
    """(hn = h + o, x = rmsnorm(hn) * gamma, rstd) over the last axis, bf16 in / out, fp32 rstd
    (include/lors_decoder.h).  o=None normalises h itself (hn is h)."""
    D = h.shape[-1]
    if h.dtype != torch.bfloat16 or gamma.dtype != torch.bfloat16 or (o is not None and o.dtype != torch.bfloat16):
        raise ArgumentError("add_rmsnorm: bf16 tensors expected")
    if gamma.shape != (D,) or (o is not None and o.shape != h.shape):
        raise ShapeError("add_rmsnorm: o must match h and gamma must be [D]")
    h = h.contiguous()
    o = None if o is None else o.contiguous()
    rows = h.numel() // D
    hn = torch.empty_like(h) if o is not None else h
    x = torch.empty_like(h)
    rstd = torch.empty(h.shape[:-1], dtype=torch.float32, device=h.device)
    N.check(N.load().lors_add_rmsnorm(_p(h), _p(o), _p(gamma.contiguous()), _p(hn) if o is not None else None, _p(x),
                                      _p(rstd), rows, D, float(eps), _stream()))
    return hn, x, rstd


def add_rmsnorm_bwd(dhn: Optional[torch.Tensor], dx: torch.Tensor, hn: torch.Tensor, gamma: torch.Tensor,
                    rstd: torch.Tensor) -> torch.Tensor:
    """Gradient of h (and o) for add_rmsnorm: dhn + the norm's backward, one rounding."""
    D = hn.shape[-1]
    dx, hn = dx.contiguous(), hn.contiguous()
    dhn = None if dhn is None else dhn.contiguous()
    dh = torch.empty_like(hn)
    N.check(N.load().lors_add_rmsnorm_bwd(_p(dhn), _p(dx), _p(hn), _p(gamma.contiguous()), _p(rstd), _p(dh),
                                          hn.numel() // D, D, _stream()))
    return dh


def cross_entropy(logits: torch.Tensor, targets: torch.Tensor):
    """(per-row loss, logsumexp) of bf16 logits [N, V] against int64 targets [N], fp32."""
    if logits.dtype != torch.bfloat16 or logits.dim() != 2 or targets.dtype != torch.int64:
        raise ArgumentError("cross_entropy: bf16 logits [N, V] and int64 targets expected")
    N_, V = logits.shape
    if targets.shape != (N_,):
        raise ShapeError(f"cross_entropy: targets must be [{N_}], got {tuple(targets.shape)}")
    logits, targets = logits.contiguous(), targets.contiguous()
    loss_rows = torch.empty(N_, dtype=torch.float32, device=logits.device)
    lse = torch.empty(N_, dtype=torch.float32, device=logits.device)
    N.check(N.load().lors_cross_entropy(_p(logits), _p(targets), _p(loss_rows), _p(lse), N_, V, _stream()))
    return loss_rows, lse


def cross_entropy_bwd(logits: torch.Tensor, targets: torch.Tensor, lse: torch.Tensor, grad_out: torch.Tensor,
                      out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """d(mean loss)/d logits scaled by the device scalar grad_out; written into `out` (may be `logits`)."""
    N_, V = logits.shape
    out = torch.empty_like(logits) if out is None else out
    g = grad_out.reshape(1).to(torch.float32).contiguous()
    N.check(N.load().lors_cross_entropy_bwd(_p(logits), _p(targets.contiguous()), _p(lse), _p(g), _p(out), N_, V,
                                            _stream()))
    return out


def swiglu_bwd(dh: torch.Tensor, g: torch.Tensor, u: torch.Tensor):
    """(dg, du) of h = silu(g) * u, bf16, one kernel."""
    dh, g, u = dh.contiguous(), g.contiguous(), u.contiguous()
    dg, du = torch.empty_like(g), torch.empty_like(u)
    N.check(N.load().lors_swiglu_bwd(_p(dh), _p(g), _p(u), _p(dg), _p(du), g.numel(), _stream()))
    return dg, du
