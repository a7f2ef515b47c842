"""Memory / speed comparators for the LoRS layer, written in plain torch.

These are NOT the product path; they exist so the bench can state
"peak memory <= plain dense-LoRA" and "bytes not allocated relative to an
SQFT-style path that materialises W_eff" (north_star) on the same inputs.

- DenseLoRAFunction: `lora` semantics (adapters.py:245-283): Y = X W^T + alpha (X b^T) a^T,
  saves X and X b^T (rL + CL elements); no sparsity preservation.
- SQFTFunction: `sqft` semantics (adapters.py:290-312): materialises
  W_eff = W + alpha (a b) . M in the forward and saves X, M (bool) and W_eff
  (2RC + CL elements); masked adapter gradients.
"""

from __future__ import annotations

import torch


class DenseLoRAFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, a, b, alpha):
        dt = w.dtype
        ab_x = x @ b.to(dt).t()                       # [L, r]
        y = x @ w.t() + alpha * (ab_x @ a.to(dt).t())
        ctx.save_for_backward(x, ab_x)
        ctx.w, ctx.a, ctx.b, ctx.alpha = w, a, b, alpha
        return y

    @staticmethod
    def backward(ctx, dy):
        x, bx = ctx.saved_tensors
        w, a, b, alpha = ctx.w, ctx.a, ctx.b, ctx.alpha
        dt = w.dtype
        da = alpha * (dy.t() @ bx).float()            # adapters.py:271
        at_dy = dy @ a.to(dt)                         # [L, r]
        db = alpha * (at_dy.t() @ x).float()          # :273
        dx = dy @ w + alpha * (at_dy @ b.to(dt))      # :274-278
        return dx, None, da.to(a.dtype), db.to(b.dtype), None


class SQFTFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, a, b, alpha):
        dt = w.dtype
        mask = w != 0                                  # adapters.py:209-211 (bool here, RC bytes)
        merged = torch.where(mask, w + alpha * (a.to(dt) @ b.to(dt)), torch.zeros_like(w))
        y = x @ merged.t()
        ctx.save_for_backward(x, mask, merged)        # saves X, M, merged (adapters.py:299)
        ctx.a, ctx.b, ctx.alpha = a, b, alpha
        return y

    @staticmethod
    def backward(ctx, dy):
        x, mask, merged = ctx.saved_tensors
        a, b, alpha = ctx.a, ctx.b, ctx.alpha
        dt = merged.dtype
        dx = dy @ merged                               # adapters.py:306
        g = (dy.t() @ x) * mask                        # :307-308, R x C materialised
        da = alpha * (g @ b.to(dt).t()).float()        # :309
        db = alpha * (a.to(dt).t() @ g).float()        # :310
        return dx, None, da.to(a.dtype), db.to(b.dtype), None


def peak_bytes_of_step(fn, *tensors) -> int:
    """Peak extra device bytes allocated during one forward+backward of `fn`
    (inputs already resident; peak measured above the pre-step baseline)."""
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    fn(*tensors)
    torch.cuda.synchronize()
    return torch.cuda.max_memory_allocated() - base
