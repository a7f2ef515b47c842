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


class _ComparatorLinear(torch.nn.Module):
    """Frozen weight buffer + fp32 adapter masters a [R, r], b [r, C] (the LoRSLinear
    parameter layout), forward through one of the comparator Functions above."""

    FN = None

    def __init__(self, weight: torch.Tensor, a: torch.Tensor, b: torch.Tensor, alpha: float = 2.0, name: str = ""):
        super().__init__()
        self.register_buffer("weight", weight.detach())
        self.a = torch.nn.Parameter(a.detach().float().clone())
        self.b = torch.nn.Parameter(b.detach().float().clone())
        self.alpha = float(alpha)
        self.name = name

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        R, C = self.weight.shape
        y = self.FN.apply(x.reshape(-1, C), self.weight, self.a, self.b, self.alpha)
        return y.view(*x.shape[:-1], R)


class DenseLoRALinear(_ComparatorLinear):
    FN = DenseLoRAFunction


class SQFTLinear(_ComparatorLinear):
    FN = SQFTFunction


def comparator_factory(kind: str, cfg, a_std: float = 1e-3, seed: int = 0):
    """Decoder linear_factory for the memory comparators: kind "dense_lora" or "sqft".
    Same seeded adapters as decoder.lors_factory, so the three decoders differ only
    in the adapter linear."""
    import math

    cls = {"dense_lora": DenseLoRALinear, "sqft": SQFTLinear}[kind]
    counter = [0]

    def make(weight, rank, name):
        g = torch.Generator(device=weight.device).manual_seed(seed * 1000003 + counter[0])
        counter[0] += 1
        R, C = weight.shape
        a = torch.randn(R, rank, generator=g, device=weight.device) * a_std
        b = torch.randn(rank, C, generator=g, device=weight.device) / math.sqrt(rank)
        return cls(weight, a, b, alpha=cfg.alpha, name=name)

    return make
