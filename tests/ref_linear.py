"""Test-only reference projections for the decoder tests (never imported by the product).

- `TorchLoRSLinear`: the `lors` layer in plain torch (materialised W_eff, STE adapter
  gradients, adapters.py:359-406), any device/dtype -- the checker for the native
  decoder on the GPU and the stand-in projection for the CPU (gloo) trainer tests.
- `OracleLoRSLinear`: the same layer through the float64 oracle on the CPU
  (SURVEY 8 c4's "test-only autograd shim" for the model-level loss curve).
"""

import numpy as np
import torch
from torch import nn

from oracle import lors_oracle as orc


class _TorchLoRS(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, a, b, alpha):
        dt = w.dtype
        weff = torch.where(w != 0, w + alpha * (a.to(dt) @ b.to(dt)), torch.zeros_like(w))
        x2 = x.reshape(-1, w.shape[1]).to(dt)
        ctx.save_for_backward(x2, w, a, b)
        ctx.alpha, ctx.shape = alpha, x.shape
        return (x2 @ weff.t()).view(*x.shape[:-1], w.shape[0])

    @staticmethod
    def backward(ctx, dy):
        x2, w, a, b = ctx.saved_tensors
        alpha, dt = ctx.alpha, w.dtype
        weff = torch.where(w != 0, w + alpha * (a.to(dt) @ b.to(dt)), torch.zeros_like(w))
        dy2 = dy.reshape(-1, w.shape[0]).to(dt)
        dx = (dy2 @ weff).view(ctx.shape)
        da = alpha * (dy2.t().float() @ (x2.float() @ b.float().t()))      # adapters.py:396,398
        db = alpha * ((dy2.float() @ a.float()).t() @ x2.float())           # :397,399
        return dx, None, da.to(a.dtype), db.to(b.dtype), None


class TorchLoRSLinear(nn.Module):
    def __init__(self, weight, rank, name="", alpha=2.0):
        super().__init__()
        R, C = weight.shape
        self.register_buffer("weight", weight.detach().clone())
        self.a = nn.Parameter(torch.zeros(R, rank, device=weight.device))
        self.b = nn.Parameter(torch.zeros(rank, C, device=weight.device))
        self.alpha, self.name = alpha, name

    def forward(self, x):
        return _TorchLoRS.apply(x, self.weight, self.a, self.b, self.alpha)


class _OracleLoRS(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, a, b, alpha):
        x_ref = x.detach().reshape(-1, w.shape[1]).double().cpu().numpy().T      # C x L
        W, A, B = (t.detach().double().cpu().numpy() for t in (w, a, b))
        y = orc.lors_forward(W, A, B, x_ref, alpha)
        ctx.save_for_backward(x)
        ctx.np = (W, A, B, x_ref, alpha, x.shape)
        return torch.from_numpy(np.ascontiguousarray(y.T)).view(*x.shape[:-1], w.shape[0]).to(x.dtype)

    @staticmethod
    def backward(ctx, dy):
        W, A, B, x_ref, alpha, shape = ctx.np
        g = orc.lors_backward(W, A, B, x_ref, dy.detach().reshape(-1, W.shape[0]).double().numpy().T, alpha)
        dx = torch.from_numpy(np.ascontiguousarray(g.dx.T)).view(shape).to(dy.dtype)
        return dx, None, torch.from_numpy(g.da).float(), torch.from_numpy(g.db).float(), None


class OracleLoRSLinear(TorchLoRSLinear):
    def forward(self, x):
        return _OracleLoRS.apply(x, self.weight, self.a, self.b, self.alpha)


def torch_factory(weight, rank, name):
    return TorchLoRSLinear(weight, rank, name)


def oracle_factory(weight, rank, name):
    return OracleLoRSLinear(weight, rank, name)
