"""Gradient-SVD adapter initialisation on the GPU (north_star 5).

Reference: `init_gradient_svd` (initialization.py:171-232) with
`fit_rank_r_rows` (:121-131) and the SVD sign convention (svd.py:155-161):
zero every a, run one probe forward/backward, then per layer, one dW alive at
a time: dW = dY X^T (optionally restricted to the mask), b = the top-r right
singular vectors of dW as rows (first nonzero entry of each >= 0), a = 0.
Runs once, untimed.  dW comes from the native `lors_grad_outer` kernel; the
singular vectors from a symmetric eigendecomposition of dW^T dW (or dW dW^T,
whichever is smaller) on the GPU, refined to full float64 accuracy for small
layers by torch.linalg.svd.
"""

from __future__ import annotations

from typing import Callable, Dict, Iterable, List, Optional

import torch
from torch import nn

from . import ops
from .errors import ArgumentError


def _sign_fix_rows(b: torch.Tensor) -> torch.Tensor:
    """Flip each row so its first nonzero entry is >= 0 (svd.py:155-161)."""
    nz = b != 0
    first = torch.argmax(nz.to(torch.int8), dim=1)
    lead = b.gather(1, first.unsqueeze(1)).squeeze(1)
    sign = torch.where(lead < 0, -torch.ones_like(lead), torch.ones_like(lead))
    return b * sign.unsqueeze(1)


def fit_rank_r_rows(dw: torch.Tensor, r: int, scale: float = 1.0, exact_limit: int = 2048) -> torch.Tensor:
    """Top-r right singular vectors of dw (R x C) as the rows of b (r x C)."""
    R, C = dw.shape
    if r < 1 or r > min(R, C):
        raise ArgumentError(f"rank {r} must satisfy 1 <= r <= min({R}, {C})")
    if max(R, C) <= exact_limit:
        _, _, vh = torch.linalg.svd(dw.double(), full_matrices=False)
        b = vh[:r]
    elif C <= R:
        # right singular vectors = eigenvectors of dW^T dW (C x C), largest first
        g = dw.double().t() @ dw.double()
        _, vecs = torch.linalg.eigh(g)
        b = vecs[:, -r:].flip(1).t()
    else:
        # via the left vectors: u_i = eigvecs of dW dW^T; v_i = dW^T u_i / s_i
        g = dw.double() @ dw.double().t()
        vals, vecs = torch.linalg.eigh(g)
        u = vecs[:, -r:].flip(1)
        s = vals[-r:].flip(0).clamp_min(0).sqrt()
        b = (dw.double().t() @ u / s.clamp_min(1e-300)).t()
    b = _sign_fix_rows(b)
    return (b * scale).to(torch.float32)


@torch.no_grad()
def singular_tail(dw: torch.Tensor, r: int) -> float:
    s = torch.linalg.svdvals(dw.double())
    return float(torch.sqrt(torch.sum(s[r:] ** 2)))


def init_gradient_svd(layers: Iterable[nn.Module], probe: Callable[[], None], masked_gradient: bool = False,
                      scale: float = 1.0, diagnostics: Optional[list] = None) -> None:
    """Initialise every LoRSLinear in `layers` from one probe step.

    `probe()` must run one forward and backward through the model (the loss
    and data are the caller's, as the reference's ProbeBatch,
    initialization.py:198-200)."""
    from .module import LoRSLinear
    layers = [m for m in layers if isinstance(m, LoRSLinear)]
    if not layers:
        raise ArgumentError("no LoRSLinear layers to initialise")
    ranks = {m.rank for m in layers}
    if len(ranks) != 1:
        raise ArgumentError(f"layers disagree on rank: {sorted(ranks)}")
    xs: Dict[nn.Module, torch.Tensor] = {}
    dys: Dict[nn.Module, torch.Tensor] = {}
    hooks = []

    def fwd_hook(mod, inp, out):
        xs[mod] = inp[0].detach().reshape(-1, mod.in_features)
        if out.requires_grad:
            out.register_hook(lambda g, mod=mod: dys.__setitem__(mod, g.detach().reshape(-1, mod.out_features)))

    with torch.no_grad():
        for m in layers:
            m.a.zero_()  # initialization.py:196
    for m in layers:
        hooks.append(m.register_forward_hook(fwd_hook))
    from .module import no_grouping
    try:
        with no_grouping():    # grouped q/k/v and gate/up nodes would bypass the per-layer hooks
            probe()
    finally:
        for h in hooks:
            h.remove()
    for m in layers:
        if m not in xs or m not in dys:
            raise ArgumentError(f"probe did not reach layer {m.name or m}")
        dt = m.weight.dtype
        x = xs.pop(m).to(dt).contiguous()
        dy = dys.pop(m).to(dt).contiguous()
        dw = ops.grad_outer(dy, x, m.weight, masked=masked_gradient)   # one dW alive at a time
        b = fit_rank_r_rows(dw, m.rank)
        if diagnostics is not None:
            proj = (dw.double() @ b.double().t()) @ b.double()
            diagnostics.append({"layer": m.name, "rows": m.out_features, "cols": m.in_features, "rank": m.rank,
                                "grad_norm": float(dw.double().norm()),
                                "projection_residual": float((dw.double() - proj).norm()),
                                "singular_tail": singular_tail(dw, m.rank)})
        del dw
        with torch.no_grad():
            m.b.copy_(b * scale)
            m.a.zero_()
