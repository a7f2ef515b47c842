"""Data-parallel fine-tuning step for a LoRS decoder.

One process per GPU (torchrun), tokens sharded by rank, W / masks / frozen
weights replicated and never communicated.  A step is: forward, next-token
cross-entropy, backward (the LoRS kernels), the averaging all-reduce of the
adapter gradients (the path's only exchange, bucketed in reverse layer order
and launched from gradient hooks so it overlaps the rest of the backward),
then AdamW on the fp32 adapter masters (the reference's bias-corrected
"adaptive" update, train.py:139-154; decoupled weight decay, 0 by default).
"""

from __future__ import annotations

from typing import Optional, Sequence

import torch
import torch.distributed as dist
from torch import nn

from .ddp import AdapterGradReducer, broadcast_adapters
from .errors import ArgumentError, NumericError


def synthetic_tokens(vocab: int, batch: int, seq: int, step: int, rank: int = 0, seed: int = 0,
                     device="cuda") -> torch.Tensor:
    """Uniform token ids [batch, seq + 1] (BASELINE configs 3-5: uniform over the vocab),
    a distinct seeded stream per (rank, step)."""
    g = torch.Generator(device="cpu").manual_seed((seed * 1_000_003 + rank) * 1_000_003 + step)
    return torch.randint(0, vocab, (batch, seq + 1), generator=g).to(device)


class Trainer:
    def __init__(self, model: nn.Module, lr: float = 2e-5, betas=(0.9, 0.999), eps: float = 1e-8,
                 weight_decay: float = 0.0, process_group=None, overlap: bool = True,
                 bucket_bytes: int = 64 << 20, params: Optional[Sequence[nn.Parameter]] = None):
        self.model = model
        self.params = list(params) if params is not None else [p for p in model.parameters() if p.requires_grad]
        if not self.params:
            raise ArgumentError("model has no trainable adapter parameters")
        self.world = dist.get_world_size(process_group) if dist.is_initialized() else 1
        self.reducer = None
        if self.world > 1:
            broadcast_adapters(self.params, process_group=process_group)
            self.reducer = AdapterGradReducer(self.params, process_group, bucket_bytes, overlap=overlap)
        fused = all(p.is_cuda for p in self.params)
        self.opt = torch.optim.AdamW(self.params, lr=lr, betas=betas, eps=eps, weight_decay=weight_decay,
                                     fused=fused)
        self.steps = 0

    def step(self, tokens: torch.Tensor) -> torch.Tensor:
        """One fine-tuning step on this rank's tokens [B, S + 1]; returns the (local) loss
        as a device scalar -- no host synchronisation."""
        loss = self.model.loss(tokens)
        loss.backward()
        if self.reducer is not None:
            self.reducer.finish()
        self.opt.step()
        self.opt.zero_grad(set_to_none=True)
        self.steps += 1
        return loss.detach()

    @staticmethod
    def check_finite(loss: torch.Tensor, step: int) -> float:
        v = float(loss)
        if v != v or v in (float("inf"), float("-inf")):
            raise NumericError(f"non-finite loss at step {step}")
        return v
