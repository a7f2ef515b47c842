"""Fused adapter-gradient collective + AdamW.

The path's only exchange is the average of the adapter gradients over the
data-parallel ranks.  Instead of an NCCL all-reduce followed by
an optimizer launch, `SymmetricAdamW` keeps the flat gradient, master and
bf16 compute-copy buffers in symmetric memory (torch.distributed.
_symmetric_memory: every rank maps every peer's buffers over NVLink) and runs
one kernel per step (`lors_adamw_p2p`): rank k owns shard k of the flat
buffers, sums that shard over all ranks' gradient buffers with peer loads,
applies AdamW with its shard of the optimizer state (ZeRO-1 style: m and v
are 1/world of the adapters) and writes the new values into every rank's
master and compute-copy buffers with peer stores.  Two device-side barriers
bracket the kernel.  Opt-in (`Trainer(optimizer="p2p")`): the round's GPU box
has one GPU, so the multi-rank path is correct by construction and its host
logic (`ShardLayout`, the shard-wise algorithm) is tested with gloo through
`ShardedAdamWReference`, which runs the same sharded algorithm with
all_reduce / all_gather.
"""

from __future__ import annotations

from typing import List, Sequence

import torch
import torch.distributed as dist
from torch import nn

from .errors import ArgumentError


class ShardLayout:
    """Flat layout of the adapter parameters and the per-rank shards: the buffer
    length is padded to a multiple of 4 * world (16-byte peer accesses)."""

    def __init__(self, params: Sequence[nn.Parameter], world: int):
        if world < 1:
            raise ArgumentError("world must be >= 1")
        self.params = list(params)
        self.offsets: List[int] = []
        off = 0
        for p in self.params:
            self.offsets.append(off)
            off += p.numel()
        self.n = off
        q = 4 * world
        self.n_pad = (off + q - 1) // q * q
        self.world = world
        self.shard = self.n_pad // world

    def bounds(self, rank: int):
        return rank * self.shard, (rank + 1) * self.shard

    def views(self, flat: torch.Tensor):
        """One view of `flat` per parameter, shaped like it."""
        return [flat[o:o + p.numel()].view_as(p) for o, p in zip(self.offsets, self.params)]

    def gather_grads(self, out: torch.Tensor) -> None:
        """Write every parameter's gradient (zeros where None) into out[:n]."""
        for o, p in zip(self.offsets, self.params):
            seg = out[o:o + p.numel()]
            if p.grad is None:
                seg.zero_()
            else:
                seg.copy_(p.grad.reshape(-1))


class _ShardedBase:
    def __init__(self, params, process_group, lr, betas, eps, weight_decay):
        self.group = process_group
        self.world = dist.get_world_size(process_group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(process_group) if dist.is_initialized() else 0
        self.layout = ShardLayout(params, self.world)
        self.params = self.layout.params
        self.lr, (self.b1, self.b2), self.eps, self.wd = float(lr), betas, float(eps), float(weight_decay)
        self.steps = 0

    def zero_grad(self, set_to_none: bool = True) -> None:
        for p in self.params:
            p.grad = None


class SymmetricAdamW(_ShardedBase):
    """Gradient average + AdamW in one peer-memory kernel per step (see module docstring)."""

    def __init__(self, params: Sequence[nn.Parameter], process_group=None, lr: float = 2e-5, betas=(0.9, 0.999),
                 eps: float = 1e-8, weight_decay: float = 0.0):
        import torch.distributed._symmetric_memory as symm_mem

        from . import _native as N
        super().__init__(params, process_group, lr, betas, eps, weight_decay)
        dev = self.params[0].device
        if not all(p.is_cuda and p.dtype == torch.float32 and p.device == dev for p in self.params):
            raise ArgumentError("SymmetricAdamW needs fp32 CUDA parameters on one device")
        group = process_group or dist.group.WORLD
        L = self.layout
        self.N = N
        self.G = symm_mem.empty(L.n_pad, dtype=torch.float32, device=dev)
        self.P = symm_mem.empty(L.n_pad, dtype=torch.float32, device=dev)
        self.S = symm_mem.empty(L.n_pad, dtype=torch.bfloat16, device=dev)
        self.hG = symm_mem.rendezvous(self.G, group)
        self.hP = symm_mem.rendezvous(self.P, group)
        self.hS = symm_mem.rendezvous(self.S, group)
        self.G.zero_()
        self.P.zero_()
        lo, hi = L.bounds(self.rank)
        self.M = torch.zeros(hi - lo, dtype=torch.float32, device=dev)
        self.V = torch.zeros(hi - lo, dtype=torch.float32, device=dev)
        with torch.no_grad():
            for p, view in zip(self.params, L.views(self.P)):
                view.copy_(p.detach())
                p.data = view
            for p, sview in zip(self.params, L.views(self.S)):
                p._lors_shadow = sview
            self.S.copy_(self.P)
        for p in self.params:
            p._lors_shadow_version = p._version
        self.hP.barrier(channel=0)

    def step(self) -> None:
        self.layout.gather_grads(self.G)
        self.steps += 1
        stream = torch.cuda.current_stream(self.G.device)
        self.hG.barrier(channel=0)          # every rank's gradients written; every rank done with P / S
        N = self.N
        N.check(N.load().lors_adamw_p2p(self.hG.buffer_ptrs_dev, self.hP.buffer_ptrs_dev, self.hS.buffer_ptrs_dev,
                                        self.M.data_ptr(), self.V.data_ptr(), self.layout.n_pad, self.rank,
                                        self.world, self.lr, self.b1, self.b2, self.eps, self.wd, self.steps,
                                        stream.cuda_stream))
        self.hP.barrier(channel=1)          # every rank's new masters and compute copies stored everywhere
        for p in self.params:
            p._lors_shadow_version = p._version


class ShardedAdamWReference(_ShardedBase):
    """The same sharded algorithm with torch.distributed collectives (gloo on CPU
    in the tests): average the gradients, update this rank's shard with its
    optimizer-state shard, all-gather the shards into every rank's masters."""

    def __init__(self, params: Sequence[nn.Parameter], process_group=None, lr: float = 2e-5, betas=(0.9, 0.999),
                 eps: float = 1e-8, weight_decay: float = 0.0):
        super().__init__(params, process_group, lr, betas, eps, weight_decay)
        L = self.layout
        dev = self.params[0].device
        self.G = torch.zeros(L.n_pad, dtype=torch.float32, device=dev)
        self.P = torch.zeros(L.n_pad, dtype=torch.float32, device=dev)
        with torch.no_grad():
            for p, view in zip(self.params, L.views(self.P)):
                view.copy_(p.detach())
                p.data = view
        lo, hi = L.bounds(self.rank)
        self.M = torch.zeros(hi - lo, dtype=torch.float32, device=dev)
        self.V = torch.zeros(hi - lo, dtype=torch.float32, device=dev)

    @torch.no_grad()
    def step(self) -> None:
        L = self.layout
        L.gather_grads(self.G)
        if self.world > 1:
            dist.all_reduce(self.G, group=self.group)
        self.steps += 1
        lo, hi = L.bounds(self.rank)
        g = self.G[lo:hi] / self.world
        p = self.P[lo:hi]
        self.M.mul_(self.b1).add_(g, alpha=1.0 - self.b1)
        self.V.mul_(self.b2).addcmul_(g, g, value=1.0 - self.b2)
        bc1 = 1.0 - self.b1 ** self.steps
        bc2 = 1.0 - self.b2 ** self.steps
        p.mul_(1.0 - self.lr * self.wd)
        p.addcdiv_(self.M, (self.V.sqrt() / bc2 ** 0.5).add_(self.eps), value=-self.lr / bc1)
        if self.world > 1:
            shards = [torch.empty_like(p) for _ in range(self.world)]
            dist.all_gather(shards, p.contiguous(), group=self.group)
            self.P.copy_(torch.cat(shards))
