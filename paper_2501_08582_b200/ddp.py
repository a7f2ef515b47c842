"""Data-parallel exchange of the LoRS adapter gradients.

The path shards by tokens: W and its mask are replicated and
never communicated; a, b (and bias) gradients are sums over tokens, so one
averaging all-reduce per step is the only exchange.  Gradients are flattened
into fp32 buckets in reverse registration order (the order backward produces
them) and reduced with torch.distributed (NCCL over NVLink on B200; gloo in
the CPU tests).  With `overlap=True` each bucket is launched asynchronously
from a post-accumulate-grad hook as soon as its last gradient lands, so the
exchange overlaps the remaining backward.
"""

from __future__ import annotations

from typing import Iterable, List, Optional

import torch
import torch.distributed as dist
from torch import nn

from .errors import ArgumentError


def adapter_parameters(model: nn.Module) -> List[nn.Parameter]:
    """The trainable LoRS parameters (a, b, bias) of every LoRSLinear in `model`."""
    from .module import LoRSLinear
    params = []
    for mod in model.modules():
        if isinstance(mod, LoRSLinear):
            params += [p for p in (mod.a, mod.b, mod.bias) if p is not None and p.requires_grad]
    return params


class AdapterGradReducer:
    def __init__(self, params: Iterable[nn.Parameter], process_group=None, bucket_bytes: int = 32 << 20,
                 overlap: bool = False):
        self.params = [p for p in params if p.requires_grad]
        if not self.params:
            raise ArgumentError("no trainable adapter parameters")
        self.group = process_group
        self.world = dist.get_world_size(process_group) if dist.is_initialized() else 1
        # buckets in reverse order: the last layer's grads are ready first
        self.buckets: List[List[nn.Parameter]] = []
        cur, size = [], 0
        for p in reversed(self.params):
            cur.append(p)
            size += p.numel() * 4
            if size >= bucket_bytes:
                self.buckets.append(cur)
                cur, size = [], 0
        if cur:
            self.buckets.append(cur)
        self.flat = [torch.empty(sum(p.numel() for p in b), dtype=torch.float32, device=b[0].device)
                     for b in self.buckets]
        self._pending = []
        self._ready = [0] * len(self.buckets)
        self._stale = set()   # buckets launched, then accumulated into again (gradient accumulation)
        self._hooks = []
        if overlap:
            where = {}
            for bi, b in enumerate(self.buckets):
                for p in b:
                    where[id(p)] = bi
            for p in self.params:
                self._hooks.append(p.register_post_accumulate_grad_hook(
                    lambda param, bi=where[id(p)]: self._grad_ready(bi)))

    # -- overlap path -------------------------------------------------------
    def _grad_ready(self, bi: int) -> None:
        self._ready[bi] += 1
        n = len(self.buckets[bi])
        if self._ready[bi] == n:
            self._launch(bi, async_op=True)
        elif self._ready[bi] > n:
            # a further backward (gradient accumulation) added to grads this bucket already
            # sent: its reduction is redone from the accumulated .grad in finish()
            self._stale.add(bi)

    def _launch(self, bi: int, async_op: bool):
        bucket, flat = self.buckets[bi], self.flat[bi]
        off = 0
        for p in bucket:
            n = p.numel()
            if p.grad is None:
                flat[off:off + n].zero_()
            else:
                flat[off:off + n].copy_(p.grad.reshape(-1))
            off += n
        if self.world == 1:
            return None
        work = dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=self.group, async_op=async_op)
        if async_op:
            self._pending.append((bi, work))
        return work

    def _scatter_back(self, bi: int) -> None:
        flat = self.flat[bi]
        if self.world > 1:
            flat.div_(self.world)
        off = 0
        for p in self.buckets[bi]:
            n = p.numel()
            g = flat[off:off + n].view_as(p)
            if p.grad is None:
                p.grad = g.to(p.dtype).clone()
            else:
                p.grad.copy_(g)
            off += n

    def finish(self) -> None:
        """Wait for overlapped buckets (or reduce everything now) and write averaged grads back."""
        launched = {bi for bi, _ in self._pending}
        for bi, work in self._pending:
            work.wait()
        for bi in range(len(self.buckets)):
            if bi not in launched or bi in self._stale:
                self._launch(bi, async_op=False)
            self._scatter_back(bi)
        self._pending.clear()
        self._stale.clear()
        self._ready = [0] * len(self.buckets)

    __call__ = finish

    def remove_hooks(self) -> None:
        for h in self._hooks:
            h.remove()
        self._hooks.clear()


def broadcast_adapters(params: Iterable[nn.Parameter], src: int = 0, process_group=None) -> None:
    """Make every rank start from rank `src`'s adapters (replicated init)."""
    if not dist.is_initialized() or dist.get_world_size(process_group) == 1:
        return
    with torch.no_grad():
        for p in params:
            dist.broadcast(p.data, src=src, group=process_group)
