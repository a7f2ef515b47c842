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


class FlatAdamW:
    """AdamW over all adapters in one launch (lors_adamw, include/lors_decoder.h).

    The fp32 adapter masters become views into one flat buffer (as a DDP bucket
    view would), the moments live in two more, and the same kernel writes the
    bf16 compute copies the LoRS kernels read (`_lors_shadow` views, see
    module.compute_copy), so a step casts no adapter.  Semantics of
    torch.optim.AdamW (decoupled weight decay, bias-corrected moments).  The step
    count lives on the device (lors_adamw_dstep), so the update can be replayed
    from a CUDA graph; `steps` mirrors it on the host."""

    def __init__(self, params: Sequence[nn.Parameter], lr: float, betas=(0.9, 0.999), eps: float = 1e-8,
                 weight_decay: float = 0.0, shadow_dtype=torch.bfloat16):
        from . import _native as N
        self.N = N
        self.params = list(params)
        dev = self.params[0].device
        if not all(p.is_cuda and p.dtype == torch.float32 and p.device == dev for p in self.params):
            raise ArgumentError("FlatAdamW needs fp32 CUDA parameters on one device")
        self.lr, (self.b1, self.b2), self.eps, self.wd = float(lr), betas, float(eps), float(weight_decay)
        n = sum(p.numel() for p in self.params)
        self.n = n
        self.P = torch.empty(n, dtype=torch.float32, device=dev)
        self.G = torch.zeros(n, dtype=torch.float32, device=dev)
        self.M = torch.zeros(n, dtype=torch.float32, device=dev)
        self.V = torch.zeros(n, dtype=torch.float32, device=dev)
        self.S = torch.empty(n, dtype=shadow_dtype, device=dev) if shadow_dtype is not None else None
        self.counter = torch.zeros(2, dtype=torch.int64, device=dev)   # updates taken, scratch
        off = 0
        self._offs = []
        with torch.no_grad():
            for p in self.params:
                k = p.numel()
                self.P[off:off + k].copy_(p.detach().reshape(-1))
                p.data = self.P[off:off + k].view_as(p)
                p._lors_grad_base = (self.G, off)   # the LoRS backward may write dA / dB here (module.grad_slots)
                self._offs.append(off)
                if self.S is not None:
                    p._lors_shadow = self.S[off:off + k].view_as(p)
                off += k
            if self.S is not None:
                self.S.copy_(self.P)
        self._mark()
        self.steps = 0

    def _mark(self) -> None:
        for p in self.params:
            p._lors_shadow_version = p._version

    def step(self) -> None:
        # gradients the LoRS backward wrote straight into their slot of G stay there; the others
        # (other layer types, accumulated micro-batches) are copied in
        g0 = self.G.data_ptr()
        in_place = [p.grad is not None and p.grad.data_ptr() == g0 + 4 * off and p.grad.is_contiguous()
                    for p, off in zip(self.params, self._offs)]
        if not any(in_place):
            grads = [p.grad.reshape(-1) if p.grad is not None else torch.zeros(p.numel(), device=self.P.device)
                     for p in self.params]
            torch.cat(grads, out=self.G)
        elif not all(in_place):
            for p, off, ok in zip(self.params, self._offs, in_place):
                if not ok:
                    dst = self.G[off:off + p.numel()]
                    if p.grad is None:
                        dst.zero_()
                    else:
                        dst.copy_(p.grad.reshape(-1))
        if self.S is not None and any(p._version != p._lors_shadow_version for p in self.params):
            self.S.copy_(self.P)             # a master was changed elsewhere: resync the compute copies
        self.steps += 1
        N = self.N
        N.check(N.load().lors_adamw_dstep(self.P.data_ptr(), self.G.data_ptr(), self.M.data_ptr(),
                                          self.V.data_ptr(), None if self.S is None else self.S.data_ptr(), self.n,
                                          self.lr, self.b1, self.b2, self.eps, self.wd, self.counter.data_ptr(),
                                          torch.cuda.current_stream(self.P.device).cuda_stream))
        self._mark()

    def zero_grad(self, set_to_none: bool = True) -> None:
        for p in self.params:
            p.grad = None
        self.G.zero_()    # the slots the next backward accumulates into start at zero


class Trainer:
    def __init__(self, model: nn.Module, lr: float = 2e-5, betas=(0.9, 0.999), eps: float = 1e-8,
                 weight_decay: float = 0.0, process_group=None, overlap: bool = True,
                 bucket_bytes: int = 64 << 20, params: Optional[Sequence[nn.Parameter]] = None,
                 optimizer: str = "auto", check_finite: bool = False, cuda_graph: bool = False,
                 tail_split: bool = False):
        self.model = model
        self.check_every_step = check_finite   # NumericError on a non-finite loss (train.py:215-217); syncs
        self.params = list(params) if params is not None else [p for p in model.parameters() if p.requires_grad]
        if not self.params:
            raise ArgumentError("model has no trainable adapter parameters")
        self.world = dist.get_world_size(process_group) if dist.is_initialized() else 1
        self.reducer = None
        if optimizer not in ("auto", "native", "torch", "p2p"):
            raise ArgumentError(f"optimizer must be auto, native, torch or p2p, got {optimizer!r}")
        if self.world > 1:
            broadcast_adapters(self.params, process_group=process_group)
            if optimizer != "p2p":    # p2p reduces the gradients inside its optimizer kernel
                self.reducer = AdapterGradReducer(self.params, process_group, bucket_bytes, overlap=overlap)
        cuda32 = all(p.is_cuda and p.dtype == torch.float32 for p in self.params)
        if optimizer == "p2p":
            from .collective import SymmetricAdamW
            self.opt = SymmetricAdamW(self.params, process_group, lr=lr, betas=betas, eps=eps,
                                      weight_decay=weight_decay)
        elif optimizer == "native" or (optimizer == "auto" and cuda32):
            self.opt = FlatAdamW(self.params, lr=lr, betas=betas, eps=eps, weight_decay=weight_decay)
        else:
            self.opt = torch.optim.AdamW(self.params, lr=lr, betas=betas, eps=eps, weight_decay=weight_decay,
                                         fused=all(p.is_cuda for p in self.params))
        self.steps = 0
        # cuda_graph: after one eager step, the whole step (forward, CE, backward, AdamW) is captured
        # once per token shape and replayed -- one graph launch instead of ~2300 kernel launches
        # from Python (tools/graph_probe.py).  One process, the native optimizer; the adapters must
        # change only through this trainer (call invalidate_graph() after loading weights).
        self.cuda_graph = bool(cuda_graph)
        if self.cuda_graph and (self.world > 1 or not isinstance(self.opt, FlatAdamW)):
            raise ArgumentError("cuda_graph needs one process and the native optimizer (FlatAdamW)")
        self._graph = None
        self._static_tokens = None
        self._static_loss = None
        self.graph_launches = 0      # native kernel launches recorded into the graph (one step)
        # the LoRS GEMMs' tail split along K (ops.set_tail_split) during this trainer's steps: off by
        # default -- a sustained step runs under the power cap, where the split's extra partial
        # traffic costs more than the idle SMs it fills (cfg3 +0.8%, cfg4 / cfg5 +0.3% without it)
        self.tail_split = bool(tail_split)

    def step(self, tokens: torch.Tensor) -> torch.Tensor:
        """One fine-tuning step on this rank's tokens [B, S + 1]; returns the (local) loss
        as a device scalar -- no host synchronisation."""
        from . import ops
        prev = ops.set_tail_split(self.tail_split)
        try:
            if self.cuda_graph:
                return self._step_graphed(tokens)
            return self._step_eager(tokens)
        finally:
            ops.set_tail_split(prev)

    def invalidate_graph(self) -> None:
        """Drop the captured step (the next step runs eagerly and captures again)."""
        self._graph = None
        self._static_tokens = None
        self._static_loss = None

    def _step_graphed(self, tokens: torch.Tensor) -> torch.Tensor:
        st = self._static_tokens
        same = st is not None and st.shape == tokens.shape and st.dtype == tokens.dtype
        if self._graph is not None and not same:
            self.invalidate_graph()                    # a new token shape: warm up and capture again
        if self._graph is None:
            if not same:
                loss = self._step_eager(tokens)        # warm-up: lazy handles and workspaces exist
                self._static_tokens = torch.empty_like(tokens, device=self.opt.P.device)
                return loss
            self._capture()
        self._static_tokens.copy_(tokens, non_blocking=True)
        self._graph.replay()
        self.opt.steps += 1
        self.steps += 1
        if self.check_every_step:
            self.check_finite(self._static_loss, self.steps - 1)
        return self._static_loss.clone()

    def _capture(self) -> None:
        from . import _native as N
        torch.cuda.synchronize()
        self.opt.zero_grad(set_to_none=True)
        torch.cuda.empty_cache()     # the warm-up step's cached blocks: the graph gets its own pool
        g = torch.cuda.CUDAGraph()
        n0 = N.launch_count()
        with torch.cuda.graph(g):
            loss = self.model.loss(self._static_tokens)
            loss.backward()
            self.opt.step()
            self.opt.zero_grad(set_to_none=True)
        self.graph_launches = N.launch_count() - n0
        self.opt.steps -= 1          # capture recorded the update without applying it
        self._static_loss = loss.detach()
        self._graph = g

    def _step_eager(self, tokens: torch.Tensor) -> torch.Tensor:
        loss = self.model.loss(tokens)
        if self.check_every_step:
            self.check_finite(loss, self.steps)
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
