"""LLaMA-shaped decoder whose seven projections per layer are LoRS linears.

This is the caller of the hot path, not part of it: BASELINE configs 3-5 fine-tune
LLaMA-2-7B / LLaMA-3-8B / LLaMA-2-13B-shaped decoders, random init, where every
q/k/v/o/gate/up/down projection is a frozen pruned weight with trainable LoRS
adapters (the reference has no transformer; the decoder follows the
public LLaMA architecture: RMSNorm, RoPE, causal attention with optional GQA,
SwiGLU MLP).  Everything except the projections is frozen plain torch:
attention goes through `torch.nn.functional.scaled_dot_product_attention`
(cuDNN / flash library kernels), the LM head is a frozen cuBLAS GEMM.

The projections come from a `linear_factory(weight, rank, name)`; the default
builds `LoRSLinear` (the native kernels).  The memory comparators (dense LoRA,
SQFT-style materialised W_eff) plug in through the same hook, so the three
decoders differ only in the adapter linear.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, replace
from typing import Callable, Dict, Optional

import torch
import torch.nn.functional as F
from torch import nn

from . import ops
from .errors import ArgumentError
from .module import LoRSLinear, groupable, lors_group, pack_group_weights
from .prune import prune_rowwise, prune_two_four

PROJECTIONS = ("q", "k", "v", "o", "gate", "up", "down")


@dataclass(frozen=True)
class DecoderConfig:
    vocab: int
    dim: int
    n_layers: int
    n_heads: int
    n_kv_heads: int
    ffn: int
    rank: int
    sparsity: str            # "rowwise" (per-row magnitude, `ratio`) or "two_four"
    ratio: float = 0.5
    seq: int = 1024
    batch: int = 4           # sequences per GPU
    rope_theta: float = 10000.0
    eps: float = 1e-5
    alpha: float = 2.0
    dtype: torch.dtype = torch.bfloat16

    @property
    def head_dim(self) -> int:
        return self.dim // self.n_heads

    def shapes(self) -> Dict[str, tuple]:
        """(out, in) of each projection."""
        kv = self.n_kv_heads * self.head_dim
        d, f = self.dim, self.ffn
        return {"q": (d, d), "k": (kv, d), "v": (kv, d), "o": (d, d), "gate": (f, d), "up": (f, d), "down": (d, f)}

    def tokens_per_step(self) -> int:
        return self.batch * self.seq


# BASELINE.json configs[2..4]
PRESETS: Dict[str, DecoderConfig] = {
    "llama2-7b": DecoderConfig(vocab=32000, dim=4096, n_layers=32, n_heads=32, n_kv_heads=32, ffn=11008, rank=16,
                               sparsity="rowwise", ratio=0.5, seq=1024, batch=4),
    "llama3-8b": DecoderConfig(vocab=128256, dim=4096, n_layers=32, n_heads=32, n_kv_heads=8, ffn=14336, rank=64,
                               sparsity="two_four", seq=2048, batch=2, rope_theta=500000.0),
    "llama2-13b": DecoderConfig(vocab=32000, dim=5120, n_layers=40, n_heads=40, n_kv_heads=40, ffn=13824, rank=64,
                                sparsity="rowwise", ratio=0.7, seq=4096, batch=1),
    # small shape for tests and smoke runs
    "tiny": DecoderConfig(vocab=1000, dim=256, n_layers=2, n_heads=4, n_kv_heads=2, ffn=512, rank=16,
                          sparsity="rowwise", ratio=0.5, seq=128, batch=2),
}


def preset(name: str, **overrides) -> DecoderConfig:
    if name not in PRESETS:
        raise ArgumentError(f"unknown decoder preset {name!r}, expected one of {sorted(PRESETS)}")
    return replace(PRESETS[name], **overrides)


# ---------------------------------------------------------------------------
# algorithmic cost (roofline numerator), from the reference cost model
# ---------------------------------------------------------------------------

def adapter_param_count(cfg: DecoderConfig) -> int:
    return cfg.n_layers * sum(cfg.rank * (R + C) for R, C in cfg.shapes().values())


def flops_per_token(cfg: DecoderConfig) -> Dict[str, float]:
    """Per-token training FLOPs: the LoRS linears from COST_MODELS["lors"]
    (adapters.py:674-681) -- 4RC + 4r(R+C) per token plus the per-step recompute
    4(r+1)RC spread over the step's tokens -- causal attention 3.5 x 2 S d per layer,
    and the frozen LM head 4 d V (forward + dX)."""
    T = cfg.tokens_per_step()
    lin = rec = lin_fwd = 0.0
    for R, C in cfg.shapes().values():
        lin += 4 * R * C + 4 * cfg.rank * (R + C)
        lin_fwd += 2 * R * C
        rec += 4 * (cfg.rank + 1) * R * C / T
    out = {
        "linear": cfg.n_layers * lin,
        "linear_fwd_main": cfg.n_layers * lin_fwd,
        "recompute": cfg.n_layers * rec,
        "attention": cfg.n_layers * 3.5 * 2 * cfg.seq * cfg.dim,
        "head": 4.0 * cfg.dim * cfg.vocab,
    }
    out["total"] = out["linear"] + out["recompute"] + out["attention"] + out["head"]
    return out


def roofline_tokens_per_s(cfg: DecoderConfig, dense_tflops: float, sparse_tflops: Optional[float] = None) -> float:
    """Tokens/s at the tensor roofline; with a 2:4 model and `sparse_tflops`, the
    forward main products are charged at the sparse peak."""
    f = flops_per_token(cfg)
    t = f["total"] / (dense_tflops * 1e12)
    if cfg.sparsity == "two_four" and sparse_tflops:
        t -= f["linear_fwd_main"] / (dense_tflops * 1e12)
        t += f["linear_fwd_main"] / (sparse_tflops * 1e12)
    return 1.0 / t


# ---------------------------------------------------------------------------
# modules
# ---------------------------------------------------------------------------

class RMSNorm(nn.Module):
    def __init__(self, dim: int, eps: float, dtype, device):
        super().__init__()
        self.register_buffer("weight", torch.ones(dim, dtype=dtype, device=device))   # frozen gamma = 1
        self.eps = eps

    def forward(self, x):
        return F.rms_norm(x, (x.shape[-1],), self.weight, self.eps)


def rope_tables(cfg: DecoderConfig, device) -> tuple:
    inv = 1.0 / (cfg.rope_theta ** (torch.arange(0, cfg.head_dim, 2, device=device, dtype=torch.float32) / cfg.head_dim))
    freqs = torch.outer(torch.arange(cfg.seq, device=device, dtype=torch.float32), inv)
    emb = torch.cat((freqs, freqs), dim=-1)
    return emb.cos().to(cfg.dtype), emb.sin().to(cfg.dtype)


def _rotate_half(x):
    h = x.shape[-1] // 2
    return torch.cat((-x[..., h:], x[..., :h]), dim=-1)


def apply_rope(x, cos, sin):
    """x [B, H, S, hd]; cos/sin [S, hd] (rotate-half convention)."""
    return x * cos + _rotate_half(x) * sin


class RopeFunction(torch.autograd.Function):
    """Fused RoPE on the GPU (ops.rope, one kernel each way): x [B, S, H, hd] (the projection output
    viewed per head) -> the rotated heads as a [B, H, S, hd] view of a [B, S, H, hd] buffer.  Attention
    reads q / k / v with those strides (v is the same kind of view of its projection output), writes its
    output the same way, so neither the heads nor the attention output need a transpose copy."""

    @staticmethod
    def forward(ctx, x, cos, sin):
        ctx.save_for_backward(cos, sin)
        return ops.rope(x, cos, sin, layout=2).transpose(1, 2)

    @staticmethod
    def backward(ctx, gy):
        cos, sin = ctx.saved_tensors
        g = gy.transpose(1, 2)             # [B, S, H, hd]; contiguous when attention's grad kept the strides
        return ops.rope(g, cos, sin, layout=2, inverse=True), None, None


class SwiGLUFunction(torch.autograd.Function):
    """silu(g) * u in one kernel each way (ops.swiglu / swiglu_bwd); saves g and u only."""

    @staticmethod
    def forward(ctx, g, u):
        ctx.save_for_backward(g, u)
        return ops.swiglu(g, u)

    @staticmethod
    def backward(ctx, dh):
        g, u = ctx.saved_tensors
        return ops.swiglu_bwd(dh, g, u)


def swiglu(g, u):
    """silu(g) * u: the fused native kernel for CUDA bf16 (multiple of 8 elements),
    the torch formula elsewhere (CPU reference decoders in the tests)."""
    if g.is_cuda and g.dtype == torch.bfloat16 and g.numel() % 8 == 0:
        return SwiGLUFunction.apply(g, u)
    return F.silu(g) * u


class AddRMSNormFunction(torch.autograd.Function):
    """hn = h + o and x = RMSNorm(hn) * gamma (gamma frozen) in one kernel (ops.add_rmsnorm); the
    backward adds the residual gradient and the norm's in one kernel too, and hands that one
    gradient to both h and o (the add's backward is the identity).  Saves hn and rstd."""

    @staticmethod
    def forward(ctx, h, o, gamma, eps):
        hn, x, rstd = ops.add_rmsnorm(h, o, gamma, eps)
        ctx.save_for_backward(hn, gamma, rstd)
        return hn, x

    @staticmethod
    def backward(ctx, dhn, dx):
        hn, gamma, rstd = ctx.saved_tensors
        dh = ops.add_rmsnorm_bwd(dhn, dx, hn, gamma, rstd)
        return dh, dh, None, None


class CrossEntropyFunction(torch.autograd.Function):
    """Mean next-token cross-entropy of bf16 logits [N, V] (ops.cross_entropy: one pass per row, no fp32
    copy of the logits); the backward writes the logits' gradient over the logits themselves (they are
    this node's own input, consumed here only), scaled on the device by the incoming gradient."""

    @staticmethod
    def forward(ctx, logits, targets):
        loss_rows, lse = ops.cross_entropy(logits, targets)
        ctx.save_for_backward(logits, targets, lse)
        return loss_rows.mean()

    @staticmethod
    def backward(ctx, g):
        logits, targets, lse = ctx.saved_tensors
        return ops.cross_entropy_bwd(logits, targets, lse, g, out=logits), None


def fused_norms(h: torch.Tensor) -> bool:
    """Whether the decoder runs the fused residual-add + RMSNorm kernels: CUDA bf16 rows whose width
    the kernel takes (LORS_FUSED_NORM=0 turns them off for A/B runs)."""
    return (h.is_cuda and h.dtype == torch.bfloat16 and h.shape[-1] % 8 == 0 and h.shape[-1] <= 8192
            and os.environ.get("LORS_FUSED_NORM", "1") != "0")


def rope_heads(x_bshd, cos, sin):
    """[B, S, H, hd] -> RoPE'd [B, H, S, hd].  CUDA bf16: the native fused kernel
    (fails loudly without the library); elsewhere (CPU reference decoders in the
    tests): the plain torch formula."""
    if x_bshd.is_cuda and x_bshd.dtype == torch.bfloat16 and x_bshd.shape[-1] % 16 == 0:
        return RopeFunction.apply(x_bshd, cos, sin)
    return apply_rope(x_bshd.transpose(1, 2), cos, sin)


class DecoderLayer(nn.Module):
    def __init__(self, cfg: DecoderConfig, linears: Dict[str, nn.Module], device):
        super().__init__()
        self.cfg = cfg
        self.attn_norm = RMSNorm(cfg.dim, cfg.eps, cfg.dtype, device)
        self.mlp_norm = RMSNorm(cfg.dim, cfg.eps, cfg.dtype, device)
        self.proj = nn.ModuleDict(linears)

    def attention(self, x, cos, sin):
        """The attention branch of normalised input x [B, S, dim] (before the residual add)."""
        cfg, p = self.cfg, self.proj
        B, S, _ = x.shape
        qkv = [p["q"], p["k"], p["v"]]
        # projections of one input as one node: concurrent GEMMs, one summed dX
        qo, ko, vo = lors_group(qkv, x) if groupable(qkv) else (m(x) for m in qkv)
        q = rope_heads(qo.view(B, S, cfg.n_heads, cfg.head_dim), cos, sin)
        k = rope_heads(ko.view(B, S, cfg.n_kv_heads, cfg.head_dim), cos, sin)
        if vo._base is not None:
            # a grouped launch's outputs share one buffer: attention saves v, so v gets its own
            # storage and the buffer is freed with q / k once they are rotated (peak HBM unchanged)
            vo = vo.clone()
        v = vo.view(B, S, cfg.n_kv_heads, cfg.head_dim).transpose(1, 2)
        att = F.scaled_dot_product_attention(q, k, v, is_causal=True,
                                             enable_gqa=cfg.n_kv_heads != cfg.n_heads)
        return p["o"](att.transpose(1, 2).reshape(B, S, cfg.dim))

    def mlp(self, x):
        p = self.proj
        gu = [p["gate"], p["up"]]
        g, u = lors_group(gu, x) if groupable(gu) else (m(x) for m in gu)
        return p["down"](swiglu(g, u))

    def forward(self, h, cos, sin):
        h = h + self.attention(self.attn_norm(h), cos, sin)
        return h + self.mlp(self.mlp_norm(h))

    def forward_fused(self, h, x, cos, sin, next_norm: "RMSNorm"):
        """(h_next, next_norm(h_next)) from the residual h and x = attn_norm(h): both residual adds
        run inside the fused add + RMSNorm kernels (the second one with the next block's norm)."""
        h, x = AddRMSNormFunction.apply(h, self.attention(x, cos, sin), self.mlp_norm.weight, self.mlp_norm.eps)
        return AddRMSNormFunction.apply(h, self.mlp(x), next_norm.weight, next_norm.eps)


def lors_factory(cfg: DecoderConfig, a_std: float = 1e-3, b_std: Optional[float] = None,
                 sparse24_forward: bool = True, seed: int = 0) -> Callable:
    """Default projection: LoRSLinear with seeded adapters (a ~ N(0, a_std^2),
    b ~ N(0, 1/r) as BASELINE config 1) -- gradient-SVD init
    (init.init_gradient_svd) can replace them afterwards."""
    b_std = 1.0 / math.sqrt(cfg.rank) if b_std is None else b_std
    counter = [0]

    def make(weight: torch.Tensor, rank: int, name: str) -> nn.Module:
        g = torch.Generator(device=weight.device).manual_seed(seed * 1000003 + counter[0])
        counter[0] += 1
        R, C = weight.shape
        a = torch.randn(R, rank, generator=g, device=weight.device) * a_std
        b = torch.randn(rank, C, generator=g, device=weight.device) * b_std
        sp = sparse24_forward and cfg.sparsity == "two_four" and weight.dtype == torch.bfloat16 and C % 64 == 0
        return LoRSLinear(weight, a=a, b=b, alpha=cfg.alpha, name=name, sparse24=sp)

    return make


class LoRSDecoder(nn.Module):
    """Embedding -> n_layers x (RMSNorm, attention, RMSNorm, SwiGLU) -> RMSNorm -> LM head.
    Frozen: embedding, norms, LM head, every projection's base weight.  Trainable:
    the projections' adapters."""

    def __init__(self, cfg: DecoderConfig, device="cuda", seed: int = 0,
                 linear_factory: Optional[Callable] = None, init_std: float = 0.02):
        super().__init__()
        self.cfg = cfg
        dev = torch.device(device)
        factory = linear_factory or lors_factory(cfg, seed=seed)
        g = torch.Generator(device=dev).manual_seed(seed)

        def normal(*shape):
            return (torch.randn(*shape, generator=g, device=dev, dtype=torch.float32) * init_std).to(cfg.dtype)

        self.register_buffer("embed", normal(cfg.vocab, cfg.dim))
        layers = []
        for i in range(cfg.n_layers):
            linears = {}
            for name, (R, C) in cfg.shapes().items():
                w = normal(R, C)
                w = prune_two_four(w) if cfg.sparsity == "two_four" else prune_rowwise(w, cfg.ratio)
                linears[name] = factory(w, cfg.rank, f"layers.{i}.{name}")
                del w
            for grp in (("q", "k", "v"), ("gate", "up")):
                # one [G R, C] buffer per group of equal-shape projections, so their forward can run
                # as one grouped launch (module.packed_weights)
                ms = [linears[n] for n in grp]
                if all(isinstance(m, LoRSLinear) and m.weight.is_cuda for m in ms):
                    pack_group_weights(ms)
            layers.append(DecoderLayer(cfg, linears, dev))
        self.layers = nn.ModuleList(layers)
        self.norm = RMSNorm(cfg.dim, cfg.eps, cfg.dtype, dev)
        self.register_buffer("head", normal(cfg.vocab, cfg.dim))
        cos, sin = rope_tables(cfg, dev)
        self.register_buffer("rope_cos", cos, persistent=False)
        self.register_buffer("rope_sin", sin, persistent=False)

    def forward(self, tokens: torch.Tensor) -> torch.Tensor:
        """tokens [B, S] int64 -> logits [B, S, V] (compute dtype)."""
        S = tokens.shape[1]
        if S > self.cfg.seq:
            raise ArgumentError(f"sequence length {S} exceeds the RoPE table ({self.cfg.seq})")
        cos, sin = self.rope_cos[:S], self.rope_sin[:S]
        h = F.embedding(tokens, self.embed)
        if fused_norms(h):
            x = self.layers[0].attn_norm(h)
            for i, layer in enumerate(self.layers):
                nxt = self.layers[i + 1].attn_norm if i + 1 < len(self.layers) else self.norm
                h, x = layer.forward_fused(h, x, cos, sin, nxt)
            return F.linear(x, self.head)
        for layer in self.layers:
            h = layer(h, cos, sin)
        return F.linear(self.norm(h), self.head)

    def loss(self, tokens: torch.Tensor) -> torch.Tensor:
        """Next-token cross-entropy over tokens [B, S + 1] (mean over B*S predictions, fp32)."""
        logits = self(tokens[:, :-1])
        targets = tokens[:, 1:].reshape(-1)
        if logits.is_cuda and logits.dtype == torch.bfloat16 and self.cfg.vocab % 8 == 0 \
                and os.environ.get("LORS_FUSED_CE", "1") != "0":
            return CrossEntropyFunction.apply(logits.reshape(-1, self.cfg.vocab), targets)
        return F.cross_entropy(logits.float().reshape(-1, self.cfg.vocab), targets)

    def adapter_parameters(self):
        return [p for p in self.parameters() if p.requires_grad]

    def projections(self):
        for layer in self.layers:
            for name in PROJECTIONS:
                yield layer.proj[name]
