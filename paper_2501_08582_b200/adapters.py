"""Reference-facing operator API for the LoRS path (mirrors adapters.py).

Same names, argument meaning and error behaviour as
/root/reference/pkg/src/lors/adapters.py, over torch CUDA tensors in the
reference orientation (X is C x L, samples as columns; Y is R x L).  The
arithmetic runs in the native library (`ops`); X is passed to it as a
zero-copy transposed view whenever it is the transpose of a contiguous
[L, C] tensor.

Variants on the path: "lors" (STE adapter gradients, adapters.py:359-406) and
"sqft_gc" (the same forward; masked-G adapter gradients, adapters.py:330-352).
The remaining reference variants (lora, sqft, spp, spp_gc) are comparators
outside the hot path and are not provided here.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import torch

from . import ops
from .errors import ArgumentError, GraphError, ShapeError
from .prune import SparseWeight

VARIANTS = ("lors", "sqft_gc")
ALL_REFERENCE_VARIANTS = ("lora", "sqft", "sqft_gc", "spp", "spp_gc", "lors")

# Negative-control hooks (adapters.py:57-60).
FAULT_INJECTION = {
    "lors_backward_sign_flip": False,
    "cost_model_off_by_one": False,
}


@dataclass
class AdapterPair:
    """Low-rank factors a (R x r) and b (r x C) with a scaling factor (adapters.py:63-87)."""

    a: torch.Tensor
    b: torch.Tensor
    alpha: float = 2.0

    def __post_init__(self):
        if self.a.shape[1] != self.b.shape[0]:
            raise ShapeError(
                f"adapter rank mismatch: a is {self.a.shape[0]}x{self.a.shape[1]}, "
                f"b is {self.b.shape[0]}x{self.b.shape[1]}")
        r = self.a.shape[1]
        if r < 1 or r > min(self.a.shape[0], self.b.shape[1]):
            raise ArgumentError(f"rank {r} must satisfy 1 <= r <= min({self.a.shape[0]}, {self.b.shape[1]})")
        if not self.alpha > 0:
            raise ArgumentError(f"alpha must be positive, got {self.alpha}")

    @property
    def rank(self) -> int:
        return self.a.shape[1]


class AdaptedLayer:
    """A frozen SparseWeight plus a trainable adapter (adapters.py:111-165)."""

    def __init__(self, base: SparseWeight, adapter: AdapterPair, variant: str,
                 bias: Optional[torch.Tensor] = None, dropout: float = 0.0, name: str = ""):
        if variant not in ALL_REFERENCE_VARIANTS:
            raise ArgumentError(f"unknown variant {variant!r}, expected one of {ALL_REFERENCE_VARIANTS}")
        if variant not in VARIANTS:
            raise ArgumentError(f"variant {variant!r} is outside the LoRS hot path; supported: {VARIANTS}")
        if not isinstance(adapter, AdapterPair):
            raise ArgumentError(f"variant {variant} requires an AdapterPair")
        if adapter.a.shape[0] != base.rows:
            raise ShapeError(f"adapter a has {adapter.a.shape[0]} rows, base has {base.rows}")
        if adapter.b.shape[1] != base.cols:
            raise ShapeError(f"adapter b has {adapter.b.shape[1]} cols, base has {base.cols}")
        if bias is not None and tuple(bias.reshape(bias.shape[0], -1).shape) != (base.rows, 1):
            raise ShapeError(f"bias must be {base.rows}x1, got {tuple(bias.shape)}")
        if not (0.0 <= dropout < 1.0):
            raise ArgumentError(f"dropout must be in [0, 1), got {dropout}")
        if dropout != 0.0:
            raise ArgumentError("the lors path runs without dropout")
        self.base = base
        self.adapter = adapter
        self.variant = variant
        self.bias = bias
        self.dropout = dropout
        self.name = name
        # Captured once, packed 1 bit per entry (adapters.py:144-146 keeps a bool
        # matrix); merge() reuses it even if a kept weight later lands on zero.
        self.original_mask_bits = ops.pack_mask(base.values)
        self.last_nodes: dict = {}

    @property
    def original_mask(self) -> torch.Tensor:
        """Unpacked bool view of the captured mask (R x C)."""
        R, C = self.base.rows, self.base.cols
        words = self.original_mask_bits.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        shifts = torch.arange(32, device=words.device, dtype=torch.int64)
        bits = (words.unsqueeze(-1) >> shifts) & 1
        return bits.reshape(R, -1)[:, :C].bool()

    @property
    def out_features(self) -> int:
        return self.base.rows

    @property
    def in_features(self) -> int:
        return self.base.cols

    @property
    def rank(self) -> int:
        return self.adapter.rank

    def trainable(self) -> dict:
        params = {"a": self.adapter.a, "b": self.adapter.b}
        if self.bias is not None:
            params["bias"] = self.bias
        return params


def make_layer(base: SparseWeight, rank: int, variant: str, alpha: float = 2.0,
               bias: Optional[torch.Tensor] = None, name: str = "") -> AdaptedLayer:
    """Layer with zeroed adapter factors (adapters.py:168-176); fp32 masters."""
    dev = base.values.device
    adapter = AdapterPair(a=torch.zeros(base.rows, rank, device=dev), b=torch.zeros(rank, base.cols, device=dev),
                          alpha=alpha)
    return AdaptedLayer(base, adapter, variant, bias=bias, name=name)


@dataclass
class VariantGrads:
    """adapters.py:179-184 (da R x r, db r x C, dx C x L, dbias R x 1), fp32 for da/db/dbias."""

    da: torch.Tensor
    db: torch.Tensor
    dx: Optional[torch.Tensor]
    dbias: Optional[torch.Tensor] = None


class _Context:
    """Single-use saved-for-backward state (adapters.py:187-206).  Holds X only."""

    __slots__ = ("layer", "consumed", "tensors")

    def __init__(self, layer: AdaptedLayer, **tensors):
        self.layer = layer
        self.consumed = False
        self.tensors = tensors

    def consume(self):
        if self.consumed:
            raise GraphError("backward context already consumed")
        self.consumed = True

    def __getattr__(self, key):
        try:
            return self.tensors[key]
        except KeyError:
            raise AttributeError(key)


def _compute(layer: AdaptedLayer):
    dt = layer.base.values.dtype
    pair = layer.adapter
    return dt, pair.a.detach().to(dt).contiguous(), pair.b.detach().to(dt).contiguous()


def _as_rows(x: torch.Tensor) -> torch.Tensor:
    """C x L reference matrix -> contiguous [L, C] (zero-copy for transposed views)."""
    xt = x.t()
    return xt if xt.is_contiguous() else xt.contiguous()


def mask_matrix(base: SparseWeight) -> torch.Tensor:
    """M = (W != 0) as 0/1 (adapters.py:209-211).  API parity only: the kernels
    never materialise it."""
    return base.mask()


def merged_weight(w: torch.Tensor, a: torch.Tensor, b: torch.Tensor, alpha: float,
                  mask_bits: Optional[torch.Tensor] = None) -> torch.Tensor:
    """W + alpha ((a b) . M) (adapters.py:214-224), via the kernels' own prologue function."""
    dt = w.dtype
    return ops.effective_weight(w, a.to(dt).contiguous(), b.to(dt).contiguous(), alpha, mask_bits)


def _check_x(layer: AdaptedLayer, x: torch.Tensor) -> None:
    if x.dim() != 2 or x.shape[0] != layer.in_features:
        raise ShapeError(f"layer expects {layer.in_features} input rows, got {'x'.join(map(str, x.shape))}")


def _check_dy(layer: AdaptedLayer, dy: torch.Tensor, l_cols: int) -> None:
    if dy.dim() != 2 or dy.shape[0] != layer.out_features or dy.shape[1] != l_cols:
        raise ShapeError(f"gradient must be {layer.out_features}x{l_cols}, got {'x'.join(map(str, dy.shape))}")


def lors_forward(layer: AdaptedLayer, x: torch.Tensor, counters=None):
    """Y = (W + alpha (ab) . M) X [+ bias]; saves only X (adapters.py:359-373)."""
    _check_x(layer, x)
    dt, a, b = _compute(layer)
    x_t = _as_rows(x.to(dt))
    bias = None if layer.bias is None else layer.bias.detach().reshape(-1).to(dt).contiguous()
    y_t, _ = ops.lors_fwd(x_t, layer.base.values, a, b, layer.adapter.alpha, bias)
    ops.require_finite("lors_forward output", y_t)      # the reference's NumericError (matrix.py:53-54)
    if counters is not None:
        counters.add_forward(layer, x_t.shape[0])
    return y_t.t(), _Context(layer, x=x_t)


def _backward(grad_y: torch.Tensor, ctx: _Context, grad_mode: str, counters=None) -> VariantGrads:
    ctx.consume()
    layer = ctx.layer
    x_t = ctx.x
    _check_dy(layer, grad_y, x_t.shape[0])
    dt, a, b = _compute(layer)  # the adapter as it is at backward time (adapters.py:387)
    dy_t = _as_rows(grad_y.to(dt))
    dx, da, db, dbias = ops.lors_bwd(x_t, layer.base.values, a, b, dy_t, layer.adapter.alpha,
                                     grad_mode=grad_mode, with_bias=layer.bias is not None,
                                     fault_da_sign=(grad_mode == "ste"
                                                    and FAULT_INJECTION["lors_backward_sign_flip"]))
    ops.require_finite("lors_backward gradients", dx, da, db, dbias)
    if counters is not None:
        counters.add_backward(layer, x_t.shape[0])
    return VariantGrads(da=da, db=db, dx=dx.t(), dbias=None if dbias is None else dbias.reshape(-1, 1))


def lors_backward(grad_y: torch.Tensor, ctx: _Context, counters=None) -> VariantGrads:
    """Recompute W_eff; dX = W_eff^T dY; STE dA = a dY (X^T b^T), dB = a (a^T dY) X^T (adapters.py:376-406)."""
    return _backward(grad_y, ctx, "ste", counters)


def sqft_gc_forward(layer: AdaptedLayer, x: torch.Tensor, counters=None):
    """Numerically the lors forward; saves only X (adapters.py:330-334)."""
    return lors_forward(layer, x, counters)


def sqft_gc_backward(grad_y: torch.Tensor, ctx: _Context, counters=None) -> VariantGrads:
    """Masked-gradient schedule: G = (dY X^T) . M, da = a G b^T, db = a a^T G (adapters.py:303-312,337-352)."""
    return _backward(grad_y, ctx, "masked", counters)


_FORWARD = {"lors": lors_forward, "sqft_gc": sqft_gc_forward}
_BACKWARD = {"lors": lors_backward, "sqft_gc": sqft_gc_backward}


def variant_forward(layer: AdaptedLayer, x: torch.Tensor, counters=None):
    return _FORWARD[layer.variant](layer, x, counters)


def variant_backward(layer: AdaptedLayer, grad_y: torch.Tensor, ctx, counters=None) -> VariantGrads:
    return _BACKWARD[layer.variant](grad_y, ctx, counters)


class CostCounters:
    """Tally of algorithmic MACs / saved elements (tape.py:38-62 semantics).

    The kernels do not count their own multiply-adds; each call books the
    cost-model figures of COST_MODELS[variant] for its shape."""

    def __init__(self):
        self.macs_forward = 0
        self.macs_backward = 0
        self.saved_elements = 0

    def add_forward(self, layer: AdaptedLayer, L: int) -> None:
        m = COST_MODELS[layer.variant]
        R, C, r = layer.out_features, layer.in_features, layer.rank
        self.macs_forward += m.macs_forward(R, C, L, r)
        self.saved_elements += m.saved_elements(R, C, L, r)

    def add_backward(self, layer: AdaptedLayer, L: int) -> None:
        m = COST_MODELS[layer.variant]
        self.macs_backward += m.macs_backward(layer.out_features, layer.in_features, L, layer.rank)


def counted_saved(layer: AdaptedLayer, ctx: _Context) -> list:
    """adapters.py:584-592: lors / sqft_gc keep only X alive."""
    return [ctx.x]


@dataclass(frozen=True)
class VariantCostModel:
    """Closed-form (R, C, L, r) cost functions (adapters.py:628-640)."""

    variant: str
    macs_forward: Callable[[int, int, int, int], int]
    macs_backward: Callable[[int, int, int, int], int]
    saved_elements: Callable[[int, int, int, int], int]


COST_MODELS = {
    "lora": VariantCostModel(
        "lora",
        macs_forward=lambda R, C, L, r: R * C * L + r * C * L + r * R * L,
        macs_backward=lambda R, C, L, r: R * C * L + 2 * r * R * L + 2 * r * C * L,
        saved_elements=lambda R, C, L, r: r * L + C * L),
    "sqft": VariantCostModel(
        "sqft",
        macs_forward=lambda R, C, L, r: R * C * L + R * C + r * R * C,
        macs_backward=lambda R, C, L, r: 2 * R * C * L + 2 * r * R * C + R * C,
        saved_elements=lambda R, C, L, r: 2 * R * C + C * L),
    "sqft_gc": VariantCostModel(
        "sqft_gc",
        macs_forward=lambda R, C, L, r: R * C * L + R * C + r * R * C,
        macs_backward=lambda R, C, L, r: 2 * R * C * L + 3 * r * R * C + 2 * R * C,
        saved_elements=lambda R, C, L, r: C * L),
    "lors": VariantCostModel(
        "lors",
        macs_forward=lambda R, C, L, r: R * C * L + r * R * C + R * C,
        macs_backward=lambda R, C, L, r: R * C * L + 2 * r * R * L + 2 * r * C * L + r * R * C + R * C,
        saved_elements=lambda R, C, L, r: C * L),
}


@dataclass
class CostPrediction:
    macs_forward: int
    macs_backward: int
    saved_elements: int

    @property
    def flops(self) -> int:
        """Algorithmic FLOPs of one forward+backward (2 per MAC)."""
        return 2 * (self.macs_forward + self.macs_backward)


def predict_cost(variant: str, R: int, C: int, L: int, r: int) -> CostPrediction:
    """adapters.py:692-706."""
    if variant not in COST_MODELS:
        raise ArgumentError(f"unknown variant {variant!r}, expected one of {tuple(COST_MODELS)}")
    if min(R, C, L, r) < 1:
        raise ArgumentError(f"dimensions must be positive, got {(R, C, L, r)}")
    m = COST_MODELS[variant]
    pred = CostPrediction(m.macs_forward(R, C, L, r), m.macs_backward(R, C, L, r), m.saved_elements(R, C, L, r))
    if FAULT_INJECTION["cost_model_off_by_one"]:
        pred.macs_backward += 1
    return pred


def merge(layer: AdaptedLayer) -> SparseWeight:
    """W + alpha (ab) . original_mask, forced +0 outside it (adapters.py:709-727)."""
    merged = merged_weight(layer.base.values, layer.adapter.a, layer.adapter.b, layer.adapter.alpha,
                           mask_bits=layer.original_mask_bits)
    return SparseWeight(merged, pattern=layer.base.pattern, ratio=layer.base.ratio)
