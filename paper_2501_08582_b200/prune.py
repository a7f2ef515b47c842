"""One-shot pruning producers (untimed setup) and the SparseWeight type.

The reference stores no bitmap: a pruned entry is exactly 0 and M = (W != 0)
(prune.py:1-8, 33-69).  These are vectorised GPU equivalents of the
reference pruners with the same tie rule ("lower index removed first"),
verified bitwise against the reference in tests/test_prune_host.py:

  prune_rowwise(w, ratio)   == prune_activation_scaled(w, calib=ones, ratio)  prune.py:100-121
  prune_magnitude(w, ratio) == prune_magnitude                               prune.py:88-97
  prune_two_four(w)         == prune_two_four (magnitude score)              prune.py:124-149
"""

from __future__ import annotations

import torch

from .errors import ArgumentError


def _normalise_zero(t: torch.Tensor) -> torch.Tensor:
    # -0.0 -> +0.0 (prune.py:47)
    return torch.where(t == 0, torch.zeros_like(t), t)


def prune_rowwise(w: torch.Tensor, ratio: float) -> torch.Tensor:
    """Per row, remove the floor(ratio * C) smallest |w| (ties: lower column first)."""
    if not (0.0 <= ratio < 1.0):
        raise ArgumentError(f"prune ratio must be in [0, 1), got {ratio}")
    out = w.clone()
    n_remove = int(ratio * w.shape[1])
    if n_remove:
        order = torch.argsort(w.abs().float(), dim=1, stable=True)
        out.scatter_(1, order[:, :n_remove], 0)
    return _normalise_zero(out)


def prune_magnitude(w: torch.Tensor, ratio: float) -> torch.Tensor:
    """Global removal of floor(ratio * R * C) smallest |w| (ties: smaller (row, col) first)."""
    if not (0.0 <= ratio < 1.0):
        raise ArgumentError(f"prune ratio must be in [0, 1), got {ratio}")
    out = w.clone().reshape(-1)
    n_remove = int(ratio * out.numel())
    if n_remove:
        order = torch.argsort(out.abs().float(), stable=True)
        out[order[:n_remove]] = 0
    return _normalise_zero(out.reshape(w.shape))


def prune_two_four(w: torch.Tensor) -> torch.Tensor:
    """Keep the two largest |w| of every aligned group of 4 along the input axis."""
    R, C = w.shape
    if C % 4:
        raise ArgumentError(f"2:4 pruning requires cols divisible by 4, got {C}")
    g = w.clone().reshape(R, C // 4, 4)
    order = torch.argsort(g.abs().float(), dim=2, stable=True)
    g.scatter_(2, order[:, :, :2], 0)
    return _normalise_zero(g.reshape(R, C))


def two_four_valid(w: torch.Tensor) -> bool:
    """Every aligned group of 4 along the input axis has <= 2 nonzeros (prune.py:72-77)."""
    R, C = w.shape
    if C % 4:
        return False
    return bool(((w != 0).reshape(R, C // 4, 4).sum(dim=2) <= 2).all())


class SparseWeight:
    """Frozen pruned weight (prune.py:33-69): values with exact zeros; mask = values != 0."""

    def __init__(self, values: torch.Tensor, pattern: str = "unstructured", ratio: float = 0.0):
        if values.dim() != 2:
            raise ArgumentError("SparseWeight values must be 2-D")
        if pattern not in ("unstructured", "two_four"):
            raise ArgumentError(f"unknown sparsity pattern {pattern!r}")
        self.values = _normalise_zero(values.detach())
        self.pattern = pattern
        self.ratio = ratio
        if pattern == "two_four" and not two_four_valid(self.values):
            raise ArgumentError("values do not satisfy the 2:4 pattern")

    @property
    def rows(self) -> int:
        return self.values.shape[0]

    @property
    def cols(self) -> int:
        return self.values.shape[1]

    def mask_bool(self) -> torch.Tensor:
        return self.values != 0

    def mask(self) -> torch.Tensor:
        return self.mask_bool().to(self.values.dtype)

    def nonzeros(self) -> int:
        return int(torch.count_nonzero(self.values))


def sparsity(sw: SparseWeight) -> float:
    return 1.0 - sw.nonzeros() / (sw.rows * sw.cols)
