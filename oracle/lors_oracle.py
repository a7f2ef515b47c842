"""CPU oracle for the LoRS masked-LoRA linear path -- TEST INFRASTRUCTURE ONLY.

This module is a float64 numpy restatement of the reference algorithm
(`/root/reference/pkg/src/lors/adapters.py`, `prune.py`).  It exists so the
GPU product can be checked against the reference's arithmetic on the GPU box,
where `/root/reference` does not exist.  Only `tests/`, `__graft_entry__.smoke()`
and `bench.py`'s CPU-baseline / `--impl reference` legs may import it; the
product package (`paper_2501_08582_b200`) never does.

Parity of this restatement is PINNED against the reference itself: the
fixtures under `tests/golden/` were produced by importing the reference
(`tests/golden/make_golden.py`) and `tests/test_oracle_golden.py` checks every
function below against them.

Layout convention: exactly the reference's -- X is C x L (samples are
columns), W is R x C, a is R x r, b is r x C, Y is R x L.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

ALPHA_DEFAULT = 2.0  # adapters.py:69


# ---------------------------------------------------------------------------
# mask / merged weight  (adapters.py:209-224)
# ---------------------------------------------------------------------------

def mask_matrix(w: np.ndarray) -> np.ndarray:
    """M = (W != 0) as float 0/1 -- adapters.py:209-211."""
    return (w != 0.0).astype(np.float64)


def merged_weight(w, a, b, alpha, mask):
    """W + alpha * ((a @ b) . M), same evaluation order -- adapters.py:214-224
    (matmul -> hadamard -> add_scaled, matrix.py:94-131)."""
    product = a @ b
    masked = product * mask
    return w + alpha * masked


# ---------------------------------------------------------------------------
# lors forward / backward  (adapters.py:359-406)
# ---------------------------------------------------------------------------

@dataclass
class Grads:
    """VariantGrads -- adapters.py:179-184."""
    da: np.ndarray
    db: np.ndarray
    dx: np.ndarray
    dbias: Optional[np.ndarray] = None


def lors_forward(w, a, b, x, alpha=ALPHA_DEFAULT, bias=None):
    """Y = (W + alpha (ab) . M) X [+ bias] -- adapters.py:359-373."""
    mask = mask_matrix(w)
    merged = merged_weight(w, a, b, alpha, mask)
    y = merged @ x
    if bias is not None:
        y = y + bias.reshape(-1, 1)
    return y


def lors_backward(w, a, b, x, dy, alpha=ALPHA_DEFAULT, with_bias=False,
                  sign_flip_fault=False):
    """Recompute merged weight; STE adapter grads -- adapters.py:376-406.

    Product order is the reference's bitwise-pinned order
    (test_adapters.py:204-228): dx, xt_bt, at_dy, da, db.
    """
    mask = mask_matrix(w)
    merged = merged_weight(w, a, b, alpha, mask)
    dx = merged.T.copy() @ dy                 # adapters.py:395
    xt_bt = x.T.copy() @ b.T.copy()           # :396
    at_dy = a.T.copy() @ dy                   # :397
    da = (dy @ xt_bt) * alpha                 # :398
    db = (at_dy @ x.T.copy()) * alpha         # :399
    if sign_flip_fault:                       # :400-401 negative control
        da = da * -1.0
    dbias = dy.sum(axis=1, keepdims=True) if with_bias else None  # :402
    return Grads(da=da, db=db, dx=dx, dbias=dbias)


def sqft_gc_backward(w, a, b, x, dy, alpha=ALPHA_DEFAULT, with_bias=False):
    """Masked-gradient schedule (_sqft_grads, adapters.py:303-312 via
    sqft_gc_backward :337-352): G = (dY X^T) . M; da = a G b^T; db = a a^T G."""
    mask = mask_matrix(w)
    merged = merged_weight(w, a, b, alpha, mask)
    dx = merged.T.copy() @ dy
    dy_xt = dy @ x.T.copy()
    masked = dy_xt * mask
    da = (masked @ b.T.copy()) * alpha
    db = (a.T.copy() @ masked) * alpha
    dbias = dy.sum(axis=1, keepdims=True) if with_bias else None
    return Grads(da=da, db=db, dx=dx, dbias=dbias)


def lors_adapter_grads(w, a, b, x, dy, alpha=ALPHA_DEFAULT):
    """(da, db) of lors_backward alone -- adapters.py:396-399 in the pinned order
    (xt_bt, at_dy, da, db); dx is token-local and is checked on token subsets."""
    xt_bt = x.T.copy() @ b.T.copy()           # :396
    at_dy = a.T.copy() @ dy                   # :397
    da = (dy @ xt_bt) * alpha                 # :398
    db = (at_dy @ x.T.copy()) * alpha         # :399
    return da, db


def sqft_gc_adapter_grads(w, a, b, x, dy, alpha=ALPHA_DEFAULT):
    """(da, db) of sqft_gc_backward alone -- _sqft_grads, adapters.py:303-312."""
    masked = (dy @ x.T.copy()) * mask_matrix(w)
    da = (masked @ b.T.copy()) * alpha
    db = (a.T.copy() @ masked) * alpha
    return da, db


def merge(w, a, b, alpha=ALPHA_DEFAULT, original_mask=None):
    """Finalize into a sparse weight -- adapters.py:709-727."""
    if original_mask is None:
        original_mask = w != 0.0
    merged = merged_weight(w, a, b, alpha, original_mask.astype(np.float64))
    merged[~original_mask] = 0.0
    return merged


# ---------------------------------------------------------------------------
# cost model  (adapters.py:643-706)
# ---------------------------------------------------------------------------

def predict_cost(variant, R, C, L, r):
    """(macs_forward, macs_backward, saved_elements) -- adapters.py:674-681."""
    if variant == "lors":
        return (R * C * L + r * R * C + R * C,
                R * C * L + 2 * r * R * L + 2 * r * C * L + r * R * C + R * C,
                C * L)
    if variant == "sqft_gc":
        return (R * C * L + R * C + r * R * C,
                2 * R * C * L + 3 * r * R * C + 2 * R * C,
                C * L)
    if variant == "sqft":
        return (R * C * L + R * C + r * R * C,
                2 * R * C * L + 2 * r * R * C + R * C,
                2 * R * C + C * L)
    if variant == "lora":
        return (R * C * L + r * C * L + r * R * L,
                R * C * L + 2 * r * R * L + 2 * r * C * L,
                r * L + C * L)
    raise ValueError(variant)


# ---------------------------------------------------------------------------
# pruning  (prune.py:72-149), vectorized but tie-rule identical
# ---------------------------------------------------------------------------

def prune_rowwise(w, ratio):
    """Per-row removal of floor(ratio*C) smallest |w|, ties: lower index
    removed first.  Equals prune_activation_scaled(w, calib=ones, ratio)
    (prune.py:100-121); stable argsort reproduces np.lexsort((arange, s))."""
    out = np.array(w, dtype=np.float64, copy=True)
    n_remove = int(ratio * out.shape[1])
    if n_remove:
        order = np.argsort(np.abs(out), axis=1, kind="stable")
        np.put_along_axis(out, order[:, :n_remove], 0.0, axis=1)
    out[out == 0.0] = 0.0  # -0.0 -> +0.0 (prune.py:47)
    return out


def prune_two_four(w):
    """Keep the top-2 |w| per aligned group of 4 along the input axis; ties
    remove the lower index first (prune.py:124-149), vectorized."""
    out = np.array(w, dtype=np.float64, copy=True)
    R, C = out.shape
    g = out.reshape(R, C // 4, 4)
    order = np.argsort(np.abs(g), axis=2, kind="stable")
    np.put_along_axis(g, order[:, :, :2], 0.0, axis=2)
    out = g.reshape(R, C)
    out[out == 0.0] = 0.0
    return out


def two_four_valid(w) -> bool:
    """prune.py:72-77."""
    R, C = w.shape
    if C % 4:
        return False
    nz = (w != 0.0).reshape(R, C // 4, 4)
    return bool((nz.sum(axis=2) <= 2).all())


def pack_mask(w) -> np.ndarray:
    """Bit-packed mask, uint32 words [R, ceil(C/32)], bit j of word k is
    column 32k+j (LSB first).  The layout `lors_pack_mask` emits."""
    R, C = w.shape
    words = (C + 31) // 32
    bits = np.zeros((R, words * 32), dtype=np.uint64)
    bits[:, :C] = (w != 0.0)
    bits = bits.reshape(R, words, 32)
    shifts = np.arange(32, dtype=np.uint64)
    return (bits << shifts).sum(axis=2).astype(np.uint32)


def sparsity(w) -> float:
    return 1.0 - np.count_nonzero(w) / w.size


# ---------------------------------------------------------------------------
# gradient-SVD init (initialization.py:121-131, svd.py:155-161)
# ---------------------------------------------------------------------------

def svd_sign_fix(v):
    """First nonzero entry of every right singular vector >= 0 (svd.py:155-161)."""
    v = v.copy()
    for idx in range(v.shape[1]):
        col = v[:, idx]
        nz = np.nonzero(col)[0]
        if nz.size and col[nz[0]] < 0.0:
            v[:, idx] = -col
    return v


def fit_rank_r_rows(dw, r):
    """b = top-r right singular vectors of dw as rows (initialization.py:121-131)."""
    _, _, vt = np.linalg.svd(dw, full_matrices=False)
    v = svd_sign_fix(vt.T)
    return v[:, :r].T.copy()


def singular_tail(dw, r):
    s = np.linalg.svd(dw, compute_uv=False)
    return float(np.sqrt(np.sum(s[r:] ** 2)))


def projection_residual(dw, b):
    return float(np.linalg.norm(dw - (dw @ b.T) @ b))


# ---------------------------------------------------------------------------
# the reference's own training task (train.py) -- loss-curve oracle
# ---------------------------------------------------------------------------

def adaptive_update(p, g, m, v, step, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """OptimState "adaptive" with bias correction, in place (train.py:139-154)."""
    m[:] = beta1 * m + (1.0 - beta1) * g
    v[:] = beta2 * v + (1.0 - beta2) * g * g
    m_hat = m / (1.0 - beta1 ** step)
    v_hat = v / (1.0 - beta2 ** step)
    p[:] = p - lr * m_hat / (np.sqrt(v_hat) + eps)


def toy_finetune(bases, a_list, b_list, x_t, t_t, batches, lr, alpha=ALPHA_DEFAULT, optimizer="adaptive"):
    """Loss per step of the reference's finetune loop on a ToyModel of lors
    layers with ReLU between them and the regression head
    (train.py:53-79 forward_loss, :196-207 _run_step, :255-277 finetune).

    x_t [N, C] and t_t [N, R_last] are the dataset in torch layout, batches is
    [steps, batch] column indices; a_list / b_list are updated in place.
    Loss = 0.5 * sum((Y - T)^2) / batch, so dY = (Y - T) / batch.
    """
    a_list = [np.array(a, dtype=np.float64) for a in a_list]      # copies: updated in place below
    b_list = [np.array(b, dtype=np.float64) for b in b_list]
    bases = [np.asarray(w, dtype=np.float64) for w in bases]
    mom = [(np.zeros_like(a), np.zeros_like(a), np.zeros_like(b), np.zeros_like(b))
           for a, b in zip(a_list, b_list)]
    losses = []
    for step, idx in enumerate(batches, start=1):
        x = np.ascontiguousarray(np.asarray(x_t, dtype=np.float64)[idx].T)   # C x L
        t = np.ascontiguousarray(np.asarray(t_t, dtype=np.float64)[idx].T)
        acts, pre = [x], []
        for i, w in enumerate(bases):
            z = lors_forward(w, a_list[i], b_list[i], acts[-1], alpha)
            pre.append(z)
            if i < len(bases) - 1:
                acts.append(np.maximum(z, 0.0))
        diff = pre[-1] - t
        n = x.shape[1]
        losses.append(0.5 * float(np.sum(diff * diff)) / n)
        dy = diff / n
        grads = [None] * len(bases)
        for i in range(len(bases) - 1, -1, -1):
            g = lors_backward(bases[i], a_list[i], b_list[i], acts[i], dy, alpha)
            grads[i] = g
            if i > 0:
                dy = g.dx * (pre[i - 1] > 0.0)
        for i, g in enumerate(grads):
            if optimizer == "sgd":                     # train.py:145-147
                a_list[i][:] = a_list[i] - lr * g.da
                b_list[i][:] = b_list[i] - lr * g.db
                continue
            ma, va, mb, vb = mom[i]
            adaptive_update(a_list[i], g.da, ma, va, step, lr)
            adaptive_update(b_list[i], g.db, mb, vb, step, lr)
    return np.array(losses), a_list, b_list


# ---------------------------------------------------------------------------
# torch-layout helpers for the parity harness
# ---------------------------------------------------------------------------

def lors_step_torch_layout(w, a, b, x_t, dy_t, alpha=ALPHA_DEFAULT, bias=None,
                           grad_mode="ste"):
    """Run forward+backward with torch-layout inputs (X_t [L,C], dY_t [L,R])
    and return torch-layout outputs (Y_t, dX_t, dA, dB, dbias)."""
    x = np.ascontiguousarray(x_t.T, dtype=np.float64)
    dy = np.ascontiguousarray(dy_t.T, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    y = lors_forward(w, a, b, x, alpha, bias)
    if grad_mode == "ste":
        g = lors_backward(w, a, b, x, dy, alpha, with_bias=bias is not None)
    else:
        g = sqft_gc_backward(w, a, b, x, dy, alpha, with_bias=bias is not None)
    dbias = None if g.dbias is None else g.dbias.reshape(-1)
    return y.T, g.dx.T, g.da, g.db, dbias


def rel_l2(got, ref) -> float:
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.linalg.norm(ref)
    num = np.linalg.norm(got - ref)
    return float(num / den) if den > 0 else float(num)
