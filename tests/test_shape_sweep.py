"""Protocol sweep of the persistent tensor-core kernels over awkward shapes (GPU).

The K1 / K2 / K3 pipelines run a recompute lookahead of two k-steps, flip the issue order in the first
steps of every tile, split the last wave along K, clip TMA boxes at ragged edges and skip the second
MMA of an all-padding token tile.  This sweep runs every path on shapes that put those cases at the
edges -- a single k-step per tile, K not a multiple of 64, fewer tiles than clusters, one token, a
token count one past a tile -- and checks forward, dX and the adapter gradients against a float64
restatement of the reference formulas (adapters.py:359-406) on the bf16 inputs, plus the bit-exact
zeros of W_eff.  Each case is checked with and without the 2:4 sparse forward where the shape allows.
"""

import itertools

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2501_08582_b200 import _native, ops
    _native.check(_native.load().lors_device_check())
    return ops


def _ref(w, a, b, x, dy, alpha):
    """float64 lors_forward / lors_backward in the torch layout (tokens are rows)."""
    w, a, b, x, dy = (t.double() for t in (w, a, b, x, dy))
    weff = w + alpha * (a @ b) * (w != 0)
    y = x @ weff.t()
    dx = dy @ weff
    da = alpha * dy.t() @ (x @ b.t())
    db = alpha * (dy @ a).t() @ x
    return y, dx, da, db


def _rel(u, v):
    v = v.double()
    return float((u.double() - v).norm() / max(float(v.norm()), 1e-30))


SHAPES = [  # (L, R, C, r)
    (1, 256, 64, 8),        # one token, one k-step per tile
    (385, 264, 72, 16),     # a token past one 384-token tile, K not a multiple of 64
    (700, 520, 200, 40),    # r padded to 64, ragged everything
    (129, 8, 1032, 8),      # one feature row group, long K
    (1536, 136, 8200, 16),  # tail split along K (>= 128 k-steps), ragged R
    (4096, 2048, 320, 64),  # many tiles, short K (5 k-steps < tile boundary handling)
]


@pytest.mark.parametrize("L,R,C,r", SHAPES)
def test_shape_sweep(ops, L, R, C, r):
    from paper_2501_08582_b200 import prune
    g = torch.Generator(device="cuda").manual_seed(L * 7 + R * 3 + C + r)
    for pattern, alpha in itertools.product(("rowwise", "two_four"), (2.0, 0.75)):
        if pattern == "two_four" and C % 4:
            continue
        w = torch.randn(R, C, device="cuda", generator=g) * 0.02
        w = (prune.prune_two_four(w) if pattern == "two_four" else prune.prune_rowwise(w, 0.5)).bfloat16()
        a = (torch.randn(R, r, device="cuda", generator=g) * 0.02).bfloat16()
        b = (torch.randn(r, C, device="cuda", generator=g) / r ** 0.5).bfloat16()
        x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
        dy = torch.randn(L, R, device="cuda", generator=g).bfloat16()
        y_ref, dx_ref, da_ref, db_ref = _ref(w, a, b, x, dy, alpha)
        y, _ = ops.lors_fwd(x, w, a, b, alpha)
        dx, da, db, _ = ops.lors_bwd(x, w, a, b, dy, alpha)
        torch.cuda.synchronize()
        errs = {"y": _rel(y, y_ref), "dx": _rel(dx, dx_ref), "da": _rel(da, da_ref), "db": _rel(db, db_ref)}
        if pattern == "two_four" and C % 64 == 0:
            meta = ops.compress_24(w)[1]
            for m in (None, meta):
                ys, _ = ops.lors_fwd(x, w, a, b, alpha, sparse24=True, meta24=m)
                torch.cuda.synchronize()
                errs["y_sparse24" + ("_meta" if m is not None else "")] = _rel(ys, y_ref)
        assert max(errs.values()) <= 2e-2, (pattern, alpha, errs)
        weff = ops.effective_weight(w, a, b, alpha)
        assert bool((weff[w == 0].view(torch.int16) == 0).all())
