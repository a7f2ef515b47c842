"""The effective weight the tensor cores multiply IS the exported one, bit for bit.

The reference routes every variant and merge() through one `merged_weight`
(/root/reference/pkg/src/lors/adapters.py:214-224, 709-727) so that they are
bitwise identical.  Here the forward (K1, K2) and dX (K3) GEMMs rebuild W_eff
tile by tile on chip and never write it out, so it is observed through an
identity operand: with X_t = I_C the forward's output is Y_t = W_eff^T exactly
(fp32 accumulation of one bf16 product and zeros, then a rounding of a value
that is already bf16), and with dY_t = I_R the dX GEMM returns W_eff.  Both
must equal `effective_weight()` (K6, the forward prologue in export mode, the
weight merge() writes) bit for bit, with the +0.0 bit pattern wherever M = 0.
The numerics of that weight are then pinned against the oracle's merged_weight
(bf16 inputs, float64) within one bf16 rounding.
"""

import numpy as np
import pytest
import torch

from oracle import lors_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2501_08582_b200 import _native, ops
    _native.check(_native.load().lors_device_check())
    return ops


def _layer(R, C, r, pattern, seed, a_scale=0.05):
    from paper_2501_08582_b200 import prune
    g = torch.Generator().manual_seed(seed)
    w = torch.randn(R, C, generator=g) * 0.02
    w = prune.prune_two_four(w) if pattern == "two_four" else prune.prune_rowwise(w, 0.5)
    a = torch.randn(R, r, generator=g) * a_scale
    b = torch.randn(r, C, generator=g) / r ** 0.5
    return [t.to(torch.bfloat16).cuda().contiguous() for t in (w, a, b)]


def _same_bits(x, y):
    return torch.equal(x.contiguous().view(torch.int16), y.contiguous().view(torch.int16))


def _masked_pos_zero(weff, w):
    return bool((weff[w == 0].view(torch.int16) == 0).all())


# (R, C, r): small ragged-free shapes, r padding (r = 8 -> 16 columns of zeros), a
# cfg-like projection, and shapes whose persistent walk cuts the last wave along K
# (tail split: 256 x 8192 forward, 8192 x 256 dX)
SHAPES = [(512, 384, 16), (384, 256, 64), (256, 512, 8), (1024, 4096, 64), (256, 8192, 16)]
ALPHAS = [2.0, 1.0 / 3.0]


@pytest.mark.parametrize("alpha", ALPHAS)
@pytest.mark.parametrize("R,C,r", SHAPES)
@pytest.mark.parametrize("mode", ["from_w", "bits"])
def test_forward_tile_is_effective_weight(ops, R, C, r, mode, alpha):
    w, a, b = _layer(R, C, r, "rowwise", seed=R + C + r)
    bits = ops.pack_mask(w) if mode == "bits" else None
    eye = torch.eye(C, dtype=torch.bfloat16, device="cuda")
    y, _ = ops.lors_fwd(eye, w, a, b, alpha, mask_bits=bits)
    weff = ops.effective_weight(w, a, b, alpha, mask_bits=bits)
    torch.cuda.synchronize()
    assert _same_bits(y.t(), weff)
    assert _masked_pos_zero(y.t(), w)
    assert _masked_pos_zero(weff, w)


@pytest.mark.parametrize("alpha", ALPHAS)
@pytest.mark.parametrize("R,C,r", [(512, 384, 16), (384, 256, 64), (4096, 1024, 64), (8192, 256, 16)])
@pytest.mark.parametrize("mode", ["from_w", "bits"])
def test_dx_tile_is_effective_weight(ops, R, C, r, mode, alpha):
    w, a, b = _layer(R, C, r, "rowwise", seed=3 * R + C + r)
    bits = ops.pack_mask(w) if mode == "bits" else None
    eye = torch.eye(R, dtype=torch.bfloat16, device="cuda")
    x = torch.zeros(R, C, dtype=torch.bfloat16, device="cuda")   # L = R tokens; X only feeds dA/dB
    dx, _, _, _ = ops.lors_bwd(x, w, a, b, eye, alpha, mask_bits=bits)
    weff = ops.effective_weight(w, a, b, alpha, mask_bits=bits)
    torch.cuda.synchronize()
    assert _same_bits(dx, weff)
    assert _masked_pos_zero(dx, w)


@pytest.mark.parametrize("alpha", ALPHAS)
@pytest.mark.parametrize("R,C,r", [(512, 384, 16), (256, 512, 64), (1024, 4096, 64)])
@pytest.mark.parametrize("with_meta", [False, True])
def test_sparse24_tile_is_effective_weight(ops, R, C, r, with_meta, alpha):
    w, a, b = _layer(R, C, r, "two_four", seed=7 * R + C + r)
    meta = ops.compress_24(w)[1] if with_meta else None
    eye = torch.eye(C, dtype=torch.bfloat16, device="cuda")
    y, _ = ops.lors_fwd(eye, w, a, b, alpha, sparse24=True, meta24=meta)
    weff = ops.effective_weight(w, a, b, alpha)
    torch.cuda.synchronize()
    assert _same_bits(y.t(), weff)
    assert _masked_pos_zero(y.t(), w)


@pytest.mark.parametrize("alpha", ALPHAS)
@pytest.mark.parametrize("R,C,r", [(512, 384, 16), (1024, 4096, 64), (250, 120, 5)])
def test_effective_weight_vs_oracle(ops, R, C, r, alpha):
    """K6 against the oracle's merged_weight on the bf16-rounded inputs: W_eff is
    bf16(W + bf16(alpha P)) (the reference's order, matmul -> hadamard -> add_scaled,
    each result rounded to bf16), so every kept entry lies within half a bf16 ulp of
    alpha P plus half an ulp of the result of the float64 value (the fp32 rank-r sum
    adds a few fp32 ulps); every pruned entry is +0.0.  (250, 120, 5) runs the FFMA
    kernel (shapes TMA cannot address)."""
    w, a, b = _layer(R, C, r, "rowwise", seed=11 * R + r, a_scale=0.5)
    weff = ops.effective_weight(w, a, b, alpha).double().cpu().numpy()
    wd, ad, bd = (t.double().cpu().numpy() for t in (w, a, b))
    ref = orc.merged_weight(wd, ad, bd, alpha, orc.mask_matrix(wd))
    keep = wd != 0
    scaled = np.abs(alpha * (ad @ bd))
    ulp = (scaled + np.abs(ref)) * 2.0 ** -8 + 4e-6   # two bf16 roundings + the fp32 rank-r sum
    assert np.all(np.abs(weff - ref)[keep] <= ulp[keep])
    assert np.all(weff[~keep] == 0) and not np.signbit(weff[~keep]).any()


def test_merge_equals_trained_weight(ops):
    """merge() (reference adapters.py:709-727) writes the weight the forward multiplied."""
    import paper_2501_08582_b200 as P
    w, a, b = _layer(768, 512, 16, "rowwise", seed=5)
    layer = P.make_layer(P.SparseWeight(w), 16, "lors")
    layer.adapter.a.copy_(a)
    layer.adapter.b.copy_(b)
    merged = P.merge(layer)
    eye = torch.eye(512, dtype=torch.bfloat16, device="cuda")
    y, _ = ops.lors_fwd(eye, w, a, b, layer.adapter.alpha)
    torch.cuda.synchronize()
    assert _same_bits(merged.values, y.t())
