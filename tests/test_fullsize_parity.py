"""Full-size parity against the pinned oracle at every shape the benchmarks time.

BASELINE config 2 (one 11008 x 4096 2:4 projection, r = 64, 8192 tokens) through the
dense-masked forward, the 2:4 sparse-tensor-core forward, the backward and the
masked-G adapter gradients; and every projection shape of configs 3-5 (LLaMA-2-7B,
LLaMA-3-8B with GQA, LLaMA-2-13B; their masks and ranks) at the decoders' 4096
tokens per step.  The oracle (oracle/lors_oracle.py, float64, pinned to the
reference's own outputs) is fed the bf16-rounded inputs.  Y and dX are
token-local, so the oracle evaluates them on a seeded subset of 192 tokens of the
full GPU run (the kernels ran on all of them); dA and dB are sums over every token
and are checked in full.  Tolerance: north_star's bf16 bar, rel-L2 <= 2e-2.
"""

import zlib

import numpy as np
import pytest
import torch

from oracle import lors_oracle as orc

pytestmark = pytest.mark.gpu
TOL = 2e-2
N_SUB = 192


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2501_08582_b200 import _native, ops
    _native.check(_native.load().lors_device_check())
    return ops


def _inputs(R, C, L, r, pattern, ratio, seed):
    from paper_2501_08582_b200 import prune
    g = torch.Generator(device="cuda").manual_seed(seed)
    w = torch.randn(R, C, device="cuda", generator=g) * 0.02
    w = prune.prune_two_four(w) if pattern == "two_four" else prune.prune_rowwise(w, ratio)
    a = torch.randn(R, r, device="cuda", generator=g) * 0.02     # adapter term ~ W's scale
    b = torch.randn(r, C, device="cuda", generator=g) / r ** 0.5
    x = torch.randn(L, C, device="cuda", generator=g)
    dy = torch.randn(L, R, device="cuda", generator=g)
    return [t.to(torch.bfloat16).contiguous() for t in (w, a, b, x, dy)]


def _f64(t):
    return t.double().cpu().numpy()


def _rel(got, ref):
    return orc.rel_l2(np.asarray(got, dtype=np.float64), ref)


def _check_step(ops, R, C, L, r, pattern, ratio, seed, sparse24=False, masked=False):
    w, a, b, x, dy = _inputs(R, C, L, r, pattern, ratio, seed)
    meta = ops.compress_24(w)[1] if sparse24 else None
    y, _ = ops.lors_fwd(x, w, a, b, 2.0, sparse24=sparse24, meta24=meta)
    dx, da, db, _ = ops.lors_bwd(x, w, a, b, dy, 2.0)
    if masked:
        _, mda, mdb, _ = ops.lors_bwd(x, w, a, b, dy, 2.0, grad_mode="masked", need_dx=False)
    torch.cuda.synchronize()
    sub = np.sort(np.random.default_rng(seed).choice(L, size=min(N_SUB, L), replace=False))
    wd, ad, bd = _f64(w), _f64(a), _f64(b)
    xs, dys = _f64(x[sub]).T, _f64(dy[sub]).T            # reference orientation: C x l, R x l
    y_ref = orc.lors_forward(wd, ad, bd, xs, 2.0)
    dx_ref = orc.lors_backward(wd, ad, bd, xs, dys, 2.0).dx
    xd, dyd = _f64(x).T, _f64(dy).T
    da_ref, db_ref = orc.lors_adapter_grads(wd, ad, bd, xd, dyd, 2.0)
    errs = {"y": _rel(_f64(y[sub]).T, y_ref), "dx": _rel(_f64(dx[sub]).T, dx_ref),
            "da": _rel(_f64(da), da_ref), "db": _rel(_f64(db), db_ref)}
    if masked:
        mda_ref, mdb_ref = orc.sqft_gc_adapter_grads(wd, ad, bd, xd, dyd, 2.0)
        errs["masked_da"] = _rel(_f64(mda), mda_ref)
        errs["masked_db"] = _rel(_f64(mdb), mdb_ref)
    print(f"{R}x{C} L={L} r={r} {pattern} sparse24={sparse24}: " + ", ".join(f"{k} {v:.2e}" for k, v in errs.items()))
    assert max(errs.values()) <= TOL, errs


def test_cfg2_dense_masked_full(ops):
    """BASELINE configs[1] at full size: dense-masked forward (K1), backward (K3 + rank-r), masked-G (K5)."""
    _check_step(ops, 11008, 4096, 8192, 64, "two_four", 0.5, seed=2, masked=True)


def test_cfg2_sparse24_full(ops):
    """BASELINE configs[1] at full size on the 2:4 sparse tensor cores (K2), with the metadata stream."""
    _check_step(ops, 11008, 4096, 8192, 64, "two_four", 0.5, seed=3, sparse24=True)


# (R, C, r, pattern, ratio) of every projection of configs 3-5 (decoder.py PRESETS)
PROJ = {
    "cfg3-qkvo": (4096, 4096, 16, "rowwise", 0.5),
    "cfg3-gate/up": (11008, 4096, 16, "rowwise", 0.5),
    "cfg3-down": (4096, 11008, 16, "rowwise", 0.5),
    "cfg4-qo": (4096, 4096, 64, "two_four", 0.5),
    "cfg4-kv": (1024, 4096, 64, "two_four", 0.5),
    "cfg4-gate/up": (14336, 4096, 64, "two_four", 0.5),
    "cfg4-down": (4096, 14336, 64, "two_four", 0.5),
    "cfg5-qkvo": (5120, 5120, 64, "rowwise", 0.7),
    "cfg5-gate/up": (13824, 5120, 64, "rowwise", 0.7),
    "cfg5-down": (5120, 13824, 64, "rowwise", 0.7),
}


@pytest.mark.parametrize("name", list(PROJ))
def test_model_projection_shapes(ops, name):
    R, C, r, pattern, ratio = PROJ[name]
    seed = zlib.crc32(name.encode()) % 1000
    _check_step(ops, R, C, 4096, r, pattern, ratio, seed=seed)
    if pattern == "two_four":   # cfg4's forwards can run on the sparse tensor cores (bench --sparse24)
        _check_step(ops, R, C, 4096, r, pattern, ratio, seed=seed + 1, sparse24=True)


def _check_fp32(ops, R, C, L, r, seed, a_std, b_std, bits=False):
    """The fp32 parity mode (FFMA kernels) against the oracle on the same fp32 inputs, rel-L2 <= 1e-4."""
    from paper_2501_08582_b200 import prune
    g = torch.Generator(device="cuda").manual_seed(seed)
    w = prune.prune_rowwise(torch.randn(R, C, device="cuda", generator=g) * 0.02, 0.5).contiguous()
    a = (torch.randn(R, r, device="cuda", generator=g) * a_std).contiguous()
    b = (torch.randn(r, C, device="cuda", generator=g) * b_std).contiguous()
    x = torch.randn(L, C, device="cuda", generator=g)
    dy = torch.randn(L, R, device="cuda", generator=g)
    mb = ops.pack_mask(w) if bits else None
    y, _ = ops.lors_fwd(x, w, a, b, 2.0, mask_bits=mb)
    dx, da, db, _ = ops.lors_bwd(x, w, a, b, dy, 2.0, mask_bits=mb)
    torch.cuda.synchronize()
    sub = np.sort(np.random.default_rng(seed).choice(L, size=min(N_SUB, L), replace=False))
    wd, ad, bd = _f64(w), _f64(a), _f64(b)
    xs, dys = _f64(x[sub]).T, _f64(dy[sub]).T
    y_ref = orc.lors_forward(wd, ad, bd, xs, 2.0)
    dx_ref = orc.lors_backward(wd, ad, bd, xs, dys, 2.0).dx
    da_ref, db_ref = orc.lors_adapter_grads(wd, ad, bd, _f64(x).T, _f64(dy).T, 2.0)
    errs = {"y": _rel(_f64(y[sub]).T, y_ref), "dx": _rel(_f64(dx[sub]).T, dx_ref),
            "da": _rel(_f64(da), da_ref), "db": _rel(_f64(db), db_ref)}
    print(f"fp32 {R}x{C} L={L} r={r} bits={bits}: " + ", ".join(f"{k} {v:.2e}" for k, v in errs.items()))
    assert max(errs.values()) <= 1e-4, errs


def test_cfg1_fp32_full(ops):
    """BASELINE configs[0] at full size in the fp32 parity mode: 4096 x 4096, 50% per-row mask, r = 16,
    A ~ N(0, 1/r), B ~ N(0, 1e-3^2), 2048 tokens (the vectorised FFMA GEMM, R and C multiples of 4)."""
    _check_fp32(ops, 4096, 4096, 2048, 16, seed=11, a_std=16 ** -0.5, b_std=1e-3)


@pytest.mark.parametrize("R,C,L,r,bits", [(1028, 516, 300, 12, False), (1028, 516, 300, 12, True),
                                          (1030, 518, 77, 5, False), (772, 1540, 257, 28, True),
                                          (640, 384, 129, 40, False)])
def test_fp32_ragged_shapes(ops, R, C, L, r, bits):
    """Ragged fp32 shapes: tile edges of the 3xTF32 kernels (R, C, r multiples of 4; r <= 16 and <= 32
    instantiations), their packed-mask path, and the FFMA kernels (R, C not multiples of 4; r > 32)."""
    _check_fp32(ops, R, C, L, r, seed=R + L, a_std=0.05, b_std=r ** -0.5, bits=bits)


def test_fp32_bias_forward(ops):
    """The 3xTF32 forward's epilogue adds the bias (lors_forward with a bias, adapters.py:359-373)."""
    g = torch.Generator(device="cuda").manual_seed(5)
    R, C, L, r = 516, 260, 200, 8
    w = (torch.randn(R, C, device="cuda", generator=g) * 0.02) * (torch.rand(R, C, device="cuda", generator=g) > 0.5)
    a = torch.randn(R, r, device="cuda", generator=g) * 0.05
    b = torch.randn(r, C, device="cuda", generator=g) / r ** 0.5
    x = torch.randn(L, C, device="cuda", generator=g)
    bias = torch.randn(R, device="cuda", generator=g)
    y, _ = ops.lors_fwd(x, w, a, b, 2.0, bias)
    y0, _ = ops.lors_fwd(x, w, a, b, 2.0)
    torch.cuda.synchronize()
    ref = orc.lors_forward(_f64(w), _f64(a), _f64(b), _f64(x).T, 2.0).T + _f64(bias)[None, :]
    assert _rel(_f64(y), ref) <= 1e-4
    assert torch.allclose(y - y0, bias.expand_as(y), rtol=0, atol=1e-5)
