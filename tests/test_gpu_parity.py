"""GPU parity: the native kernels vs the reference (golden fixtures) and the oracle.

Patterned on the reference's own suites (pkg/tests/test_adapters.py,
test_acceptance.py criteria 1-3, 5): forward/backward against the defining
expressions, masked-forward bitwise identity between lors and sqft_gc,
single-use contexts, shape validation, merge preserving the mask, and the
fault-injection negative control.  Tolerances (north_star): fp32 rel-L2 <= 1e-4,
bf16 rel-L2 <= 2e-2 (oracle fed the bf16-rounded inputs).
"""

import json
import os

import numpy as np
import pytest
import torch

from oracle import lors_oracle as orc

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")
TOL = {torch.float32: 1e-4, torch.bfloat16: 2e-2}


def _manifest():
    with open(os.path.join(GOLD, "manifest.json")) as f:
        return json.load(f)


CASES = _manifest()["cases"]


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2501_08582_b200 as P
    from paper_2501_08582_b200 import _native
    _native.check(_native.load().lors_device_check())
    return P


def _dev(a, dt):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dt).cuda().contiguous()


def _rel(got, ref):
    return orc.rel_l2(got.double().cpu().numpy(), ref)


def _bits_zero(t):
    it = {torch.float32: torch.int32, torch.bfloat16: torch.int16}[t.dtype]
    return bool((t.view(it) == 0).all())


# ---------------------------------------------------------------------------
# reference-produced fixtures
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("case", CASES, ids=[c["key"] for c in CASES])
def test_golden_lors_step(P, case, dt):
    from paper_2501_08582_b200 import ops
    d = dict(np.load(os.path.join(GOLD, f"lors_{case['key']}.npz")))
    if dt == torch.float32 or case["bf16_inputs"]:
        ref = d  # reference outputs on exactly these inputs
        y_ref, dx_ref, da_ref, db_ref = d["y"].T, d["dx"].T, d["da"], d["db"]
        mda, mdb = d["m_da"], d["m_db"]
    else:  # oracle on the bf16-rounded inputs
        q = {k: torch.from_numpy(d[k]).to(dt).double().numpy() for k in ("w", "a", "b", "x", "dy")}
        bias = None if "bias" not in d else torch.from_numpy(d["bias"]).to(dt).double().numpy()
        y_ref, dx_ref, da_ref, db_ref, _ = orc.lors_step_torch_layout(q["w"], q["a"], q["b"], q["x"].T,
                                                                      q["dy"].T, 2.0, bias)
        m = orc.sqft_gc_backward(q["w"], q["a"], q["b"], q["x"], q["dy"])
        mda, mdb = m.da, m.db
        ref = dict(d, bias=bias) if bias is not None else d
    w, a, b = _dev(d["w"], dt), _dev(d["a"], dt), _dev(d["b"], dt)
    x_t, dy_t = _dev(d["x"].T, dt), _dev(d["dy"].T, dt)
    bias = _dev(ref["bias"], dt) if "bias" in d else None
    y, _ = ops.lors_fwd(x_t, w, a, b, 2.0, bias)
    dx, da, db, dbias = ops.lors_bwd(x_t, w, a, b, dy_t, 2.0, with_bias=bias is not None)
    tol = TOL[dt]
    assert _rel(y, y_ref) <= tol
    assert _rel(dx, dx_ref) <= tol
    assert _rel(da, da_ref) <= tol
    assert _rel(db, db_ref) <= tol
    if bias is not None:
        assert _rel(dbias, d["dbias"]) <= tol
    _, mda_g, mdb_g, _ = ops.lors_bwd(x_t, w, a, b, dy_t, 2.0, grad_mode="masked", need_dx=False)
    assert _rel(mda_g, mda) <= tol
    assert _rel(mdb_g, mdb) <= tol


@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("case", CASES, ids=[c["key"] for c in CASES])
def test_golden_merge_preserves_mask_bitexact(P, case, dt):
    from paper_2501_08582_b200 import ops
    d = dict(np.load(os.path.join(GOLD, f"lors_{case['key']}.npz")))
    w, a, b = _dev(d["w"], dt), _dev(d["a"], dt), _dev(d["b"], dt)
    weff = ops.effective_weight(w, a, b, 2.0)
    assert _bits_zero(weff[w == 0])
    if dt == torch.float32:
        assert _rel(weff, d["merged"]) <= 1e-6
    bits = ops.pack_mask(w)
    weff2 = ops.effective_weight(w, a, b, 2.0, mask_bits=bits)
    assert torch.equal(weff.view(torch.uint8), weff2.view(torch.uint8))


# ---------------------------------------------------------------------------
# reference-API mirror (test_adapters.py patterns)
# ---------------------------------------------------------------------------

def random_layer(P, seed, variant, R, C, r, alpha=2.0, zero_frac=0.5, bias=False, dt=torch.float32):
    rng = np.random.default_rng(seed)
    w = rng.normal(size=(R, C))
    flat = np.argsort(np.abs(w), axis=None)
    w.reshape(-1)[flat[: int(zero_frac * R * C)]] = 0.0
    base = P.SparseWeight(_dev(w, dt))
    layer = P.make_layer(base, rank=r, variant=variant, alpha=alpha,
                         bias=_dev(rng.normal(size=(R,)), dt) if bias else None)
    layer.adapter.a = _dev(rng.normal(size=(R, r)), torch.float32)
    layer.adapter.b = _dev(rng.normal(size=(r, C)), torch.float32)
    return layer, w


def test_forward_matches_defining_expression(P):
    for i, variant in enumerate(P.VARIANTS):
        layer, w = random_layer(P, 100 + i, variant, R=6, C=8, r=2, bias=(i % 2 == 0))
        x = np.random.default_rng(7 + i).normal(size=(8, 5))
        y, _ = P.variant_forward(layer, _dev(x, torch.float32))
        a, b = layer.adapter.a.double().cpu().numpy(), layer.adapter.b.double().cpu().numpy()
        want = orc.lors_forward(w, a, b, x, 2.0,
                                None if layer.bias is None else layer.bias.double().cpu().numpy())
        assert _rel(y, want) <= 1e-6


def test_masked_forwards_bitwise_identical(P):
    for seed in range(5):
        outs = []
        x = _dev(np.random.default_rng(seed).normal(size=(7, 3)), torch.float32)
        for variant in P.VARIANTS:
            layer, _ = random_layer(P, seed, variant, R=5, C=7, r=2)
            y, _ = P.variant_forward(layer, x)
            outs.append(y.contiguous())
        assert torch.equal(outs[0], outs[1])


def test_context_is_single_use(P):
    layer, _ = random_layer(P, 21, "lors", R=4, C=4, r=1)
    x = _dev(np.random.default_rng(21).normal(size=(4, 3)), torch.float32)
    g = torch.ones(4, 3, device="cuda")
    _, ctx = P.variant_forward(layer, x)
    P.variant_backward(layer, g, ctx)
    with pytest.raises(P.GraphError):
        P.variant_backward(layer, g, ctx)


def test_shape_and_argument_validation(P):
    layer, _ = random_layer(P, 22, "sqft_gc", R=4, C=5, r=1)
    with pytest.raises(P.ShapeError):
        P.variant_forward(layer, torch.ones(4, 3, device="cuda"))
    _, ctx = P.variant_forward(layer, torch.ones(5, 3, device="cuda"))
    with pytest.raises(P.ShapeError):
        P.variant_backward(layer, torch.ones(4, 2, device="cuda"), ctx)
    z = lambda *s: torch.zeros(*s, device="cuda")  # noqa: E731
    with pytest.raises(P.ShapeError):
        P.AdapterPair(z(4, 2), z(3, 5))
    with pytest.raises(P.ArgumentError):
        P.AdapterPair(z(4, 5), z(5, 4))
    with pytest.raises(P.ArgumentError):
        P.AdapterPair(z(4, 2), z(2, 5), alpha=0.0)
    base = P.SparseWeight(torch.ones(4, 6, device="cuda"))
    with pytest.raises(P.ArgumentError):
        P.AdaptedLayer(base, P.AdapterPair(z(4, 2), z(2, 6)), "nope")
    with pytest.raises(P.ShapeError):
        P.AdaptedLayer(base, P.AdapterPair(z(5, 2), z(2, 6)), "lors")
    with pytest.raises(P.ShapeError):
        P.make_layer(base, rank=2, variant="lors", bias=torch.ones(3, device="cuda"))


def test_lors_grads_against_oracle_and_ste_surrogate(P):
    """dA/dB are the STE surrogate's gradients; dX the masked function's (test_adapters.py:138-187)."""
    layer, w = random_layer(P, 200, "lors", R=5, C=6, r=2, bias=True)
    rng = np.random.default_rng(50)
    x0, g = rng.normal(size=(6, 4)), rng.normal(size=(5, 4))
    _, ctx = P.variant_forward(layer, _dev(x0, torch.float32))
    grads = P.variant_backward(layer, _dev(g, torch.float32), ctx)
    a, b = layer.adapter.a.double().cpu().numpy(), layer.adapter.b.double().cpu().numpy()
    ref = orc.lors_backward(w, a, b, x0, g, 2.0, with_bias=True)
    for got, want in ((grads.da, ref.da), (grads.db, ref.db), (grads.dx, ref.dx), (grads.dbias, ref.dbias)):
        assert _rel(got, want) <= 1e-5
    # STE: the unmasked surrogate's gradient wrt a is alpha * g (b x)^T
    assert _rel(grads.da, 2.0 * g @ (b @ x0).T) <= 1e-5


def test_fault_injection_is_caught(P):
    layer, w = random_layer(P, 31, "lors", R=16, C=24, r=4)
    rng = np.random.default_rng(31)
    x0, g = rng.normal(size=(24, 8)), rng.normal(size=(16, 8))
    a, b = layer.adapter.a.double().cpu().numpy(), layer.adapter.b.double().cpu().numpy()
    ref = orc.lors_backward(w, a, b, x0, g)
    P.FAULT_INJECTION["lors_backward_sign_flip"] = True
    try:
        _, ctx = P.variant_forward(layer, _dev(x0, torch.float32))
        bad = P.variant_backward(layer, _dev(g, torch.float32), ctx)
    finally:
        P.FAULT_INJECTION["lors_backward_sign_flip"] = False
    assert _rel(bad.da, ref.da) > 1.0  # parity harness trips
    assert _rel(bad.db, ref.db) <= 1e-5


def test_merge_inside_mask_after_updates(P):
    layer, w = random_layer(P, 41, "lors", R=32, C=48, r=4)
    merged = P.merge(layer).values
    assert _bits_zero(merged[torch.from_numpy(w == 0).cuda()])
    layer.base.values[0, 0] = 0.0 if w[0, 0] != 0 else layer.base.values[0, 0]
    merged2 = P.merge(layer).values  # uses the mask captured at construction
    assert torch.count_nonzero(merged2) >= torch.count_nonzero(merged) - 1


def test_empty_batch(P):
    from paper_2501_08582_b200 import ops
    w = torch.randn(64, 32, device="cuda")
    a, b = torch.randn(64, 4, device="cuda"), torch.randn(4, 32, device="cuda")
    x = torch.empty(0, 32, device="cuda")
    y, _ = ops.lors_fwd(x, w, a, b)
    assert y.shape == (0, 64)
    dx, da, db, _ = ops.lors_bwd(x, w, a, b, torch.empty(0, 64, device="cuda"))
    assert dx.shape == (0, 32) and float(da.abs().sum()) == 0.0 and float(db.abs().sum()) == 0.0


# ---------------------------------------------------------------------------
# utilities: pack_mask, compress_24, grad_outer vs the oracle
# ---------------------------------------------------------------------------

def test_pack_mask_and_compress24(P):
    from paper_2501_08582_b200 import ops, prune
    rng = np.random.default_rng(3)
    w = orc.prune_two_four(rng.normal(size=(48, 96)))
    wd = _dev(w, torch.bfloat16)
    bits = ops.pack_mask(wd).cpu().numpy().view(np.uint32)
    np.testing.assert_array_equal(bits, orc.pack_mask(w))
    vals, meta, flag = ops.compress_24(wd)
    assert int(flag.item()) == 0
    m = meta.cpu().numpy()
    v = vals.float().cpu().numpy()
    for n in range(48):
        for g in range(96 // 4):
            nib = (int(m[n, g // 2]) >> (4 * (g % 2))) & 0xF
            i0, i1 = nib & 3, nib >> 2
            assert i0 < i1
            dense = np.zeros(4)
            dense[i0], dense[i1] = v[n, 2 * g], v[n, 2 * g + 1]
            np.testing.assert_array_equal(dense, torch.from_numpy(w[n, 4 * g:4 * g + 4]).bfloat16().float().numpy())
    bad = _dev(rng.normal(size=(8, 16)), torch.bfloat16)
    assert int(ops.compress_24(bad)[2].item()) == 1
    assert prune.two_four_valid(wd)


@pytest.mark.parametrize("masked", [False, True])
def test_grad_outer(P, masked):
    from paper_2501_08582_b200 import ops
    rng = np.random.default_rng(5)
    L, R, C = 40, 24, 36
    w = orc.prune_rowwise(rng.normal(size=(R, C)), 0.5)
    dy, x = rng.normal(size=(L, R)), rng.normal(size=(L, C))
    dw = ops.grad_outer(_dev(dy, torch.float32), _dev(x, torch.float32), _dev(w, torch.float32), masked)
    want = dy.T @ x
    if masked:
        want = want * (w != 0)
    assert _rel(dw, want) <= 1e-5


# ---------------------------------------------------------------------------
# full BASELINE sizes
# ---------------------------------------------------------------------------

def _cfg_tensors(R, C, L, r, dt, pattern, seed=0):
    from paper_2501_08582_b200 import prune
    g = torch.Generator(device="cuda").manual_seed(seed)
    w = torch.randn(R, C, device="cuda", generator=g) * 0.02
    w = prune.prune_two_four(w) if pattern == "two_four" else prune.prune_rowwise(w, 0.5)
    a = torch.randn(R, r, device="cuda", generator=g) * 1e-3   # north_star B ~ N(0, 1e-3^2)
    b = torch.randn(r, C, device="cuda", generator=g) / r ** 0.5  # north_star A ~ N(0, 1/r)
    x = torch.randn(L, C, device="cuda", generator=g)
    dy = torch.randn(L, R, device="cuda", generator=g)
    return [t.to(dt).contiguous() for t in (w, a, b, x, dy)]


def test_config1_fp32_full_size_vs_oracle(P):
    """BASELINE config 1 at full size: fp32 mode within rel-L2 1e-4 of the f64 reference path."""
    from paper_2501_08582_b200 import ops
    w, a, b, x, dy = _cfg_tensors(4096, 4096, 2048, 16, torch.float32, "rowwise")
    y, _ = ops.lors_fwd(x, w, a, b, 2.0)
    dx, da, db, _ = ops.lors_bwd(x, w, a, b, dy, 2.0)
    weff = ops.effective_weight(w, a, b, 2.0)
    assert _bits_zero(weff[w == 0])
    ref = orc.lors_step_torch_layout(*[t.double().cpu().numpy() for t in (w, a, b, x, dy)], alpha=2.0)
    for got, want in zip((y, dx, da, db), ref[:4]):
        assert _rel(got, want) <= 1e-4


def test_config2_bf16_full_size_properties(P):
    """BASELINE config 2 size (11008x4096, L=8192, r=64, 2:4) in bf16 against a torch
    fp32 reference of the same op (kept for this floating-point kernel), plus linearity."""
    from paper_2501_08582_b200 import ops
    w, a, b, x, dy = _cfg_tensors(11008, 4096, 8192, 64, torch.bfloat16, "two_four")
    y, _ = ops.lors_fwd(x, w, a, b, 2.0)
    dx, da, db, _ = ops.lors_bwd(x, w, a, b, dy, 2.0)
    wf, af, bf, xf, dyf = (t.float() for t in (w, a, b, x, dy))
    weff = torch.where(wf != 0, wf + 2.0 * (af @ bf), torch.zeros_like(wf))
    assert (_rel(y, (xf @ weff.t()).double().cpu().numpy()) <= 2e-2)
    assert (_rel(dx, (dyf @ weff).double().cpu().numpy()) <= 2e-2)
    p = xf @ bf.t()
    assert _rel(da, (2.0 * dyf.t() @ p).double().cpu().numpy()) <= 2e-2
    assert _rel(db, (2.0 * (dyf @ af).t() @ xf).double().cpu().numpy()) <= 2e-2
    # token-split property (size-independent), bit-exact with the tail split off
    with _env("LORS_NO_TAIL_SPLIT", "1"):
        y0, _ = ops.lors_fwd(x, w, a, b, 2.0)
        y1, _ = ops.lors_fwd(x[:4096].contiguous(), w, a, b, 2.0)
    assert torch.equal(y1, y0[:4096])


# ---------------------------------------------------------------------------
# gradient-SVD adapter init on the GPU (initialization.py:171-232)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("masked", [False, True])
def test_init_gradient_svd_two_layer_probe(P, masked):
    from paper_2501_08582_b200.init import init_gradient_svd
    rng = np.random.default_rng(9)
    C0, H, O, L, r = 48, 40, 24, 64, 4
    w1 = orc.prune_rowwise(rng.normal(size=(H, C0)), 0.5)
    w2 = orc.prune_rowwise(rng.normal(size=(O, H)), 0.5)
    x = rng.normal(size=(L, C0))
    g = rng.normal(size=(L, O))
    l1 = P.LoRSLinear(_dev(w1, torch.float32), rank=r)
    l2 = P.LoRSLinear(_dev(w2, torch.float32), rank=r)
    with torch.no_grad():
        l1.a.normal_()
        l2.a.normal_()   # init must zero a before probing
    xd, gd = _dev(x, torch.float32), _dev(g, torch.float32)

    def probe():
        y = l2(torch.relu(l1(xd)))
        (y * gd).sum().backward()

    diag = []
    init_gradient_svd([l1, l2], probe, masked_gradient=masked, diagnostics=diag)
    # oracle: a = 0 so W_eff = W
    y1 = x @ w1.T
    h = np.maximum(y1, 0)
    dy2 = g
    dy1 = (dy2 @ w2) * (y1 > 0)
    for layer, dy, xin, w in ((l1, dy1, x, w1), (l2, dy2, h, w2)):
        dw = dy.T @ xin
        if masked:
            dw = dw * (w != 0)
        want = orc.fit_rank_r_rows(dw, r)
        np.testing.assert_allclose(layer.b.detach().double().cpu().numpy(), want, atol=2e-3)
        assert float(layer.a.abs().sum()) == 0.0
    for d in diag:
        assert abs(d["projection_residual"] - d["singular_tail"]) <= 1e-3 * max(1.0, d["grad_norm"])


def test_init_gradient_svd_on_grouped_decoder(P):
    """The decoder runs q/k/v and gate/up as grouped autograd nodes (module.lors_group), which bypass
    the per-layer forward hooks; init_gradient_svd turns grouping off for its probe, so every one of
    the 7 projections per layer gets b = its top-r right singular vectors (orthonormal rows, first
    nonzero entry >= 0, svd.py:155-161) and a = 0 (initialization.py:171-232)."""
    from paper_2501_08582_b200 import decoder as D
    from paper_2501_08582_b200.init import init_gradient_svd
    from paper_2501_08582_b200.module import groupable
    from paper_2501_08582_b200.trainer import synthetic_tokens
    cfg = D.preset("tiny")
    model = D.LoRSDecoder(cfg, device="cuda", seed=0)
    layer0 = model.layers[0].proj
    assert groupable([layer0["q"], layer0["k"], layer0["v"]])
    toks = synthetic_tokens(cfg.vocab, cfg.batch, cfg.seq, 0, device="cuda")
    before = [p.b.detach().clone() for p in model.projections()]
    init_gradient_svd(list(model.projections()), lambda: model.loss(toks).backward())
    for proj, b0 in zip(model.projections(), before):
        b = proj.b.detach().double()
        assert not torch.equal(proj.b.detach(), b0)
        assert float(proj.a.abs().sum()) == 0.0
        gram = b @ b.t()
        assert torch.allclose(gram, torch.eye(cfg.rank, dtype=torch.float64, device="cuda"), atol=1e-4)
        first = b.gather(1, (b != 0).to(torch.int8).argmax(dim=1, keepdim=True))
        assert bool((first >= 0).all())


# ---------------------------------------------------------------------------
# 2:4 sparse-tensor-core forward (north_star 4)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("shape", [(256, 256, 64, 16), (300, 264, 192, 32), (512, 384, 256, 64)])
def test_sparse24_forward_matches_dense_and_oracle(P, shape):
    from paper_2501_08582_b200 import ops, prune
    L, R, C, r = shape
    g = torch.Generator(device="cuda").manual_seed(L + R)
    w = prune.prune_two_four(torch.randn(R, C, device="cuda", generator=g) * 0.02)
    w[: R // 4] = torch.where(torch.rand(R // 4, C, device="cuda", generator=g) < 0.3,
                              torch.zeros_like(w[: R // 4]), w[: R // 4])   # sparser groups: padding path
    a = torch.randn(R, r, device="cuda", generator=g) * 0.05
    b = torch.randn(r, C, device="cuda", generator=g) / r ** 0.5
    x = torch.randn(L, C, device="cuda", generator=g)
    w, a, b, x = (t.to(torch.bfloat16).contiguous() for t in (w, a, b, x))
    ys, _ = ops.lors_fwd(x, w, a, b, 2.0, sparse24=True)
    yd, _ = ops.lors_fwd(x, w, a, b, 2.0)
    ref = orc.lors_forward(*(t.double().cpu().numpy() for t in (w, a, b)), x.double().cpu().numpy().T, 2.0)
    assert _rel(ys, ref.T) <= 2e-2
    assert _rel(ys, yd.double().cpu().numpy()) <= 1e-3
    # precomputed kept-position metadata (lors_compress_24): same tiles, same bits
    _, meta, flag = ops.compress_24(w)
    assert int(flag.item()) == 0
    ym, _ = ops.lors_fwd(x, w, a, b, 2.0, sparse24=True, meta24=meta)
    assert torch.equal(ym.view(torch.int16), ys.view(torch.int16))


def test_masked_grad_tensor_core_path_vs_oracle(P):
    """The tcgen05 masked-G kernel (aligned shapes) against sqft_gc_backward, incl. ragged R/C/L."""
    from paper_2501_08582_b200 import ops
    for (L, R, C, r) in [(200, 136, 264, 16), (320, 256, 512, 64), (64, 128, 256, 32)]:
        rng = np.random.default_rng(L + R + C)
        w = orc.prune_rowwise(rng.normal(0, 0.02, size=(R, C)), 0.5)
        a, b = rng.normal(0, 0.05, size=(R, r)), rng.normal(0, 1 / np.sqrt(r), size=(r, C))
        x, dy = rng.normal(size=(L, C)), rng.normal(size=(L, R))
        q = [torch.from_numpy(v).to(torch.bfloat16) for v in (w, a, b, x, dy)]
        ref = orc.sqft_gc_backward(*(t.double().numpy() for t in q[:3]), q[3].double().numpy().T,
                                   q[4].double().numpy().T)
        wd, ad, bd, xd, dyd = (t.cuda().contiguous() for t in q)
        for bits in (None, ops.pack_mask(wd)):
            _, da, db, _ = ops.lors_bwd(xd, wd, ad, bd, dyd, 2.0, grad_mode="masked", need_dx=False, mask_bits=bits)
            assert _rel(da, ref.da) <= 2e-2
            assert _rel(db, ref.db) <= 2e-2


@pytest.mark.gpu
def test_backward_reads_adapter_at_backward_time(P):
    """The backward reuses the forward's bf16 adapter copies only while the fp32
    masters are unmodified; an in-place change between forward and backward is
    read at backward time (reference b2, adapters.py:387-394)."""
    from paper_2501_08582_b200 import ops
    from paper_2501_08582_b200.module import LoRSLinear
    g = torch.Generator(device="cuda").manual_seed(11)
    w = torch.randn(256, 128, device="cuda", generator=g) * 0.02
    w = torch.where(w.abs() < 0.01, torch.zeros_like(w), w).bfloat16()
    layer = LoRSLinear(w, a=torch.randn(256, 16, device="cuda", generator=g) * 0.05,
                       b=torch.randn(16, 128, device="cuda", generator=g) * 0.2)
    x = torch.randn(64, 128, device="cuda", generator=g).bfloat16().requires_grad_(True)
    dy = torch.randn(64, 256, device="cuda", generator=g).bfloat16()
    y = layer(x)
    with torch.no_grad():
        layer.a.mul_(3.0)                       # modified between forward and backward
    y.backward(dy)
    _, da, db, _ = ops.lors_bwd(x.detach(), w, layer.a.detach().bfloat16(), layer.b.detach().bfloat16(), dy, 2.0)
    assert torch.equal(layer.b.grad, db)       # dB = alpha a^T dY X uses the updated a
    assert torch.equal(layer.a.grad, da)


@pytest.mark.gpu
def test_overlapped_backward_equals_single_call(P):
    """ops.lors_bwd's two-stream split (LORS_FLAG_DX_ONLY + NO_DX) gives the same results
    as one C-ABI call computing everything on one stream: dX and dbias bit-identical,
    dA / dB to fp32 summation order (their split-K partial sums are atomic reductions)."""
    from paper_2501_08582_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(21)
    L, R, C, r = 1000, 512, 384, 24
    w = torch.randn(R, C, device="cuda", generator=g) * 0.02
    w = torch.where(w.abs() < 0.012, torch.zeros_like(w), w).bfloat16()
    a = (torch.randn(R, r, device="cuda", generator=g) * 0.05).bfloat16()
    b = (torch.randn(r, C, device="cuda", generator=g) * 0.2).bfloat16()
    x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
    dy = torch.randn(L, R, device="cuda", generator=g).bfloat16()
    one = ops.lors_bwd(x, w, a, b, dy, 2.0, with_bias=True, overlap=False)
    two = ops.lors_bwd(x, w, a, b, dy, 2.0, with_bias=True, overlap=True)
    torch.cuda.synchronize()
    assert torch.equal(one[0], two[0]) and torch.equal(one[3], two[3])
    for u, v in zip(one[1:3], two[1:3]):
        assert float((u - v).norm() / u.norm()) < 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("r,mask_mode,with_bias", [(16, "from_w", True), (24, "bits", False), (40, "from_w", False),
                                                   (64, "bits", True)])
def test_persistent_multi_tile_shapes(P, r, mask_mode, with_bias):
    """Shapes with more pair tiles than co-resident CTA pairs (several tiles per
    persistent CTA pair), ragged token count, every padded-rank variant, packed-bit
    and from-W masks, bias: forward / dX / dA / dB against a torch fp32 reference,
    masked W_eff entries bit-exact +0, and the token-split property."""
    from paper_2501_08582_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(100 + r)
    L, R, C = 3001, 4352, 1280                      # 17 feature pairs x 8 token tiles = 136 pair tiles
    w = torch.randn(R, C, device="cuda", generator=g) * 0.02
    w = torch.where(w.abs() < 0.015, torch.zeros_like(w), w).bfloat16()
    a = (torch.randn(R, r, device="cuda", generator=g) * 0.05).bfloat16()
    b = (torch.randn(r, C, device="cuda", generator=g) * 0.3).bfloat16()
    x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
    dy = torch.randn(L, R, device="cuda", generator=g).bfloat16()
    bias = (torch.randn(R, device="cuda", generator=g) * 0.1).bfloat16() if with_bias else None
    bits = ops.pack_mask(w) if mask_mode == "bits" else None
    y, _ = ops.lors_fwd(x, w, a, b, 2.0, bias, bits)
    dx, da, db, dbias = ops.lors_bwd(x, w, a, b, dy, 2.0, mask_bits=bits, with_bias=with_bias)
    wf, af, bf, xf, dyf = (t.float() for t in (w, a, b, x, dy))
    weff = torch.where(wf != 0, wf + 2.0 * (af @ bf), torch.zeros_like(wf))
    yref = xf @ weff.t() + (bias.float() if with_bias else 0.0)
    assert _rel(y, yref.double().cpu().numpy()) <= 2e-2
    assert _rel(dx, (dyf @ weff).double().cpu().numpy()) <= 2e-2
    assert _rel(da, (2.0 * dyf.t() @ (xf @ bf.t())).double().cpu().numpy()) <= 2e-2
    assert _rel(db, (2.0 * (dyf @ af).t() @ xf).double().cpu().numpy()) <= 2e-2
    if with_bias:
        assert _rel(dbias, dyf.sum(0).double().cpu().numpy()) <= 1e-3
    we = ops.effective_weight(w, a, b, 2.0, bits)
    assert bool((we[w == 0].view(torch.int16) == 0).all())
    # token-split property (batch invariance) holds with the tail split off: a split
    # tile sums its K parts in a different order than one continuous accumulation
    with _env("LORS_NO_TAIL_SPLIT", "1"):
        y1, _ = ops.lors_fwd(x, w, a, b, 2.0, bias, bits)
        y2, _ = ops.lors_fwd(x[1000:].contiguous(), w, a, b, 2.0, bias, bits)
    assert torch.equal(y2, y1[1000:])
    assert _rel(y, y1.double().cpu().numpy()) <= 1e-2


class _env:
    def __init__(self, k, v):
        self.k, self.v = k, v

    def __enter__(self):
        self.old = os.environ.get(self.k)
        os.environ[self.k] = self.v

    def __exit__(self, *exc):
        if self.old is None:
            os.environ.pop(self.k, None)
        else:
            os.environ[self.k] = self.old


@pytest.mark.gpu
@pytest.mark.parametrize("L,R,C,r", [(1024, 1024, 16384, 16),     # fwd: 16 tiles, each split in 2 along K
                                     (512, 2048, 12288, 16),      # fwd: 16 tiles split
                                     (4096, 4096, 11008, 64),     # fwd: 176 tiles, a 28-tile tail split
                                     (2048, 11008, 8192, 32),     # dX: 176 tiles, tail split (K = 11008)
                                     (4096, 4096, 4096, 16),      # 176 tiles at K = 4096 (64 k-steps)
                                     (777, 512, 8192, 8)])        # fwd: 8 ragged tiles split
def test_tail_split_parity_and_determinism(P, L, R, C, r):
    """Persistent walk with the last wave's tiles cut along K (fp32 partials summed
    by the last part to finish): forward and dX against a torch fp32 reference and
    against the unsplit walk, bit-identical from run to run."""
    from paper_2501_08582_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(L + r)
    w = torch.randn(R, C, device="cuda", generator=g) * 0.02
    w = torch.where(w.abs() < 0.015, torch.zeros_like(w), w).bfloat16()
    a = (torch.randn(R, r, device="cuda", generator=g) * 0.05).bfloat16()
    b = (torch.randn(r, C, device="cuda", generator=g) * 0.3).bfloat16()
    x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
    dy = torch.randn(L, R, device="cuda", generator=g).bfloat16()
    bias = (torch.randn(R, device="cuda", generator=g) * 0.1).bfloat16()
    wf, af, bf, xf, dyf = (t.float() for t in (w, a, b, x, dy))
    weff = torch.where(wf != 0, wf + 2.0 * (af @ bf), torch.zeros_like(wf))
    yref = (xf @ weff.t() + bias.float()).double().cpu().numpy()
    dxref = (dyf @ weff).double().cpu().numpy()
    outs = []
    for _ in range(3):
        y, _ = ops.lors_fwd(x, w, a, b, 2.0, bias)
        dx = ops.lors_bwd(x, w, a, b, dy, 2.0, with_bias=True, overlap=False)[0]
        outs.append((y, dx))
    with _env("LORS_NO_TAIL_SPLIT", "1"):
        y0, _ = ops.lors_fwd(x, w, a, b, 2.0, bias)
        dx0 = ops.lors_bwd(x, w, a, b, dy, 2.0, with_bias=True, overlap=False)[0]
    torch.cuda.synchronize()
    for y, dx in outs[1:]:
        assert torch.equal(y, outs[0][0]) and torch.equal(dx, outs[0][1])
    y, dx = outs[0]
    assert _rel(y, yref) <= 2e-2 and _rel(dx, dxref) <= 2e-2
    # the split changes only the fp32 summation order: bf16 outputs within one ulp-ish
    assert float((y.float() - y0.float()).abs().max()) <= 2 ** -6 * float(y0.float().abs().max())
    assert float((dx.float() - dx0.float()).abs().max()) <= 2 ** -6 * float(dx0.float().abs().max())


@pytest.mark.gpu
@pytest.mark.parametrize("L,R,C,r", [(1000, 3000, 512, 24), (4096, 11008, 1024, 64), (300, 256, 256, 16)])
def test_q_da_pass_partitions(P, L, R, C, r):
    """The one-pass Q / dA kernel (K4b) under different R-group sizes (ragged tokens
    and rows, one to many groups): dA / dB against a torch fp32 reference of
    lors_backward's da / db (adapters.py:396-399)."""
    from paper_2501_08582_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(L + R + r)
    w = (torch.randn(R, C, device="cuda", generator=g) * 0.02).bfloat16()
    a = (torch.randn(R, r, device="cuda", generator=g) * 0.05).bfloat16()
    b = (torch.randn(r, C, device="cuda", generator=g) * 0.3).bfloat16()
    x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
    dy = torch.randn(L, R, device="cuda", generator=g).bfloat16()
    af, bf, xf, dyf = (t.float() for t in (a, b, x, dy))
    p = (xf @ bf.t()).bfloat16().float()          # P rounded to bf16 as the kernel path does
    q = (dyf @ af).bfloat16().float()
    da_ref = (2.0 * dyf.t() @ p).double().cpu().numpy()
    db_ref = (2.0 * q.t() @ xf).double().cpu().numpy()
    for tr in (None, "1", "2", "5", "24"):
        with _env("LORS_QDA_TR", tr) if tr else _nullenv():
            _, da, db, _ = ops.lors_bwd(x, w, a, b, dy, 2.0, need_dx=False, overlap=False)
        torch.cuda.synchronize()
        assert _rel(da, da_ref) <= 1e-3, tr
        assert _rel(db, db_ref) <= 1e-2, tr


class _nullenv:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


@pytest.mark.gpu
@pytest.mark.parametrize("with_bias,grad_mode,mask_mode", [(False, "ste", "from_w"), (True, "ste", "from_w"),
                                                           (False, "masked", "bits")])
def test_group_node_matches_separate_layers(P, with_bias, grad_mode, mask_mode):
    """LoRSGroupFunction (projections of one input on concurrent streams, one summed
    dX) against the same LoRSLinear layers called one by one: outputs bit-identical,
    adapter / bias / input gradients equal up to fp32 / bf16 summation order."""
    from paper_2501_08582_b200 import LoRSLinear, lors_group
    g = torch.Generator(device="cuda").manual_seed(5)
    C, L = 1024, 1500
    layers = []
    for R, r in ((1024, 16), (512, 16), (2048, 24)):
        w = torch.randn(R, C, device="cuda", generator=g) * 0.02
        w = torch.where(w.abs() < 0.013, torch.zeros_like(w), w).bfloat16()
        a = torch.randn(R, r, device="cuda", generator=g) * 0.05
        b = torch.randn(r, C, device="cuda", generator=g) * 0.2
        bias = torch.randn(R, device="cuda", generator=g) * 0.1 if with_bias else None
        layers.append(LoRSLinear(w, a=a, b=b, alpha=2.0, bias=bias, grad_mode=grad_mode, mask_mode=mask_mode))
    x = torch.randn(3, L // 3, C, device="cuda", generator=g).bfloat16()
    dys = [torch.randn(3, L // 3, m.out_features, device="cuda", generator=g).bfloat16() for m in layers]

    def run(grouped):
        for m in layers:
            m.zero_grad(set_to_none=True)
        xg = x.clone().requires_grad_(True)
        outs = lors_group(layers, xg) if grouped else [m(xg) for m in layers]
        torch.autograd.backward(list(outs), dys)
        torch.cuda.synchronize()
        grads = [(m.a.grad.clone(), m.b.grad.clone(), None if m.bias is None else m.bias.grad.clone())
                 for m in layers]
        return [o.detach().clone() for o in outs], xg.grad.clone(), grads

    o1, gx1, gr1 = run(False)
    o2, gx2, gr2 = run(True)
    for u, v in zip(o1, o2):
        assert torch.equal(u, v)
    assert float((gx1.float() - gx2.float()).norm() / gx1.float().norm()) < 5e-3
    # (P = X b^T and Q = dY a are split-K sums in fp32 rounded to bf16: their
    # atomics' order can flip a rounding, ~1e-5..1e-4 of dA / dB between any two runs)
    for (a1, b1, c1), (a2, b2, c2) in zip(gr1, gr2):
        assert float((a1 - a2).norm() / a1.norm()) < 1e-3
        assert float((b1 - b2).norm() / b1.norm()) < 1e-3
        if c1 is not None:
            assert float((c1.float() - c2.float()).norm() / c1.float().norm()) < 1e-2


@pytest.mark.gpu
def test_overlapped_backward_with_tail_split_is_deterministic(P):
    """The two-stream backward on a shape whose dX walk splits its tail (K = 11008): dX bit-identical
    across runs and to the single-stream call, while other allocations churn between calls (the split's
    workspace must stay owned until the streams are joined)."""
    from paper_2501_08582_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(77)
    L, R, C, r = 2048, 11008, 8192, 32
    w = (torch.randn(R, C, device="cuda", generator=g) * 0.02).bfloat16()
    a = (torch.randn(R, r, device="cuda", generator=g) * 0.05).bfloat16()
    b = (torch.randn(r, C, device="cuda", generator=g) * 0.3).bfloat16()
    x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
    dy = torch.randn(L, R, device="cuda", generator=g).bfloat16()
    ref = ops.lors_bwd(x, w, a, b, dy, 2.0, overlap=False)
    outs = []
    for i in range(3):
        junk = [torch.empty(1 << (18 + k), dtype=torch.uint8, device="cuda") for k in range(4)]
        outs.append(ops.lors_bwd(x, w, a, b, dy, 2.0, overlap=True))
        del junk
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o[0], ref[0])
        for u, v in zip(o[1:3], ref[1:3]):
            assert float((u - v).norm() / v.norm()) < 1e-3


def test_central_finite_differences_fp32(P):
    """Central finite differences through the GPU path (fp32 FFMA mode), the reference's own check
    (test_adapters.py:138-187, bench.py:97-111): loss = <Y, G>; dX against FD of the masked function,
    dA / dB against FD of the unmasked surrogate W + alpha a b (STE).  The loss is linear in each of
    X, a, b, so central differences are exact up to fp32 rounding."""
    from paper_2501_08582_b200 import ops
    rng = np.random.default_rng(7)
    R, C, L, r, alpha, eps = 6, 5, 4, 2, 2.0, 0.25
    w = rng.normal(size=(R, C)) * 0.5
    w[rng.random((R, C)) < 0.4] = 0.0
    a, b = rng.normal(size=(R, r)) * 0.3, rng.normal(size=(r, C)) * 0.3
    x, gy = rng.normal(size=(L, C)), rng.normal(size=(L, R))
    d = lambda t: _dev(t, torch.float32)  # noqa: E731

    def loss(wm, am, bm, xm):
        y, _ = ops.lors_fwd(d(xm), d(wm), d(am), d(bm), alpha)
        return float((y.double().cpu().numpy() * gy).sum())

    dx, da, db, _ = ops.lors_bwd(d(x), d(w), d(a), d(b), d(gy), alpha)
    fd_x = np.zeros_like(x)
    for i in range(L):
        for j in range(C):
            e = np.zeros_like(x)
            e[i, j] = eps
            fd_x[i, j] = (loss(w, a, b, x + e) - loss(w, a, b, x - e)) / (2 * eps)
    # the unmasked surrogate: every entry of W treated as kept (a dense W with the same values where
    # kept and a tiny nonzero elsewhere keeps all positions "on" without changing the kept values)
    w_dense = np.where(w == 0.0, 1e-30, w)
    fd_a, fd_b = np.zeros_like(a), np.zeros_like(b)
    for i in range(R):
        for j in range(r):
            e = np.zeros_like(a)
            e[i, j] = eps
            fd_a[i, j] = (loss(w_dense, a + e, b, x) - loss(w_dense, a - e, b, x)) / (2 * eps)
    for i in range(r):
        for j in range(C):
            e = np.zeros_like(b)
            e[i, j] = eps
            fd_b[i, j] = (loss(w_dense, a, b + e, x) - loss(w_dense, a, b - e, x)) / (2 * eps)
    assert _rel(dx, fd_x) <= 1e-5
    assert _rel(da, fd_a) <= 1e-5
    assert _rel(db, fd_b) <= 1e-5


@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
def test_all_ones_mask_collapses_masked_onto_ste(P, dt):
    """With no pruned entries, the masked-G gradients (sqft_gc) equal the STE ones (lors) -- the
    reference's acceptance criterion (1) collapse (test_acceptance.py:90-148), on both kernels' paths."""
    from paper_2501_08582_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(9)
    L, R, C, r = 700, 512, 768, 16
    w = (torch.randn(R, C, device="cuda", generator=g) * 0.02 + 0.05).to(dt)     # no zeros
    assert bool((w != 0).all())
    a = (torch.randn(R, r, device="cuda", generator=g) * 0.05).to(dt)
    b = (torch.randn(r, C, device="cuda", generator=g) * 0.2).to(dt)
    x = torch.randn(L, C, device="cuda", generator=g).to(dt)
    dy = torch.randn(L, R, device="cuda", generator=g).to(dt)
    s = ops.lors_bwd(x, w, a, b, dy, 2.0, grad_mode="ste", overlap=False)
    m = ops.lors_bwd(x, w, a, b, dy, 2.0, grad_mode="masked", overlap=False)
    tol = 1e-5 if dt == torch.float32 else 2e-2
    assert torch.equal(s[0], m[0])
    for u, v in zip(s[1:3], m[1:3]):
        assert float((u - v).norm() / v.norm()) <= tol


@pytest.mark.parametrize("L", [1, 3, 17, 129])
@pytest.mark.parametrize("grad_mode", ["ste", "masked"])
def test_tiny_token_counts_bf16(P, L, grad_mode):
    """A handful of tokens through every tensor-core kernel (persistent GEMMs, Q/dA pass, K5 pairs):
    forward, dX and adapter gradients against the float64 oracle on the bf16-rounded inputs."""
    from paper_2501_08582_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(L)
    R, C, r = 520, 264, 24
    w = torch.randn(R, C, device="cuda", generator=g) * 0.02
    w = torch.where(w.abs() < 0.012, torch.zeros_like(w), w).bfloat16()
    a = (torch.randn(R, r, device="cuda", generator=g) * 0.05).bfloat16()
    b = (torch.randn(r, C, device="cuda", generator=g) * 0.2).bfloat16()
    x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
    dy = torch.randn(L, R, device="cuda", generator=g).bfloat16()
    y, _ = ops.lors_fwd(x, w, a, b, 2.0)
    dx, da, db, _ = ops.lors_bwd(x, w, a, b, dy, 2.0, grad_mode=grad_mode)
    wn, an, bn, xn, dyn = (t.double().cpu().numpy() for t in (w, a, b, x, dy))
    assert _rel(y, orc.lors_forward(wn, an, bn, xn.T, 2.0).T) <= 2e-2
    ref = (orc.lors_backward(wn, an, bn, xn.T, dyn.T, 2.0) if grad_mode == "ste"
           else orc.sqft_gc_backward(wn, an, bn, xn.T, dyn.T, 2.0))
    assert _rel(dx, ref.dx.T) <= 2e-2
    assert _rel(da, ref.da) <= 2e-2
    assert _rel(db, ref.db) <= 2e-2
