"""GPU: the grouped forward (lors_fwd_group) -- G projections of one input in one persistent launch --
gives every projection's output bit for bit as its own lors_fwd (the same tiles, recompute and
weff_pair), masks stay exact, and the argument checks of the C ABI hold.  Per projection the
arithmetic is lors_forward (adapters.py:359-373), checked against the float64 oracle."""

import numpy as np
import pytest
import torch

from oracle import lors_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2501_08582_b200 import ops
    return ops


def _group(G, R, C, r, seed):
    from paper_2501_08582_b200 import prune
    g = torch.Generator(device="cuda").manual_seed(seed)
    w = prune.prune_rowwise(torch.randn(G * R, C, device="cuda", generator=g) * 0.05, 0.5).bfloat16()
    a = (torch.randn(G * R, r, device="cuda", generator=g) * 0.05).bfloat16()
    b = (torch.randn(G * r, C, device="cuda", generator=g) / r ** 0.5).bfloat16()
    return w, a, b


@pytest.mark.parametrize("G,R,C,r,L", [(3, 256, 128, 16, 300), (2, 512, 320, 32, 384), (3, 256, 256, 64, 1000),
                                       (2, 768, 192, 16, 1), (4, 256, 64, 16, 130)])
@pytest.mark.parametrize("alpha", [2.0, 1.0 / 3.0])
def test_group_matches_per_projection_bitwise(ops, G, R, C, r, L, alpha):
    w, a, b = _group(G, R, C, r, seed=G * 1000 + R + C + r + L)
    x = torch.randn(L, C, device="cuda").bfloat16()
    y = ops.lors_fwd_group(x, w, a, b, G, alpha)
    assert y.shape == (G, L, R)
    for i in range(G):
        yi, _ = ops.lors_fwd(x, w[i * R:(i + 1) * R].contiguous(), a[i * R:(i + 1) * R].contiguous(),
                             b[i * r:(i + 1) * r].contiguous(), alpha)
        assert torch.equal(y[i], yi), f"projection {i} differs from its own lors_fwd"


def test_group_against_oracle_and_mask(ops):
    G, R, C, r, L = 3, 256, 192, 16, 200
    w, a, b = _group(G, R, C, r, seed=7)
    x = torch.randn(L, C, device="cuda").bfloat16()
    y = ops.lors_fwd_group(x, w, a, b, G, 2.0).float().cpu().numpy()
    xf = x.float().cpu().numpy().astype(np.float64)
    for i in range(G):
        wi = w[i * R:(i + 1) * R].float().cpu().numpy().astype(np.float64)
        ai = a[i * R:(i + 1) * R].float().cpu().numpy().astype(np.float64)
        bi = b[i * r:(i + 1) * r].float().cpu().numpy().astype(np.float64)
        ref = orc.lors_forward(wi, ai, bi, xf.T, 2.0).T
        err = np.linalg.norm(y[i] - ref) / np.linalg.norm(ref)
        assert err <= 2e-2, f"projection {i}: rel-L2 {err}"
    # identity input: Y = W_eff^T rows -> exactly +0 wherever W == 0
    eye = torch.eye(C, device="cuda").bfloat16()
    ye = ops.lors_fwd_group(eye, w, a, b, G, 2.0)
    for i in range(G):
        weff_t = ye[i]                                   # [C, R] = W_eff^T
        zero = (w[i * R:(i + 1) * R] == 0).T
        assert torch.all(weff_t[zero].view(torch.int16) == 0)


def test_group_argument_checks(ops):
    from paper_2501_08582_b200.errors import ArgumentError, ShapeError
    w, a, b = _group(2, 200, 128, 16, seed=1)            # R % 256 != 0
    x = torch.randn(64, 128, device="cuda").bfloat16()
    with pytest.raises(ArgumentError):
        ops.lors_fwd_group(x, w, a, b, 2, 2.0)
    w, a, b = _group(2, 256, 128, 24, seed=2)            # r not 16 / 32 / 64
    with pytest.raises(ArgumentError):
        ops.lors_fwd_group(x, w, a, b, 2, 2.0)
    w, a, b = _group(2, 256, 128, 16, seed=3)
    with pytest.raises(ShapeError):
        ops.lors_fwd_group(x, w, a, b[:-1], 2, 2.0)


def test_decoder_grouped_forward_is_bitwise_the_per_projection_path(ops, monkeypatch):
    """The decoder packs q/k/v and gate/up weights ([G R, C] buffers) so their forwards run as one
    grouped launch; loss and every adapter gradient equal the concurrent per-projection path's."""
    from paper_2501_08582_b200 import decoder as dec
    from paper_2501_08582_b200.trainer import synthetic_tokens
    cfg = dec.preset("tiny", n_kv_heads=4)          # q, k, v all 256 x 256: one group
    m = dec.LoRSDecoder(cfg, device="cuda", seed=3)
    layer = m.layers[0].proj
    assert layer["q"].weight._base is not None and layer["q"].weight._base is layer["v"].weight._base
    assert layer["gate"].weight._base is layer["up"].weight._base
    tok = synthetic_tokens(cfg.vocab, cfg.batch, cfg.seq, step=0, device="cuda")
    monkeypatch.setenv("LORS_DETERMINISTIC", "1")   # dA / dB bitwise reproducible run to run
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("LORS_GROUP_FWD", flag)
        m.zero_grad(set_to_none=True)
        loss = m.loss(tok)
        loss.backward()
        out[flag] = (loss.detach().clone(), {n: p.grad.detach().clone() for n, p in m.named_parameters()})
    assert torch.equal(out["1"][0], out["0"][0])      # the forward is bit-identical
    for n, g in out["0"][1].items():                  # (attention's backward is not bitwise reproducible)
        g1 = out["1"][1][n]
        assert float((g1 - g).double().norm()) <= 1e-3 * float(g.double().norm()) + 1e-30, n


@pytest.mark.parametrize("L,R,C,r", [(4096, 4096, 11008, 64), (2048, 11008, 8192, 32)])
def test_no_tail_split_flag_is_the_unsplit_walk(ops, L, R, C, r):
    """LORS_FLAG_NO_TAIL_SPLIT (ops.set_tail_split(False), what Trainer steps use) runs the forward and
    dX walks unsplit: bit-identical to the LORS_NO_TAIL_SPLIT build-time switch, and the flag is
    restored by the trainer's step."""
    import os
    g = torch.Generator(device="cuda").manual_seed(L + r)
    w = torch.randn(R, C, device="cuda", generator=g) * 0.02
    w = torch.where(w.abs() < 0.015, torch.zeros_like(w), w).bfloat16()
    a = (torch.randn(R, r, device="cuda", generator=g) * 0.05).bfloat16()
    b = (torch.randn(r, C, device="cuda", generator=g) * 0.3).bfloat16()
    x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
    dy = torch.randn(L, R, device="cuda", generator=g).bfloat16()
    prev = ops.set_tail_split(False)
    try:
        y1, _ = ops.lors_fwd(x, w, a, b, 2.0)
        dx1 = ops.lors_bwd(x, w, a, b, dy, 2.0, overlap=False)[0]
    finally:
        ops.set_tail_split(prev)
    os.environ["LORS_NO_TAIL_SPLIT"] = "1"
    try:
        y0, _ = ops.lors_fwd(x, w, a, b, 2.0)
        dx0 = ops.lors_bwd(x, w, a, b, dy, 2.0, overlap=False)[0]
    finally:
        os.environ.pop("LORS_NO_TAIL_SPLIT", None)
    assert torch.equal(y1, y0) and torch.equal(dx1, dx0)
