"""Module-level contract of the LoRS linear (GPU).

- Saved set: the reference's lors variant saves X only for backward (adapters.py:372, counted by
  `counted_saved`, adapters.py:584-592, KAT test_adapters.py:68-89: saved = C L); with save_p the
  rank-r product P = X b^T (r L elements) is kept too.  Checked with a saved-tensor hook on the
  autograd node, for the single projection and for the grouped q/k/v node.
- NumericError: the reference raises on any non-finite result (matrix.py:44-45, 53-54;
  train.py:215-217); here the reference-facing API always checks, the module / trainer on request.
"""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2501_08582_b200 as P
    from paper_2501_08582_b200 import _native
    _native.check(_native.load().lors_device_check())
    return P


def _saved_during(fn):
    saved = []

    def pack(t):
        saved.append(t)
        return t

    with torch.autograd.graph.saved_tensors_hooks(pack, lambda t: t):
        out = fn()
    return saved, out


def _layer(P, R=512, C=384, r=16, dt=torch.bfloat16, **kw):
    g = torch.Generator(device="cuda").manual_seed(R + C)
    w = P.prune.prune_rowwise(torch.randn(R, C, device="cuda", generator=g) * 0.02, 0.5).to(dt)
    a = torch.randn(R, r, device="cuda", generator=g) * 0.02
    b = torch.randn(r, C, device="cuda", generator=g) / r ** 0.5
    return P.LoRSLinear(w, a=a, b=b, **kw)


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float32])
def test_saves_only_x(P, dt):
    layer = _layer(P, dt=dt)
    L = 256
    x = torch.randn(2, L // 2, layer.in_features, device="cuda", dtype=dt, requires_grad=True)
    saved, y = _saved_during(lambda: layer(x))
    assert len(saved) == 1
    assert saved[0].numel() == L * layer.in_features == P.predict_cost("lors", layer.out_features,
                                                                        layer.in_features, L, layer.rank).saved_elements
    assert saved[0].data_ptr() == x.data_ptr()          # X itself, not a copy
    y.sum().backward()
    assert layer.a.grad is not None and x.grad is not None


def test_save_p_adds_rank_r_product(P):
    layer = _layer(P, save_p=True)
    L = 256
    x = torch.randn(L, layer.in_features, device="cuda", dtype=torch.bfloat16)
    saved, _ = _saved_during(lambda: layer(x))
    assert sorted(t.numel() for t in saved) == sorted([L * layer.in_features, L * layer.rank])


def test_grouped_node_saves_only_x(P):
    """q/k/v as one LoRSGroupFunction node: one saved tensor, the shared input."""
    from paper_2501_08582_b200.module import groupable, lors_group
    layers = [_layer(P, R=R) for R in (512, 256, 256)]
    assert groupable(layers)
    x = torch.randn(128, 384, device="cuda", dtype=torch.bfloat16, requires_grad=True)
    saved, outs = _saved_during(lambda: lors_group(layers, x))
    assert len(saved) == 1 and saved[0].numel() == x.numel()
    sum(o.float().sum() for o in outs).backward()
    assert all(m.a.grad is not None for m in layers)


def test_numeric_error_reference_api(P):
    """variant_forward on an input holding inf raises NumericError like the reference."""
    w = P.prune.prune_rowwise(torch.randn(64, 48, device="cuda") * 0.02, 0.5)
    layer = P.make_layer(P.SparseWeight(w), 8, "lors")
    x = torch.randn(48, 32, device="cuda")
    x[3, 5] = float("inf")
    with pytest.raises(P.NumericError):
        P.variant_forward(layer, x)


def test_numeric_error_module_opt_in(P):
    layer = _layer(P, check_finite=True)
    x = torch.randn(64, layer.in_features, device="cuda", dtype=torch.bfloat16)
    layer(x)                                             # finite: fine
    x[0, 0] = float("nan")
    with pytest.raises(P.NumericError):
        layer(x)
    quiet = _layer(P)                                     # default: no host sync, no check
    assert not torch.isfinite(quiet(x)).all()


def test_trainer_check_finite(P):
    from paper_2501_08582_b200 import decoder as D
    from paper_2501_08582_b200.trainer import Trainer, synthetic_tokens
    cfg = D.preset("tiny")
    model = D.LoRSDecoder(cfg, device="cuda", seed=0)
    tr = Trainer(model, lr=1e-3, check_finite=True)
    tr.step(synthetic_tokens(cfg.vocab, cfg.batch, cfg.seq, 0, device="cuda"))
    model.embed[0].fill_(float("nan"))
    with pytest.raises(P.NumericError):
        tr.step(torch.zeros(cfg.batch, cfg.seq + 1, dtype=torch.long, device="cuda"))
