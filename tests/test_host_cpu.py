"""Host-side logic that runs without a GPU: pruning producers (bitwise vs the
reference fixtures), the cost model, module/adapter validation."""

import os

import numpy as np
import pytest
import torch

import paper_2501_08582_b200 as P
from oracle import lors_oracle as orc

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_prune_producers_bitwise_vs_reference_fixtures():
    d = dict(np.load(os.path.join(GOLD, "prune_kats.npz")))
    for i in range(4):
        w = torch.from_numpy(d[f"p{i}_w"])
        np.testing.assert_array_equal(P.prune_rowwise(w, 0.5).numpy(), d[f"p{i}_rowwise"])
        if f"p{i}_two_four" in d:
            got = P.prune_two_four(w)
            np.testing.assert_array_equal(got.numpy(), d[f"p{i}_two_four"])
            assert P.two_four_valid(got)
    np.testing.assert_array_equal(P.prune_magnitude(torch.tensor([[1.0, -4.0], [2.0, 3.0]]), 0.5).numpy(),
                                  d["kat_magnitude"])


@pytest.mark.parametrize("seed", range(10))
def test_prune_rowwise_matches_oracle_with_ties(seed):
    rng = np.random.default_rng(seed)
    w = rng.normal(size=(7, 12))
    w[:, 3] = w[:, 2]
    w[2] = 0.5
    np.testing.assert_array_equal(P.prune_rowwise(torch.from_numpy(w), 0.5).numpy(), orc.prune_rowwise(w, 0.5))
    np.testing.assert_array_equal(P.prune_two_four(torch.from_numpy(w)).numpy(), orc.prune_two_four(w))


def test_sparse_weight_normalises_negative_zero_and_validates():
    sw = P.SparseWeight(torch.tensor([[-0.0, 1.0, 0.0, 2.0]]), pattern="two_four")
    assert torch.signbit(sw.values).tolist() == [[False, False, False, False]]
    with pytest.raises(P.ArgumentError):
        P.SparseWeight(torch.ones(1, 4), pattern="two_four")
    with pytest.raises(P.ArgumentError):
        P.SparseWeight(torch.ones(1, 4), pattern="weird")


def test_cost_model_matches_oracle_and_kat():
    assert (P.predict_cost("lors", 4, 4, 4, 1).macs_forward, P.predict_cost("lors", 4, 4, 4, 1).macs_backward,
            P.predict_cost("lors", 4, 4, 4, 1).saved_elements) == (96, 160, 16)
    rng = np.random.default_rng(11)
    for _ in range(50):
        R, C, L, r = (int(v) for v in rng.integers(1, 50, size=4))
        for variant in ("lors", "sqft_gc", "sqft", "lora"):
            p = P.predict_cost(variant, R, C, L, r)
            assert (p.macs_forward, p.macs_backward, p.saved_elements) == orc.predict_cost(variant, R, C, L, r)
    with pytest.raises(P.ArgumentError):
        P.predict_cost("nope", 1, 1, 1, 1)
    # cfg2 = 1520.87 GFLOP per fwd+bwd step
    assert abs(P.predict_cost("lors", 11008, 4096, 8192, 64).flops / 1e9 - 1520.87) < 0.01
    assert abs(P.predict_cost("lors", 4096, 4096, 2048, 16).flops / 1e9 - 139.65) < 0.01


def test_cost_model_fault_injection():
    P.FAULT_INJECTION["cost_model_off_by_one"] = True
    try:
        assert P.predict_cost("lors", 4, 4, 4, 1).macs_backward == 161
    finally:
        P.FAULT_INJECTION["cost_model_off_by_one"] = False


def test_module_constructor_validation_cpu():
    w = torch.randn(8, 6)
    with pytest.raises(P.ArgumentError):
        P.LoRSLinear(w)
    with pytest.raises(P.ArgumentError):
        P.LoRSLinear(w, rank=7)
    with pytest.raises(P.ShapeError):
        P.LoRSLinear(w, a=torch.zeros(8, 2), b=torch.zeros(3, 6))
    with pytest.raises(P.ArgumentError):
        P.LoRSLinear(w, rank=2, alpha=0.0)
    with pytest.raises(P.ArgumentError):
        P.LoRSLinear(w, rank=2, grad_mode="other")
    m = P.LoRSLinear(w, rank=2, bias=torch.zeros(8))
    assert sorted(m.state_dict().keys()) == ["a", "b", "bias", "weight"]
    assert not m.weight.requires_grad and m.a.requires_grad and m.b.requires_grad
    assert float(m.a.abs().sum()) == 0.0 and float(m.b.abs().sum()) == 0.0  # make_layer zero init


def test_adapter_pair_validation_cpu():
    with pytest.raises(P.ShapeError):
        P.AdapterPair(torch.zeros(4, 2), torch.zeros(3, 5))
    with pytest.raises(P.ArgumentError):
        P.AdapterPair(torch.zeros(4, 5), torch.zeros(5, 4))
    with pytest.raises(P.ArgumentError):
        P.AdapterPair(torch.zeros(4, 2), torch.zeros(2, 5), alpha=-1.0)


def test_fit_rank_r_rows_matches_reference_svd_fixtures():
    """GPU init's SVD step (run here on CPU tensors) vs the reference's Jacobi SVD."""
    from paper_2501_08582_b200.init import fit_rank_r_rows, singular_tail
    d = dict(np.load(os.path.join(GOLD, "svd_init.npz")))
    for i, r in enumerate((3, 4, 5)):
        dw = torch.from_numpy(d[f"s{i}_dw"])
        for lim in (2048, 1):   # exact SVD path and the eigh (large-layer) path
            b = fit_rank_r_rows(dw, r, exact_limit=lim)
            np.testing.assert_allclose(b.double().numpy(), d[f"s{i}_b"], atol=2e-5)
        assert abs(singular_tail(dw, r) - float(d[f"s{i}_tail"])) < 1e-9


def test_pack_group_weights_host_logic():
    """pack_group_weights moves equal-shape frozen weights into one [G R, C] buffer (values, shapes and
    state_dict names unchanged); packed_weights accepts exactly the layouts lors_fwd_group can run."""
    import torch
    from paper_2501_08582_b200.module import LoRSLinear, pack_group_weights, packed_weights
    g = torch.Generator().manual_seed(0)
    ws = [torch.randn(256, 64, generator=g).bfloat16() for _ in range(3)]
    ls = [LoRSLinear(w, rank=16) for w in ws]
    before = [m.weight.clone() for m in ls]
    keys = [sorted(m.state_dict()) for m in ls]
    assert pack_group_weights(ls)
    base = ls[0].weight._base
    assert base is not None and tuple(base.shape) == (768, 64)
    assert all(m.weight._base is base for m in ls)
    assert all(torch.equal(m.weight, w) for m, w in zip(ls, before))
    assert [sorted(m.state_dict()) for m in ls] == keys
    args = ([m.weight for m in ls], [None] * 3, [m.a for m in ls], [m.params() for m in ls])
    assert packed_weights(*args) is base
    assert packed_weights(args[0][:2], args[1][:2], args[2][:2], args[3][:2]) is None      # not the whole buffer
    assert packed_weights(args[0], [None, torch.zeros(256), None], args[2], args[3]) is None   # bias
    # unequal shapes are left alone
    assert not pack_group_weights([LoRSLinear(torch.randn(256, 64).bfloat16(), rank=16),
                                   LoRSLinear(torch.randn(512, 64).bfloat16(), rank=16)])
