"""Bitwise run-to-run reproducibility of the adapter gradients (LORS_FLAG_DETERMINISTIC).

The reference replays a fine-tuning run bitwise (/root/reference/pkg/tests/test_train.py:169-178,
test_acceptance.py:373-392).  The fast backward sums split-K partials with atomics and TMA
reduce-adds, whose order varies; the deterministic mode writes every split's partial to a
workspace slab and sums the slabs in a fixed order, so dA / dB (and the forward, dX, which never
used atomics) are identical bit for bit across runs, and still match the oracle.
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


def _inputs(R, C, L, r, seed):
    from paper_2501_08582_b200 import prune
    g = torch.Generator(device="cuda").manual_seed(seed)
    w = prune.prune_rowwise(torch.randn(R, C, device="cuda", generator=g) * 0.02, 0.5)
    a = torch.randn(R, r, device="cuda", generator=g) * 0.02
    b = torch.randn(r, C, device="cuda", generator=g) / r ** 0.5
    x = torch.randn(L, C, device="cuda", generator=g)
    dy = torch.randn(L, R, device="cuda", generator=g)
    return [t.to(torch.bfloat16).contiguous() for t in (w, a, b, x, dy)]


def _bits(t):
    return t.contiguous().view(torch.int32).clone()


# shapes whose rank-r products split along K (L = 4096 and 8192 tokens; R, C up to 11008)
@pytest.mark.parametrize("R,C,L,r", [(4096, 4096, 4096, 64), (11008, 4096, 8192, 64), (4096, 11008, 4096, 16),
                                     (1024, 512, 640, 8)])
@pytest.mark.parametrize("grad_mode", ["ste", "masked"])
def test_adapter_grads_bitwise_reproducible(ops, R, C, L, r, grad_mode):
    w, a, b, x, dy = _inputs(R, C, L, r, seed=R + L + r)
    runs = []
    for i in range(3):
        scratch = torch.empty(int(64e6) * (i + 1), dtype=torch.uint8, device="cuda")   # move the allocator around
        dx, da, db, _ = ops.lors_bwd(x, w, a, b, dy, 2.0, grad_mode=grad_mode, deterministic=True)
        torch.cuda.synchronize()
        runs.append((dx.view(torch.int16).clone(), _bits(da), _bits(db)))
        del scratch, dx, da, db
    for other in runs[1:]:
        for u, v in zip(runs[0], other):
            assert torch.equal(u, v)
    # and still the reference's numbers (oracle on the bf16 inputs)
    _, da, db, _ = ops.lors_bwd(x, w, a, b, dy, 2.0, grad_mode=grad_mode, deterministic=True, need_dx=False)
    wd, ad, bd, xd, dyd = (t.double().cpu().numpy() for t in (w, a, b, x, dy))
    fn = orc.lors_adapter_grads if grad_mode == "ste" else orc.sqft_gc_adapter_grads
    da_ref, db_ref = fn(wd, ad, bd, xd.T, dyd.T, 2.0)
    assert orc.rel_l2(da.double().cpu().numpy(), da_ref) <= 2e-2
    assert orc.rel_l2(db.double().cpu().numpy(), db_ref) <= 2e-2


def test_fp32_adapter_grads_bitwise_reproducible(ops):
    """The fp32 parity mode under LORS_FLAG_DETERMINISTIC: P, Q, dA, dB each from one CTA per output
    tile in k order (the fast mode splits them along the reduction with fp32 atomics)."""
    g = torch.Generator(device="cuda").manual_seed(3)
    R, C, L, r = 2048, 1024, 2048, 16
    w = (torch.randn(R, C, device="cuda", generator=g) * 0.02) * (torch.rand(R, C, device="cuda", generator=g) > 0.5)
    a = torch.randn(R, r, device="cuda", generator=g) * 0.05
    b = torch.randn(r, C, device="cuda", generator=g) / r ** 0.5
    x = torch.randn(L, C, device="cuda", generator=g)
    dy = torch.randn(L, R, device="cuda", generator=g)
    runs = []
    for _ in range(3):
        _, da, db, _ = ops.lors_bwd(x, w, a, b, dy, 2.0, need_dx=False, deterministic=True)
        torch.cuda.synchronize()
        runs.append((_bits(da), _bits(db)))
    for other in runs[1:]:
        for u, v in zip(runs[0], other):
            assert torch.equal(u, v)
    _, da_f, db_f, _ = ops.lors_bwd(x, w, a, b, dy, 2.0, need_dx=False, deterministic=False)
    for u, v in ((da_f, da), (db_f, db)):
        assert float((u - v).norm() / v.norm()) < 1e-5


def test_fast_and_deterministic_modes_agree(ops):
    """Same sums in another order: the two modes differ only by fp32 summation order, which can
    flip the bf16 rounding of a few intermediate P / Q entries (adapters.py:396-397 products are
    rounded to the compute dtype before dA / dB): relative differences ~1e-4."""
    w, a, b, x, dy = _inputs(11008, 4096, 8192, 64, seed=7)
    _, da0, db0, _ = ops.lors_bwd(x, w, a, b, dy, 2.0, need_dx=False, deterministic=False)
    _, da1, db1, _ = ops.lors_bwd(x, w, a, b, dy, 2.0, need_dx=False, deterministic=True)
    torch.cuda.synchronize()
    for u, v in ((da0, da1), (db0, db1)):
        assert float((u - v).norm() / v.norm()) < 1e-3


def test_training_replays_bitwise(ops, monkeypatch):
    """Two identical fine-tuning runs of a small LoRS decoder (fused AdamW on the adapters) end
    with bitwise identical adapters and losses (test_train.py:169-178)."""
    from paper_2501_08582_b200 import decoder as D
    from paper_2501_08582_b200.trainer import Trainer, synthetic_tokens
    monkeypatch.setenv("LORS_DETERMINISTIC", "1")
    cfg = D.preset("tiny", dim=512, ffn=1024, n_heads=8, n_kv_heads=8, seq=256, batch=4)

    def run():
        model = D.LoRSDecoder(cfg, device="cuda", seed=3)
        tr = Trainer(model, lr=1e-3)
        losses = [tr.step(synthetic_tokens(cfg.vocab, cfg.batch, cfg.seq, s, device="cuda")) for s in range(6)]
        torch.cuda.synchronize()
        return torch.stack(losses).cpu(), [_bits(p.detach()) for p in model.adapter_parameters()]

    from torch.nn.attention import SDPBackend, sdpa_kernel
    with sdpa_kernel(SDPBackend.MATH):     # attention's own backward without atomics
        l0, p0 = run()
        l1, p1 = run()
    assert torch.equal(l0.view(torch.int32), l1.view(torch.int32))
    assert all(torch.equal(u, v) for u, v in zip(p0, p1))
    assert np.isfinite(l0.numpy()).all()
