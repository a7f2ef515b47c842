"""LLaMA-shaped LoRS decoder and its data-parallel trainer.

CPU: the model-level cost figures of SURVEY 8 d3 / BASELINE.md, the decoder's
structure with the test-only torch projection, and the world-size-2 gloo
trainer (DDP step == single-process step on the concatenated batch).
GPU: the native decoder against the torch and float64-oracle projections, the
2:4 sparse-tensor-core forward inside the model, mask preservation through
training, and a model-level loss curve.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
import torch.nn.functional as F

from paper_2501_08582_b200 import decoder as dec
from paper_2501_08582_b200.trainer import Trainer, synthetic_tokens


# --------------------------------------------------------------------------- cost KATs

@pytest.mark.parametrize("name,adapters_m,gflop_tok,roof_spec", [
    ("llama2-7b", 39.98, 27.64, 81418),
    ("llama3-8b", 167.77, 33.01, 86431),
    ("llama2-13b", 250.35, 59.09, 38081),
])
def test_model_cost_matches_survey(name, adapters_m, gflop_tok, roof_spec):
    cfg = dec.preset(name)
    assert abs(dec.adapter_param_count(cfg) / 1e6 - adapters_m) < 0.01
    assert abs(dec.flops_per_token(cfg)["total"] / 1e9 - gflop_tok) < 0.01
    assert abs(dec.roofline_tokens_per_s(cfg, 2250.0, 4500.0) - roof_spec) / roof_spec < 2e-3


def test_cfg3_cost_breakdown():
    f = dec.flops_per_token(dec.preset("llama2-7b"))
    assert abs(f["linear"] / 1e9 - 26.06) < 0.01
    assert abs(f["attention"] / 1e9 - 0.94) < 0.01
    assert abs(f["head"] / 1e9 - 0.52) < 0.01
    assert abs(f["recompute"] / 1e9 - 0.11) < 0.01


# --------------------------------------------------------------------------- CPU structure

def _tiny(**kw):
    return dec.preset("tiny", **kw)


def test_tiny_decoder_structure_cpu():
    from ref_linear import torch_factory
    cfg = _tiny(dtype=torch.float32)
    m = dec.LoRSDecoder(cfg, device="cpu", linear_factory=torch_factory)
    names = sorted(n for n, _ in m.named_parameters())
    assert len(names) == 2 * 7 * cfg.n_layers and all(n.endswith((".a", ".b")) for n in names)
    assert sum(p.numel() for p in m.parameters()) == dec.adapter_param_count(cfg)
    for proj in m.projections():
        w = proj.weight
        assert float((w == 0).float().mean()) == pytest.approx(0.5, abs=1e-6)   # per-row 50%
    tok = synthetic_tokens(cfg.vocab, cfg.batch, cfg.seq, step=0, device="cpu")
    loss = m.loss(tok)
    assert abs(float(loss.detach()) - np.log(cfg.vocab)) < 1.0
    loss.backward()
    assert all(p.grad is not None for p in m.parameters())


def test_two_four_preset_prunes_two_of_four_cpu():
    from ref_linear import torch_factory
    from paper_2501_08582_b200.prune import two_four_valid
    m = dec.LoRSDecoder(_tiny(dtype=torch.float32, sparsity="two_four"), device="cpu", linear_factory=torch_factory)
    for proj in m.projections():
        assert two_four_valid(proj.weight)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ddp_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from ref_linear import torch_factory
        cfg = _tiny(dtype=torch.float32, n_layers=1, seq=32)
        torch.manual_seed(0)
        m = dec.LoRSDecoder(cfg, device="cpu", linear_factory=torch_factory, seed=0)
        with torch.no_grad():
            for p in m.parameters():
                p.normal_(0, 0.05)
        tr = Trainer(m, lr=1e-2, overlap=True, bucket_bytes=4096)
        for step in range(2):
            tr.step(synthetic_tokens(cfg.vocab, cfg.batch, cfg.seq, step=step, rank=rank, device="cpu"))
        q.put((rank, {n: p.detach().numpy().copy() for n, p in m.named_parameters()}))
    finally:
        dist.destroy_process_group()


def test_trainer_ddp_world2_equals_single_process():
    """Two gloo ranks with overlapped bucketed all-reduce end with exactly the adapters
    one process gets from the two ranks' batches concatenated (the mean loss over
    equal-size shards has the averaged gradient)."""
    from ref_linear import torch_factory
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ddp_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = _tiny(dtype=torch.float32, n_layers=1, seq=32)
    torch.manual_seed(0)
    m = dec.LoRSDecoder(cfg, device="cpu", linear_factory=torch_factory, seed=0)
    with torch.no_grad():
        for p in m.parameters():
            p.normal_(0, 0.05)
    tr = Trainer(m, lr=1e-2)
    for step in range(2):
        tok = torch.cat([synthetic_tokens(cfg.vocab, cfg.batch, cfg.seq, step=step, rank=r, device="cpu")
                         for r in range(world)])
        tr.step(tok)
    for n, p in m.named_parameters():
        for r in range(world):
            np.testing.assert_allclose(res[r][n], p.detach().numpy(), rtol=1e-5, atol=1e-6)
    for n in res[0]:
        np.testing.assert_array_equal(res[0][n], res[1][n])


# --------------------------------------------------------------------------- GPU

def _native_and_ref(cfg, ref_factory, ref_dtype, ref_device, seed=0):
    m = dec.LoRSDecoder(cfg, device="cuda", seed=seed)
    ref = dec.LoRSDecoder(dec.replace(cfg, dtype=ref_dtype), device=ref_device, linear_factory=ref_factory,
                          seed=seed)
    ref.load_state_dict(m.state_dict())
    return m, ref


def _grads(model):
    return {n: p.grad.detach().double().cpu() for n, p in model.named_parameters()}


def _rel(a, b):
    return float((a - b).norm() / b.norm())


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-4), (torch.bfloat16, 2e-2)])
def test_native_decoder_matches_torch_reference(dtype, tol):
    from ref_linear import torch_factory
    cfg = _tiny(dtype=dtype)
    m, ref = _native_and_ref(cfg, torch_factory, torch.float32, "cuda")
    tok = synthetic_tokens(cfg.vocab, cfg.batch, cfg.seq, step=0, device="cuda")
    l1 = m.loss(tok)
    l1.backward()
    l2 = ref.loss(tok)
    l2.backward()
    assert abs(float(l1.detach()) - float(l2.detach())) / float(l2.detach()) < tol
    g1, g2 = _grads(m), _grads(ref)
    worst = max(_rel(g1[n], g2[n]) for n in g2)
    assert worst < (5 * tol if dtype == torch.bfloat16 else tol), worst


@pytest.mark.gpu
def test_native_decoder_sparse24_forward_matches_dense_masked():
    cfg = _tiny(sparsity="two_four", dim=256, ffn=512)
    m = dec.LoRSDecoder(cfg, device="cuda", seed=1)
    dense = dec.LoRSDecoder(cfg, device="cuda", seed=1,
                            linear_factory=dec.lors_factory(cfg, seed=1, sparse24_forward=False))
    dense.load_state_dict(m.state_dict())
    assert all(p.sparse24 for p in m.projections()) and not any(p.sparse24 for p in dense.projections())
    tok = synthetic_tokens(cfg.vocab, cfg.batch, cfg.seq, step=0, device="cuda")
    with torch.no_grad():
        a, b = m(tok[:, :-1]).float(), dense(tok[:, :-1]).float()
    assert _rel(a.cpu().double(), b.cpu().double()) < 1e-2


@pytest.mark.gpu
def test_decoder_training_preserves_masks_bit_exactly():
    from paper_2501_08582_b200 import ops
    cfg = _tiny()
    m = dec.LoRSDecoder(cfg, device="cuda")
    tr = Trainer(m, lr=1e-2)
    for step in range(3):
        tr.step(synthetic_tokens(cfg.vocab, cfg.batch, cfg.seq, step=step, device="cuda"))
    for proj in m.projections():
        weff = proj.effective_weight()
        assert torch.all(weff[proj.weight == 0].view(torch.int16) == 0)
        assert torch.count_nonzero(weff) <= torch.count_nonzero(proj.weight)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-4), (torch.bfloat16, 1e-2)])
def test_decoder_loss_curve_vs_float64_oracle(dtype, tol):
    """a reduced LLaMA-shaped decoder trained 30 steps through the native
    kernels tracks the same decoder whose projections call the float64 oracle on the
    CPU (test-only shim) within 1% (bf16) / 1e-4 (fp32)."""
    from ref_linear import oracle_factory
    cfg = _tiny(dtype=dtype, n_layers=2, seq=64)
    m, ref = _native_and_ref(cfg, oracle_factory, torch.float64, "cpu")
    t1, t2 = Trainer(m, lr=1e-3), Trainer(ref, lr=1e-3)
    l1, l2 = [], []
    tok = synthetic_tokens(cfg.vocab, cfg.batch, cfg.seq, step=0, device="cpu")   # fit one batch
    for step in range(30):
        l1.append(float(t1.step(tok.cuda())))
        l2.append(float(t2.step(tok)))
    l1, l2 = np.array(l1), np.array(l2)
    rel = np.abs(l1 - l2) / l2
    print(f"{dtype}: decoder loss {l2[0]:.4f} -> {l2[-1]:.4f}; max rel deviation {rel.max():.2e}")
    assert l2[-1] < l2[0] - 1.0
    assert rel.max() <= tol


@pytest.mark.gpu
def test_fused_rope_matches_torch_formula():
    """ops.rope / RopeFunction (fused RoPE + head transpose) against the torch
    rotate-half formula in fp32, forward and backward, GQA head counts."""
    cfg = dec.preset("tiny", dtype=torch.bfloat16, seq=64)
    cos, sin = dec.rope_tables(cfg, "cuda")
    g = torch.Generator(device="cuda").manual_seed(3)
    for H in (4, 2):
        x = torch.randn(2, 64, H, cfg.head_dim, device="cuda", generator=g).bfloat16().requires_grad_(True)
        gy = torch.randn(2, H, 64, cfg.head_dim, device="cuda", generator=g).bfloat16()
        y = dec.rope_heads(x, cos, sin)
        y.backward(gy)
        xr = x.detach().float().requires_grad_(True)
        yr = dec.apply_rope(xr.transpose(1, 2), cos.float(), sin.float())
        yr.backward(gy.float())
        assert y.shape == (2, H, 64, cfg.head_dim) and y.transpose(1, 2).is_contiguous()   # heads as strides
        assert float((y.float() - yr).norm() / yr.norm()) < 5e-3
        assert float((x.grad.float() - xr.grad).norm() / xr.grad.norm()) < 5e-3
        # the transposing layouts of the same kernel
        from paper_2501_08582_b200 import ops
        y0 = ops.rope(x.detach(), cos, sin, layout=0)
        assert y0.is_contiguous() and torch.equal(y0, y.detach().contiguous())
        y1 = ops.rope(y0, cos, sin, layout=1, inverse=True)
        assert float((y1.float() - x.detach().float()).norm() / x.detach().float().norm()) < 1e-2


@pytest.mark.gpu
def test_fused_swiglu_matches_torch():
    """ops.swiglu / SwiGLUFunction against silu(g) * u in fp32, forward and backward."""
    g0 = torch.Generator(device="cuda").manual_seed(5)
    gate = (torch.randn(3, 100, 88, device="cuda", generator=g0) * 2).bfloat16().requires_grad_(True)
    up = torch.randn(3, 100, 88, device="cuda", generator=g0).bfloat16().requires_grad_(True)
    dh = torch.randn(3, 100, 88, device="cuda", generator=g0).bfloat16()
    h = dec.swiglu(gate, up)
    h.backward(dh)
    gr, ur = gate.detach().float().requires_grad_(True), up.detach().float().requires_grad_(True)
    hr = torch.nn.functional.silu(gr) * ur
    hr.backward(dh.float())
    rel = lambda a, b: float((a.float() - b).norm() / b.norm())  # noqa: E731
    assert rel(h, hr) < 5e-3 and rel(gate.grad, gr.grad) < 5e-3 and rel(up.grad, ur.grad) < 5e-3


@pytest.mark.gpu
def test_flat_adamw_matches_torch_adamw():
    """trainer.FlatAdamW (one fused launch, bf16 compute copies refreshed in place)
    against torch.optim.AdamW on identical parameters and gradients for several
    steps (decoupled weight decay, bias correction); the compute copies equal the
    rounded masters and are what compute_copy returns."""
    from paper_2501_08582_b200.module import compute_copy
    from paper_2501_08582_b200.trainer import FlatAdamW
    g = torch.Generator(device="cuda").manual_seed(9)
    shapes = [(64, 16), (16, 48), (300, 8), (8, 300), (7,)]
    p1 = [torch.nn.Parameter(torch.randn(s, device="cuda", generator=g)) for s in shapes]
    p2 = [torch.nn.Parameter(p.detach().clone()) for p in p1]
    o1 = FlatAdamW(p1, lr=3e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.05)
    o2 = torch.optim.AdamW(p2, lr=3e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.05)
    for step in range(6):
        for a, b in zip(p1, p2):
            gr = torch.randn(a.shape, device="cuda", generator=g) * (10.0 ** (step % 3 - 2))
            a.grad, b.grad = gr.clone(), gr.clone()
        o1.step()
        o2.step()
        o1.zero_grad()
        o2.zero_grad()
        for a, b in zip(p1, p2):
            assert torch.allclose(a, b, rtol=1e-5, atol=1e-7)
            assert compute_copy(a, torch.bfloat16) is a._lors_shadow
            assert torch.equal(compute_copy(a, torch.bfloat16), a.detach().bfloat16())
    assert int(o1.counter[0]) == 6 and o1.steps == 6   # the device step count (lors_adamw_dstep)
    with torch.no_grad():                              # an outside in-place change: the cast path takes over
        p1[0].mul_(2.0)
    assert torch.equal(compute_copy(p1[0], torch.bfloat16), p1[0].detach().bfloat16())


@pytest.mark.gpu
def test_backward_writes_adapter_grads_into_the_flat_buffer():
    """With FlatAdamW, the LoRS backward (grouped and single projections) writes dA / dB straight into
    the optimizer's zeroed flat gradient buffer and autograd keeps those views as .grad (no per-layer
    fp32 gradient buffers, no concatenation); a second backward before the step accumulates on top."""
    from paper_2501_08582_b200 import decoder as D
    from paper_2501_08582_b200.trainer import FlatAdamW, synthetic_tokens
    cfg = D.preset("tiny")
    model = D.LoRSDecoder(cfg, device="cuda", seed=5)
    params = model.adapter_parameters()
    opt = FlatAdamW(params, lr=1e-3)
    toks = synthetic_tokens(cfg.vocab, cfg.batch, cfg.seq, 0, device="cuda")
    model.loss(toks).backward()
    g0 = opt.G.data_ptr()
    in_place = [p.grad.data_ptr() == g0 + 4 * off for p, off in zip(params, opt._offs)]
    assert all(in_place), sum(in_place)
    first = [p.grad.clone() for p in params]
    model.loss(toks).backward()                 # accumulation: same tokens, twice the gradient
    for p, f in zip(params, first):
        assert torch.allclose(p.grad, 2 * f, rtol=1e-3, atol=1e-7)
    opt.zero_grad()
    assert float(opt.G.abs().sum()) == 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 3, 4])
def test_sum_into_matches_fp32_sum(n):
    """ops.sum_into (lors_add3): the grouped projections' input gradient, summed in fp32 and
    rounded once -- bit-equal to torch's fp32 sum rounded to bf16 for two or three terms."""
    from paper_2501_08582_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(n)
    ts = [torch.randn(513, 136, device="cuda", generator=g).bfloat16() for _ in range(n)]
    ref = sum(t.float() for t in ts)
    out = ops.sum_into([t.clone() for t in ts])
    if n <= 3:
        assert torch.equal(out, ref.bfloat16())
    else:
        assert torch.allclose(out.float(), ref, rtol=1e-2, atol=1e-2)


@pytest.mark.gpu
def test_cuda_graph_trainer_matches_eager():
    """Trainer(cuda_graph=True): one eager warm-up step, then the whole step (forward, CE, backward
    through the LoRS kernels, AdamW with the device step count) captured once and replayed.  Same
    losses and adapters as the eager trainer from the same initialisation and tokens, step by step
    (tolerance: the eager and replayed runs may sum the split-K partials in a different order); a
    new token shape re-captures; the captured step records the native launches it replays."""
    from paper_2501_08582_b200 import decoder as D
    from paper_2501_08582_b200.trainer import Trainer, synthetic_tokens
    cfg = D.preset("tiny")
    runs = []
    for graph in (False, True):
        model = D.LoRSDecoder(cfg, device="cuda", seed=3)
        tr = Trainer(model, lr=1e-3, cuda_graph=graph)
        losses = []
        for s in range(5):
            seq = cfg.seq if s < 4 else cfg.seq // 2          # the last step changes the shape
            losses.append(float(tr.step(synthetic_tokens(cfg.vocab, cfg.batch, seq, s, device="cuda"))))
        runs.append((losses, [p.detach().clone() for p in model.adapter_parameters()], tr))
    (l0, p0, t0), (l1, p1, t1) = runs
    assert t1._graph is None and t1.steps == t0.steps == 5 and t1.opt.steps == 5 and int(t1.opt.counter[0]) == 5
    assert t1.graph_launches > 0
    for a, b in zip(l0, l1):
        assert abs(a - b) <= 1e-3 * abs(a), (l0, l1)
    for a, b in zip(p0, p1):
        assert torch.allclose(a, b, rtol=1e-3, atol=1e-6)


@pytest.mark.gpu
@pytest.mark.parametrize("D,rows", [(4096, 700), (256, 33), (5120, 64), (2056, 5), (8192, 3), (8, 2)])
def test_fused_add_rmsnorm_matches_torch(D, rows):
    """lors_add_rmsnorm / _bwd against the torch formula (h + o, F.rms_norm) in fp32: forward outputs
    and the gradient that reaches h and o (residual + norm paths)."""
    from paper_2501_08582_b200.decoder import AddRMSNormFunction
    g = torch.Generator(device="cuda").manual_seed(D + rows)
    h = torch.randn(rows, D, device="cuda", generator=g).bfloat16().requires_grad_(True)
    o = torch.randn(rows, D, device="cuda", generator=g).bfloat16().requires_grad_(True)
    gamma = (1 + 0.1 * torch.randn(D, device="cuda", generator=g)).bfloat16()
    dhn = torch.randn(rows, D, device="cuda", generator=g).bfloat16()
    dx = torch.randn(rows, D, device="cuda", generator=g).bfloat16()
    hn, x = AddRMSNormFunction.apply(h, o, gamma, 1e-5)
    torch.autograd.backward([hn, x], [dhn, dx])
    hf, of = h.detach().float(), o.detach().float()
    hnr = (hf + of).bfloat16().float().requires_grad_(True)
    xr = F.rms_norm(hnr, (D,), gamma.float(), 1e-5)
    (hnr * dhn.float()).sum().add((xr * dx.float()).sum()).backward()
    assert torch.equal(hn, (hf + of).bfloat16())
    assert float((x.float() - xr).norm() / xr.norm()) < 5e-3
    ref = hnr.grad
    for got in (h.grad, o.grad):
        assert float((got.float() - ref).norm() / ref.norm()) < 5e-3


@pytest.mark.gpu
@pytest.mark.parametrize("N,V", [(300, 1000), (64, 128256), (7, 32000)])
def test_fused_cross_entropy_matches_torch(N, V):
    """CrossEntropyFunction (one-pass logsumexp, in-place gradient) against F.cross_entropy on the fp32
    upcast of the same bf16 logits: loss and logits gradient, incl. a non-unit incoming gradient."""
    from paper_2501_08582_b200.decoder import CrossEntropyFunction
    g = torch.Generator(device="cuda").manual_seed(N + V)
    base = (3 * torch.randn(N, V, device="cuda", generator=g)).bfloat16()
    t = torch.randint(0, V, (N,), device="cuda", generator=g)
    lr = base.float().requires_grad_(True)
    ref = F.cross_entropy(lr, t)
    (2.5 * ref).backward()
    logits = base.clone().requires_grad_(True)
    x = logits * 1          # a non-leaf input, as the LM head output is
    loss = CrossEntropyFunction.apply(x, t)
    (2.5 * loss).backward()
    assert abs(float(loss) - float(ref)) < 1e-3 * max(1.0, abs(float(ref)))
    assert float((logits.grad.float() - lr.grad).norm() / lr.grad.norm()) < 1e-2
