"""The fused gradient collective + AdamW (collective.py).

CPU (gloo, world size 2 and 3): the sharded algorithm the peer-memory kernel
runs -- ShardLayout's padding / shard bounds / parameter views, gradient
averaging, AdamW on each rank's shard with its optimizer-state shard, the
all-gather of the shards -- equals single-process AdamW on the averaged
gradients.  GPU (one B200, a one-rank NCCL group over symmetric memory): the
lors_adamw_p2p kernel equals torch AdamW and refreshes the bf16 compute copies."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
from torch import nn

SHAPES = [(37, 5), (5, 29), (37,), (3,)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_layout():
    from paper_2501_08582_b200.collective import ShardLayout
    params = [nn.Parameter(torch.zeros(s)) for s in SHAPES]
    for world in (1, 2, 3, 8):
        L = ShardLayout(params, world)
        assert L.n == 37 * 5 + 5 * 29 + 37 + 3
        assert L.n_pad % (4 * world) == 0 and L.n_pad >= L.n and L.n_pad - L.n < 4 * world
        assert L.bounds(world - 1)[1] == L.n_pad and L.bounds(0)[0] == 0
        flat = torch.arange(L.n_pad, dtype=torch.float32)
        views = L.views(flat)
        assert [tuple(v.shape) for v in views] == [tuple(p.shape) for p in params]
        assert views[1].reshape(-1)[0] == 37 * 5


def _grads(rank, step):
    g = torch.Generator().manual_seed(1000 * step + rank)
    return [torch.randn(s, generator=g) for s in SHAPES]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2501_08582_b200.collective import ShardedAdamWReference
        torch.manual_seed(0)
        params = [nn.Parameter(torch.randn(s)) for s in SHAPES]
        opt = ShardedAdamWReference(params, lr=1e-2, weight_decay=0.1)
        for step in range(4):
            for p, gr in zip(params, _grads(rank, step)):
                p.grad = gr
            opt.step()
            opt.zero_grad()
        q.put((rank, [p.detach().clone().tolist() for p in params]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_adamw_equals_adamw_on_averaged_grads(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    torch.manual_seed(0)
    ref = [nn.Parameter(torch.randn(s)) for s in SHAPES]
    opt = torch.optim.AdamW(ref, lr=1e-2, weight_decay=0.1)
    for step in range(4):
        per_rank = [_grads(r, step) for r in range(world)]
        for i, p in enumerate(ref):
            p.grad = sum(g[i] for g in per_rank) / world
        opt.step()
    for rank, vals in res:
        for v, p in zip(vals, ref):
            assert torch.allclose(torch.tensor(v), p.detach(), rtol=1e-5, atol=1e-6)


@pytest.mark.gpu
def test_symmetric_adamw_one_rank_matches_adamw():
    from paper_2501_08582_b200.collective import SymmetricAdamW
    from paper_2501_08582_b200.module import compute_copy
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        g = torch.Generator(device="cuda").manual_seed(4)
        shapes = [(64, 16), (16, 48), (300, 8), (7,)]
        p1 = [nn.Parameter(torch.randn(s, device="cuda", generator=g)) for s in shapes]
        p2 = [nn.Parameter(p.detach().clone()) for p in p1]
        o1 = SymmetricAdamW(p1, lr=3e-3, weight_decay=0.05)
        o2 = torch.optim.AdamW(p2, lr=3e-3, weight_decay=0.05)
        for step in range(5):
            for a, b in zip(p1, p2):
                gr = torch.randn(a.shape, device="cuda", generator=g)
                a.grad, b.grad = gr.clone(), gr.clone()
            o1.step()
            o2.step()
            o1.zero_grad()
            o2.zero_grad()
            for a, b in zip(p1, p2):
                assert torch.allclose(a, b, rtol=1e-5, atol=1e-7)
                assert torch.equal(compute_copy(a, torch.bfloat16), a.detach().bfloat16())
    finally:
        dist.destroy_process_group()
