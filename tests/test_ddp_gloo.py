"""World-size-2 gloo tests (CPU) of the data-parallel exchange of adapter
gradients: every rank must end with the average of the ranks' gradients,
bucketed or not, overlapped through grad hooks or not.  The kernels are not
involved (they need a B200); the gradients are set directly."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
from torch import nn


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, overlap, bucket_bytes, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2501_08582_b200.ddp import AdapterGradReducer, broadcast_adapters
        torch.manual_seed(rank)
        params = [nn.Parameter(torch.randn(37, 5)), nn.Parameter(torch.randn(5, 29)), nn.Parameter(torch.randn(37))]
        broadcast_adapters(params, src=0)
        red = AdapterGradReducer(params, bucket_bytes=bucket_bytes, overlap=overlap)
        # a fake "backward": rank-dependent grads; with overlap the hooks launch buckets
        loss = sum(((rank + 1) * (i + 1) * p).sum() for i, p in enumerate(params))
        loss.backward()
        red.finish()
        got = [p.grad.clone() for p in params]
        vals = [p.data.clone() for p in params]
        q.put((rank, [g.tolist() for g in got], [v.tolist() for v in vals]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("overlap,bucket_bytes", [(False, 1 << 20), (True, 64), (True, 1 << 20), (False, 64)])
def test_adapter_grad_average_world2(overlap, bucket_bytes):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, overlap, bucket_bytes, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    # expected average grad of param i: mean_r (r+1)(i+1) = 1.5 (i+1)
    for rank, grads, vals in res:
        for i, g in enumerate(grads):
            t = torch.tensor(g)
            assert torch.allclose(t, torch.full_like(t, 1.5 * (i + 1)))
    # broadcast made the adapters identical
    for a, b in zip(res[0][2], res[1][2]):
        assert torch.equal(torch.tensor(a), torch.tensor(b))


def _accum_worker(rank, world, port, overlap, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2501_08582_b200.ddp import AdapterGradReducer
        params = [nn.Parameter(torch.zeros(37, 5)), nn.Parameter(torch.zeros(5, 29)), nn.Parameter(torch.zeros(37))]
        red = AdapterGradReducer(params, bucket_bytes=64, overlap=overlap)
        for micro in range(2):   # gradient accumulation: two backward passes, one finish()
            loss = sum(((rank + 1) * (micro + 1) * (i + 1) * p).sum() for i, p in enumerate(params))
            loss.backward()
        red.finish()
        q.put((rank, [p.grad.clone().tolist() for p in params]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("overlap", [True, False])
def test_reducer_gradient_accumulation_world2(overlap):
    """Two backward passes before finish(): the buckets the first pass launched from its hooks are
    reduced again from the accumulated .grad, so every rank ends with the average over ranks of
    the summed micro-batch gradients (ddp.py, AdapterGradReducer._stale)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_accum_worker, args=(r, world, port, overlap, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # grad of param i = mean_r (r+1) * (1 + 2) * (i+1) = 1.5 * 3 * (i+1)
    for _, grads in res:
        for i, g in enumerate(grads):
            t = torch.tensor(g)
            assert torch.allclose(t, torch.full_like(t, 4.5 * (i + 1)))
