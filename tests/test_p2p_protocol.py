"""The peer-memory protocol of SymmetricAdamW (collective.py) across two real processes (CPU, gloo).

On the GPU, every rank's flat gradient / master / bf16-copy buffers live in symmetric memory and one
kernel per rank (lors_adamw_p2p, csrc/lors_decoder.cu) reads shard `rank` of every peer's gradient
buffer, applies AdamW with the rank's optimizer-state shard and stores the result into every peer's
master and compute-copy buffers, between two device barriers (hG.barrier(channel=0) before,
hP.barrier(channel=1) after).  The round's GPU box has one GPU, so here the symmetric buffers are
process-shared CPU tensors, the barriers are dist.barrier() at the same two points of step(), and
the kernel is restated element-wise in the kernel's own arithmetic order.  Ranks reach the first
barrier at different times (jitter), so a protocol that read peers' gradients before the barrier, or
read the new masters before the second one, would see stale data and fail the comparison with
single-process AdamW on the averaged gradients.
"""

import os
import socket
import time

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
from torch import nn

SHAPES = [(37, 5), (5, 29), (37,), (3,), (64, 16)]
STEPS = 4
HP = dict(lr=1e-2, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.1)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _grads(rank, step):
    g = torch.Generator().manual_seed(1000 * step + rank)
    return [torch.randn(s, generator=g) for s in SHAPES]


def _init_params():
    torch.manual_seed(0)
    return [nn.Parameter(torch.randn(s)) for s in SHAPES]


def adamw_p2p_restated(G, P, S, m, v, n_pad, rank, world, lr, b1, b2, eps, wd, step):
    """lors_adamw_p2p_kernel's arithmetic for one rank (csrc/lors_decoder.cu): shard `rank` of the
    flat buffers; peer loads of every rank's gradients, peer stores of the new masters / bf16 copies."""
    shard = n_pad // world
    lo, hi = rank * shard, (rank + 1) * shard
    decay = np.float32(1.0 - lr * wd)
    step_size = np.float32(lr / (1.0 - b1 ** step))
    inv_sqrt_bc2 = np.float32(1.0 / np.sqrt(1.0 - b2 ** step))
    g = torch.zeros(hi - lo)
    for p in range(world):                       # reduce over the ranks (NVLink loads)
        g += G[p][lo:hi]
    g = g * np.float32(1.0 / world)
    p0 = P[rank][lo:hi].clone()
    m.mul_(b1).add_((1.0 - b1) * g)              # fmaf(b1, m, (1 - b1) g)
    v.mul_(b2).add_((1.0 - b2) * g * g)
    pn = p0 * decay - step_size * m / (v.sqrt() * inv_sqrt_bc2 + eps)
    for p in range(world):                       # all-gather (NVLink stores)
        P[p][lo:hi] = pn
        S[p][lo:hi] = pn.to(torch.bfloat16)


def _worker(rank, world, port, G, P, S, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2501_08582_b200.collective import ShardLayout
        params = _init_params()
        L = ShardLayout(params, world)
        with torch.no_grad():                    # SymmetricAdamW.__init__: params become views of P[rank]
            for p, view in zip(params, L.views(P[rank])):
                view.copy_(p.detach())
                p.data = view
        lo, hi = L.bounds(rank)
        m, v = torch.zeros(hi - lo), torch.zeros(hi - lo)
        dist.barrier()                           # hP.barrier(channel=0) at construction
        b1, b2 = HP["betas"]
        for step in range(1, STEPS + 1):
            for p, g in zip(params, _grads(rank, step)):
                p.grad = g
            L.gather_grads(G[rank])              # step(): this rank's gradients into its symmetric buffer
            time.sleep(0.02 * ((rank + step) % world))
            dist.barrier()                       # hG.barrier(channel=0): every rank's gradients written
            adamw_p2p_restated(G, P, S, m, v, L.n_pad, rank, world, HP["lr"], b1, b2, HP["eps"],
                               HP["weight_decay"], step)
            dist.barrier()                       # hP.barrier(channel=1): new masters stored everywhere
            for p in params:
                p.grad = None
        q.put((rank, [p.detach().clone().numpy() for p in params], S[rank][:L.n].float().numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_p2p_protocol_matches_single_process_adamw(world):
    from paper_2501_08582_b200.collective import ShardLayout
    n_pad = ShardLayout([nn.Parameter(torch.zeros(s)) for s in SHAPES], world).n_pad
    G = [torch.zeros(n_pad).share_memory_() for _ in range(world)]
    P = [torch.zeros(n_pad).share_memory_() for _ in range(world)]
    S = [torch.zeros(n_pad, dtype=torch.bfloat16).share_memory_() for _ in range(world)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, G, P, S, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (ps, s)) for r, ps, s in (q.get(timeout=120) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single process: AdamW on the averaged gradients
    ref = _init_params()
    opt = torch.optim.AdamW(ref, **HP)
    for step in range(1, STEPS + 1):
        per_rank = [_grads(r, step) for r in range(world)]
        for i, p in enumerate(ref):
            p.grad = sum(g[i] for g in per_rank) / world
        opt.step()
    flat_ref = torch.cat([p.detach().reshape(-1) for p in ref])
    for r in range(world):
        ps, s = res[r]
        for got, want in zip(ps, ref):
            np.testing.assert_allclose(got, want.detach().numpy(), rtol=1e-5, atol=1e-6)
        # the bf16 compute copy every rank holds is its (peer-written) master rounded to bf16
        flat = torch.cat([torch.from_numpy(x).reshape(-1) for x in ps])
        np.testing.assert_array_equal(s, flat.to(torch.bfloat16).float().numpy())
        np.testing.assert_allclose(flat.numpy(), flat_ref.numpy(), rtol=1e-5, atol=1e-6)
    for r in range(1, world):
        for a, b in zip(res[0][0], res[r][0]):
            np.testing.assert_array_equal(a, b)
