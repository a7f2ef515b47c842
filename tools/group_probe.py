"""Grouped projections (q/k/v, gate/up of cfg3) vs the same GEMMs one after another: does the concurrent
launch overlap the partial last rounds of the persistent kernels?  Forward and dX, CUDA events, sustained."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2501_08582_b200 import ops, prune  # noqa: E402
from paper_2501_08582_b200.module import LoRSLinear, lors_group  # noqa: E402

L = 4096
g = torch.Generator(device="cuda").manual_seed(0)


def layer(R, C, r=16):
    w = prune.prune_rowwise(torch.randn(R, C, device="cuda", generator=g) * 0.02, 0.5).bfloat16()
    a = torch.randn(R, r, device="cuda", generator=g) * 1e-3
    b = torch.randn(r, C, device="cuda", generator=g) / r ** 0.5
    return LoRSLinear(w, a=a, b=b, alpha=2.0)


def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


for name, shapes in (("qkv", [(4096, 4096)] * 3), ("gate/up", [(11008, 4096)] * 2)):
    ls = [layer(R, C) for R, C in shapes]
    x = torch.randn(L, 4096, device="cuda", generator=g).bfloat16()
    with torch.no_grad():
        grouped = timed(lambda: lors_group(ls, x))
        single = timed(lambda: [m(x) for m in ls])
        one = timed(lambda: ls[0](x))
    print(f"{name}: grouped fwd {grouped:.1f} us, sequential {single:.1f} us, one projection {one:.1f} us "
          f"(x{len(ls)} = {one * len(ls):.1f})", flush=True)
