"""Timing-only probe for a single grouped forward launch: one K1 over the concatenated [G R, C] weight
(one shared b: wrong adapter math, identical work and tile count) against the concurrent per-projection
launches of lors_group (cfg3 q/k/v and gate/up, 4096 tokens), sustained, CUDA events."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2501_08582_b200 import ops, prune  # noqa: E402
from paper_2501_08582_b200.module import LoRSLinear, lors_group  # noqa: E402

L, r = 4096, 16
g = torch.Generator(device="cuda").manual_seed(0)


def timed(fn, n=40):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


for rep in range(2):
    for name, G, R in (("qkv", 3, 4096), ("gate/up", 2, 11008)):
        C = 4096
        wc = prune.prune_rowwise(torch.randn(G * R, C, device="cuda", generator=g) * 0.02, 0.5).bfloat16()
        ac = (torch.randn(G * R, r, device="cuda", generator=g) * 1e-3).bfloat16()
        b = (torch.randn(r, C, device="cuda", generator=g) / r ** 0.5).bfloat16()
        ls = [LoRSLinear(wc[i * R:(i + 1) * R], a=ac[i * R:(i + 1) * R].float(), b=b.float(), alpha=2.0)
              for i in range(G)]
        x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
        with torch.no_grad():
            grouped = timed(lambda: lors_group(ls, x))
            one = timed(lambda: ops.lors_fwd(x, wc, ac, b, 2.0))
        print(f"{name}: concurrent per-projection {grouped:.1f} us, one launch over [{G}x{R}, {C}] {one:.1f} us",
              flush=True)
        del wc, ac, ls, x
