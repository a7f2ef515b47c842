"""A/B of the grouped forward (lors_fwd_group: one persistent launch over G projections) against the
concurrent per-projection launches of lors_group, cfg3 q/k/v and gate/up at 4096 tokens, r = 16,
sustained (40 launches back to back), alternating the two four times."""
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


for name, G, R in (("qkv", 3, 4096), ("gate/up", 2, 11008)):
    C = 4096
    wc = prune.prune_rowwise(torch.randn(G * R, C, device="cuda", generator=g) * 0.02, 0.5).bfloat16()
    ac = (torch.randn(G * R, r, device="cuda", generator=g) * 1e-3).bfloat16()
    bc = (torch.randn(G * r, C, device="cuda", generator=g) / r ** 0.5).bfloat16()
    ls = [LoRSLinear(wc[i * R:(i + 1) * R], a=ac[i * R:(i + 1) * R].float(), b=bc[i * r:(i + 1) * r].float(),
                     alpha=2.0) for i in range(G)]
    x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
    res = {"concurrent": [], "grouped": []}
    with torch.no_grad():
        y = ops.lors_fwd_group(x, wc, ac, bc, G, 2.0)
        ref = lors_group(ls, x)
        same = all(torch.equal(y[i], ref[i]) for i in range(G))
        for rep in range(4):
            res["concurrent"].append(timed(lambda: lors_group(ls, x)))
            res["grouped"].append(timed(lambda: ops.lors_fwd_group(x, wc, ac, bc, G, 2.0)))
    print(f"{name}: bit-identical {same}; " + "; ".join(f"{k} " + " ".join(f"{v:.0f}" for v in vs) + " us"
                                                     for k, vs in res.items()), flush=True)
    del wc, ac, bc, ls, x
