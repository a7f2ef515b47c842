"""cfg2 backward without dX (the rank-r products only), for ncu launch lists."""
import sys, torch
sys.path.insert(0, ".")
from paper_2501_08582_b200 import ops, prune
L, R, C, r = 8192, 11008, 4096, 64
if len(sys.argv) > 1:
    L, R, C, r = map(int, sys.argv[1:5])
dt = torch.bfloat16
g = torch.Generator(device="cuda").manual_seed(0)
w = prune.prune_two_four(torch.randn(R, C, device="cuda", generator=g) * 0.02).to(dt)
a = (torch.randn(R, r, device="cuda", generator=g) * 1e-3).to(dt)
b = (torch.randn(r, C, device="cuda", generator=g) / r ** 0.5).to(dt)
x = torch.randn(L, C, device="cuda", generator=g).to(dt)
dy = torch.randn(L, R, device="cuda", generator=g).to(dt)
for _ in range(3):
    ops.lors_bwd(x, w, a, b, dy, 2.0, need_dx=False)
torch.cuda.synchronize()
print("ok")
