"""Run fwd + bwd once at cfg2 (for ncu captures)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2501_08582_b200 import ops, prune
L, R, C, r = 8192, 11008, 4096, 64
dt = torch.bfloat16
g = torch.Generator(device="cuda").manual_seed(0)
w = prune.prune_two_four(torch.randn(R, C, device="cuda", generator=g) * 0.02).to(dt)
a = (torch.randn(R, r, device="cuda", generator=g) * 1e-3).to(dt)
b = (torch.randn(r, C, device="cuda", generator=g) / r ** 0.5).to(dt)
x = torch.randn(L, C, device="cuda", generator=g).to(dt)
dy = torch.randn(L, R, device="cuda", generator=g).to(dt)
for _ in range(2):
    ops.lors_fwd(x, w, a, b, 2.0)
    ops.lors_bwd(x, w, a, b, dy, 2.0)
torch.cuda.synchronize()
print("ok")
