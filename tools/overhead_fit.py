"""Fit K1/K3 time = a + b * C at fixed R, L to expose the per-tile fixed cost."""
import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2501_08582_b200 import ops
torch.manual_seed(0)
R, L, r = 11008, 8192, 64
def t(fn, n=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n * 1e3
for C in (256, 512, 1024, 2048, 4096):
    w = (torch.randn(R, C, device="cuda") * 0.02).bfloat16()
    w[:, ::2] = 0
    a = (torch.randn(R, r, device="cuda") * 1e-3).bfloat16(); b = (torch.randn(r, C, device="cuda") / 8).bfloat16()
    x = torch.randn(L, C, device="cuda").bfloat16(); dy = torch.randn(L, R, device="cuda").bfloat16()
    tf = t(lambda: ops.lors_fwd(x, w, a, b))
    mm = t(lambda: x @ w.t())
    print(f"C={C}: fwd {tf:.1f} us  cuBLAS {mm:.1f} us  per-k-step(fwd) {tf / (C // 64):.2f} us")
