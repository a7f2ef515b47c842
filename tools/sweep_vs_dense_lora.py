"""LoRS fwd+bwd step (ops level, CUDA events) against the dense-LoRA step done with cuBLAS
(torch matmuls: X W^T + alpha (X b^T) a^T forward; dY W + alpha (dY a) b, dA, dB backward) over
shapes and ranks.  Prints one line per shape."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_08582_b200 import ops, prune

def t(fn, n=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3

def dense_lora(x, w, a, b, dy):
    p = x @ b.t()
    y = x @ w.t() + 2.0 * (p @ a.t())
    q = dy @ a
    dx = dy @ w + 2.0 * (q @ b)
    da = 2.0 * (dy.t() @ p).float()
    db = 2.0 * (q.t() @ x).float()
    return y, dx, da, db

g = torch.Generator(device="cuda").manual_seed(0)
print(f"{'L':>6} {'R':>6} {'C':>6} {'r':>3}  lors_us  denseLoRA_us  ratio")
for (L, R, C) in ((8192, 11008, 4096), (8192, 4096, 11008), (4096, 4096, 4096), (16384, 4096, 4096),
                  (8192, 14336, 4096), (4096, 5120, 5120)):
    w = prune.prune_rowwise(torch.randn(R, C, device="cuda", generator=g) * 0.02, 0.5).bfloat16()
    x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
    dy = torch.randn(L, R, device="cuda", generator=g).bfloat16()
    for r in (16, 64):
        a = (torch.randn(R, r, device="cuda", generator=g) * 1e-3).bfloat16()
        b = (torch.randn(r, C, device="cuda", generator=g) / r ** 0.5).bfloat16()
        tl = t(lambda: (ops.lors_fwd(x, w, a, b, 2.0), ops.lors_bwd(x, w, a, b, dy, 2.0)))
        td = t(lambda: dense_lora(x, w, a, b, dy))
        print(f"{L:6d} {R:6d} {C:6d} {r:3d}  {tl:7.0f}  {td:12.0f}  {td / tl:5.2f}", flush=True)
