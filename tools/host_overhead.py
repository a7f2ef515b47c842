"""Host-side enqueue cost of the ops wrappers (no synchronisation inside the loop)."""
import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_08582_b200 import ops, prune
L, R, C, r = 8192, 11008, 4096, 64
g = torch.Generator(device="cuda").manual_seed(0)
w = prune.prune_two_four(torch.randn(R, C, device="cuda", generator=g) * 0.02).bfloat16()
a = (torch.randn(R, r, device="cuda", generator=g) * 1e-3).bfloat16()
b = (torch.randn(r, C, device="cuda", generator=g) / r ** 0.5).bfloat16()
x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
dy = torch.randn(L, R, device="cuda", generator=g).bfloat16()
for name, fn in (("fwd", lambda: ops.lors_fwd(x, w, a, b, 2.0)),
                 ("bwd", lambda: ops.lors_bwd(x, w, a, b, dy, 2.0)),
                 ("bwd no-dx", lambda: ops.lors_bwd(x, w, a, b, dy, 2.0, need_dx=False))):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    n = 20
    t0 = time.perf_counter()
    for _ in range(n): fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name}: host {1e6 * (t1 - t0) / n:.0f} us/call, wall {1e6 * (t2 - t0) / n:.0f} us/call", flush=True)
