"""Run the forward and dX GEMMs of one projection shape a few times (for ncu captures).

    python tools/prof_shape.py L R C r
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2501_08582_b200 import ops  # noqa: E402

L, R, C, r = (int(v) for v in sys.argv[1:5])
g = torch.Generator(device="cuda").manual_seed(0)
w = (torch.randn(R, C, device="cuda", generator=g) * 0.02)
w = torch.where(w.abs() < 0.0135, torch.zeros_like(w), w).bfloat16()   # ~50% per-row-ish sparsity
a = (torch.randn(R, r, device="cuda", generator=g) * 1e-3).bfloat16()
b = (torch.randn(r, C, device="cuda", generator=g) / r ** 0.5).bfloat16()
x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
dy = torch.randn(L, R, device="cuda", generator=g).bfloat16()
for _ in range(3):
    ops.lors_fwd(x, w, a, b, 2.0)
    ops._lors_bwd_call(x, w, a, b, dy, 2.0, None, None, "ste", True, False, False, dx_only=True)
torch.cuda.synchronize()
print("ok")
