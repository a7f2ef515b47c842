"""Run the masked-G backward (K5) at cfg2 a few times (for ncu captures)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2501_08582_b200 import ops, prune  # noqa: E402

L, R, C, r = 8192, 11008, 4096, 64
g = torch.Generator(device="cuda").manual_seed(0)
w = prune.prune_two_four(torch.randn(R, C, device="cuda", generator=g) * 0.02).bfloat16()
a = (torch.randn(R, r, device="cuda", generator=g) * 1e-3).bfloat16()
b = (torch.randn(r, C, device="cuda", generator=g) / r ** 0.5).bfloat16()
x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
dy = torch.randn(L, R, device="cuda", generator=g).bfloat16()
for _ in range(3):
    ops._lors_bwd_call(x, w, a, b, dy, 2.0, None, None, "masked", False, False, False)
torch.cuda.synchronize()
print("ok")
