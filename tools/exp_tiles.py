"""Experiment: forward / dX GEMM time per projection shape (no split toggles), for
comparing library builds (LORS_B200_LIB=... variants from tools/exp_variants.sh)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_08582_b200 import ops  # noqa: E402
from tools.exp_split import SHAPES, timeit  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
for name, L, R, C, r in SHAPES:
    w = (torch.randn(R, C, device="cuda", generator=g) * 0.02).bfloat16()
    a = (torch.randn(R, r, device="cuda", generator=g) * 0.05).bfloat16()
    b = (torch.randn(r, C, device="cuda", generator=g) * 0.3).bfloat16()
    x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
    dy = torch.randn(L, R, device="cuda", generator=g).bfloat16()
    tf = min(timeit(lambda: ops.lors_fwd(x, w, a, b, 2.0)) for _ in range(3))
    td = min(timeit(lambda: ops._lors_bwd_call(x, w, a, b, dy, 2.0, None, None, "ste", True, False, False,
                                               dx_only=True)) for _ in range(3))
    print(f"{name:14s} fwd {tf:7.1f} us  dX {td:7.1f} us", flush=True)
