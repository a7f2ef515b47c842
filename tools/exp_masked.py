"""Experiment: backward time with the masked-G gradient (K5, grad_mode="masked") vs the STE rank-r
products, cfg2 and LLaMA-7B shapes; kernel-level breakdown with torch.profiler."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_08582_b200 import ops  # noqa: E402
from tools.exp_split import timeit  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
for name, L, R, C, r in (("cfg2", 8192, 11008, 4096, 64), ("7b qkvo", 4096, 4096, 4096, 16),
                         ("7b gate/up", 4096, 11008, 4096, 16)):
    w = (torch.randn(R, C, device="cuda", generator=g) * 0.02)
    w = torch.where(w.abs() < 0.0135, torch.zeros_like(w), w).bfloat16()
    a = (torch.randn(R, r, device="cuda", generator=g) * 0.05).bfloat16()
    b = (torch.randn(r, C, device="cuda", generator=g) * 0.3).bfloat16()
    x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
    dy = torch.randn(L, R, device="cuda", generator=g).bfloat16()
    res = []
    for mode in ("ste", "masked"):
        t = timeit(lambda: ops._lors_bwd_call(x, w, a, b, dy, 2.0, None, None, mode, False, False, False), n=10)
        res.append(t)
    fl = 2.0 * L * R * C
    print(f"{name:12s} adapter grads: ste {res[0]:7.1f} us, masked-G {res[1]:7.1f} us "
          f"({fl / res[1] / 1e6:.0f} TF/s on the G GEMM)", flush=True)
