"""Experiment: time of the rank-r backward products (P, Q, dA, dB, no dX) per
projection shape; run with and without LORS_NO_QDA_PASS=1 to compare the fused
Q/dA pass against the separate skinny GEMMs."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_08582_b200 import ops  # noqa: E402
from tools.exp_split import timeit  # noqa: E402

SHAPES = [("cfg2", 8192, 11008, 4096, 64), ("cfg3 qkvo", 4096, 4096, 4096, 16),
          ("cfg3 gate/up", 4096, 11008, 4096, 16), ("cfg3 down", 4096, 4096, 11008, 16),
          ("cfg5 gate/up", 4096, 13824, 5120, 64), ("cfg4 kv", 4096, 1024, 4096, 64)]

g = torch.Generator(device="cuda").manual_seed(0)
for name, L, R, C, r in SHAPES:
    w = (torch.randn(R, C, device="cuda", generator=g) * 0.02).bfloat16()
    a = (torch.randn(R, r, device="cuda", generator=g) * 0.05).bfloat16()
    b = (torch.randn(r, C, device="cuda", generator=g) * 0.3).bfloat16()
    x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
    dy = torch.randn(L, R, device="cuda", generator=g).bfloat16()
    t = timeit(lambda: ops._lors_bwd_call(x, w, a, b, dy, 2.0, None, None, "ste", False, False, False), n=30)
    gb = (2 * L * C * 2 + 2 * L * R * 2) / 1e9
    print(f"{name:14s} rank-r bwd {t:7.1f} us   (X twice + dY twice = {gb * 1e3:.0f} MB -> "
          f"{gb / (t * 1e-6):.0f} GB/s equiv)", flush=True)

if os.environ.get("PROFILE"):
    from torch.profiler import profile, ProfilerActivity
    for name, L, R, C, r in SHAPES[:2]:
        w = (torch.randn(R, C, device="cuda", generator=g) * 0.02).bfloat16()
        a = (torch.randn(R, r, device="cuda", generator=g) * 0.05).bfloat16()
        b = (torch.randn(r, C, device="cuda", generator=g) * 0.3).bfloat16()
        x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
        dy = torch.randn(L, R, device="cuda", generator=g).bfloat16()
        for _ in range(3):
            ops._lors_bwd_call(x, w, a, b, dy, 2.0, None, None, "ste", False, False, False)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(5):
                ops._lors_bwd_call(x, w, a, b, dy, 2.0, None, None, "ste", False, False, False)
            torch.cuda.synchronize()
        print(name)
        for e in prof.key_averages():
            if e.device_type == torch.autograd.DeviceType.CUDA or getattr(e, "device_time_total", 0) > 0:
                print(f"   {e.device_time_total / e.count:8.1f} us x{e.count // 5}  {e.key[:90]}")
