"""The 2:4 sparse forward (K2) at BASELINE configs[1] (11008 x 4096 2:4 weight, r = 64, 8192 tokens, with
the precomputed metadata), launched 4 times, for an ncu capture with source-level stall sampling:
    ncu --set full --import-source on -k regex:tc_lors_gemm -s 2 -c 1 python tools/prof_sp24.py"""
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
meta = ops.compress_24(w)[1]
for _ in range(4):
    ops.lors_fwd(x, w, a, b, 2.0, sparse24=True, meta24=meta)
torch.cuda.synchronize()
print("ok")
