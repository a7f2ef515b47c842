"""The bench line's dominant kernel for ncu: the LoRS forward GEMM (K1) of a cfg3 gate projection
(11008 x 4096, 50% per-row mask, r = 16) at the decoder step's 4096 tokens, launched 4 times.
    ncu --set full -k regex:tc_lors_gemm -s 2 -c 1 python tools/prof_dominant.py"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2501_08582_b200 import ops, prune  # noqa: E402
L, R, C, r = 4096, 11008, 4096, 16
g = torch.Generator(device="cuda").manual_seed(0)
w = prune.prune_rowwise(torch.randn(R, C, device="cuda", generator=g) * 0.02, 0.5).bfloat16()
a = (torch.randn(R, r, device="cuda", generator=g) * 1e-3).bfloat16()
b = (torch.randn(r, C, device="cuda", generator=g) / r ** 0.5).bfloat16()
x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
for _ in range(4):
    ops.lors_fwd(x, w, a, b, 2.0)
torch.cuda.synchronize()
print("ok")
