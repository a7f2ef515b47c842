"""Same tile structure, forward vs dX, for ncu: K1 on a 11008 x 4096 projection (Mout 11008, K 4096)
and K3 on the 4096 x 11008 one (Mout 11008, K 4096), 4096 tokens, r = 16, twice each.
    ncu --set full -k regex:tc_lors_gemm -s 1 -c 3 python tools/prof_dx_fwd.py  (fwd #2, dX #1, dX #2)"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2501_08582_b200 import ops, prune  # noqa: E402
L, r = 4096, 16
g = torch.Generator(device="cuda").manual_seed(0)


def layer(R, C):
    w = prune.prune_rowwise(torch.randn(R, C, device="cuda", generator=g) * 0.02, 0.5).bfloat16()
    a = (torch.randn(R, r, device="cuda", generator=g) * 1e-3).bfloat16()
    b = (torch.randn(r, C, device="cuda", generator=g) / r ** 0.5).bfloat16()
    return w, a, b


w1, a1, b1 = layer(11008, 4096)
x1 = torch.randn(L, 4096, device="cuda", generator=g).bfloat16()
w2, a2, b2 = layer(4096, 11008)
x2 = torch.randn(L, 11008, device="cuda", generator=g).bfloat16()
dy2 = torch.randn(L, 4096, device="cuda", generator=g).bfloat16()
for _ in range(2):
    ops.lors_fwd(x1, w1, a1, b1, 2.0)
for _ in range(2):
    ops._lors_bwd_call(x2, w2, a2, b2, dy2, 2.0, None, None, "ste", True, False, False, dx_only=True)
torch.cuda.synchronize()
print("ok")
