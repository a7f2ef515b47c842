"""BASELINE configs[0] (fp32 parity mode: 4096 x 4096, r = 16, 2048 tokens) forward and dX through the FFMA
kernels, for an ncu capture:  ncu --set full -k regex:simt_lors_gemm -c 2 python tools/prof_f32.py"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2501_08582_b200 import ops, prune  # noqa: E402
L, R, C, r = 2048, 4096, 4096, 16
g = torch.Generator(device="cuda").manual_seed(0)
w = prune.prune_rowwise(torch.randn(R, C, device="cuda", generator=g) * 0.02, 0.5)
a = torch.randn(R, r, device="cuda", generator=g) / r ** 0.5
b = torch.randn(r, C, device="cuda", generator=g) * 1e-3
x = torch.randn(L, C, device="cuda", generator=g)
dy = torch.randn(L, R, device="cuda", generator=g)
bits = ops.pack_mask(w)
for _ in range(2):
    ops.lors_fwd(x, w, a, b, 2.0, mask_bits=bits)
    ops.lors_bwd(x, w, a, b, dy, 2.0, mask_bits=bits, overlap=False)
torch.cuda.synchronize()
print("ok")
