"""Every native kernel once on small shapes, for compute-sanitizer (memcheck / synccheck / racecheck):
K1 / K2 / K3 (both alpha forms, from_w and packed bits, a ragged token count that exercises TMA
out-of-bounds fills and a tail split), K4 / K4b, K5, the deterministic reductions, K6 export,
pack_mask / compress_24 / grad_outer, and the fp32 FFMA kernels.
    compute-sanitizer --tool memcheck python tools/sanitize_small.py"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2501_08582_b200 import ops, prune  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
for (L, R, C, r) in ((300, 512, 256, 16), (200, 256, 8192, 64)):
    for dt in (torch.bfloat16, torch.float32):
        w = prune.prune_two_four(torch.randn(R, C, device="cuda", generator=g) * 0.02).to(dt)
        a = (torch.randn(R, r, device="cuda", generator=g) * 0.02).to(dt)
        b = (torch.randn(r, C, device="cuda", generator=g) / r ** 0.5).to(dt)
        x = torch.randn(L, C, device="cuda", generator=g).to(dt)
        dy = torch.randn(L, R, device="cuda", generator=g).to(dt)
        bits = ops.pack_mask(w)
        for alpha in (2.0, 1.0 / 3.0):
            ops.lors_fwd(x, w, a, b, alpha)
            ops.lors_fwd(x, w, a, b, alpha, mask_bits=bits)
            ops.lors_bwd(x, w, a, b, dy, alpha)
            ops.lors_bwd(x, w, a, b, dy, alpha, mask_bits=bits, deterministic=True)
            ops.lors_bwd(x, w, a, b, dy, alpha, grad_mode="masked")
            ops.lors_bwd(x, w, a, b, dy, alpha, grad_mode="masked", deterministic=True)
            ops.effective_weight(w, a, b, alpha)
            if dt == torch.bfloat16:
                meta = ops.compress_24(w)[1]
                ops.lors_fwd(x, w, a, b, alpha, sparse24=True)
                ops.lors_fwd(x, w, a, b, alpha, sparse24=True, meta24=meta)
        ops.grad_outer(dy, x, w, masked=True)
torch.cuda.synchronize()
print("sanitize run ok")
