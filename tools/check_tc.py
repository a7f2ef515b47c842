"""Localise tcgen05 kernel bugs: each product vs a torch fp32 reference."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2501_08582_b200 import ops, prune

def rel(a, b):
    a = a.float(); b = b.float()
    return float((a - b).norm() / max(b.norm(), 1e-30))

torch.manual_seed(0)
for (L, R, C, r) in [(256, 128, 64, 16), (512, 384, 256, 64), (300, 264, 136, 32), (1024, 1024, 512, 64)]:
    dt = torch.bfloat16
    w = prune.prune_rowwise(torch.randn(R, C, device="cuda") * 0.02, 0.5).to(dt)
    a = (torch.randn(R, r, device="cuda") * 0.05).to(dt)
    b = (torch.randn(r, C, device="cuda") / r ** 0.5).to(dt)
    x = torch.randn(L, C, device="cuda").to(dt)
    dy = torch.randn(L, R, device="cuda").to(dt)
    wf, af, bf, xf, dyf = (t.float() for t in (w, a, b, x, dy))
    weff = torch.where(wf != 0, wf + 2.0 * (af @ bf), torch.zeros_like(wf))
    y, p = ops.lors_fwd(x, w, a, b, 2.0, emit_p=True)
    dx, da, db, _ = ops.lors_bwd(x, w, a, b, dy, 2.0)
    torch.cuda.synchronize()
    P = xf @ bf.t(); Q = dyf @ af
    print(f"L={L} R={R} C={C} r={r}: y {rel(y, xf @ weff.t()):.2e}  P {rel(p, P):.2e}  dx {rel(dx, dyf @ weff):.2e}  "
          f"dA {rel(da, 2 * dyf.t() @ P):.2e}  dB {rel(db, 2 * Q.t() @ xf):.2e}", flush=True)
    bits = ops.pack_mask(w)
    yb, _ = ops.lors_fwd(x, w, a, b, 2.0, mask_bits=bits)
    dxb, dab, dbb, _ = ops.lors_bwd(x, w, a, b, dy, 2.0, mask_bits=bits)
    torch.cuda.synchronize()
    print("   bits-mode identical:", torch.equal(y, yb), torch.equal(dx, dxb), torch.equal(da, dab), flush=True)
