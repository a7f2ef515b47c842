"""2:4 sparse-tensor-core forward vs the dense-masked forward and a torch fp32 reference."""
import sys, torch
sys.path.insert(0, ".")
from paper_2501_08582_b200 import ops, prune

def rel(a, b):
    a = a.float(); b = b.float()
    return float((a - b).norm() / max(b.norm(), 1e-30))

torch.manual_seed(0)
shapes = [(256, 256, 64, 16), (512, 384, 256, 64), (300, 264, 192, 32), (1024, 1024, 512, 64)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in sys.argv[1:5])]
for (L, R, C, r) in shapes:
    dt = torch.bfloat16
    w = prune.prune_two_four(torch.randn(R, C, device="cuda") * 0.02).to(dt)
    # make some groups sparser than 2:4 (padding path)
    w[: R // 4, : C // 2] = torch.where(torch.rand(R // 4, C // 2, device="cuda") < 0.3,
                                         torch.zeros_like(w[: R // 4, : C // 2]), w[: R // 4, : C // 2])
    a = (torch.randn(R, r, device="cuda") * 0.05).to(dt)
    b = (torch.randn(r, C, device="cuda") / r ** 0.5).to(dt)
    x = torch.randn(L, C, device="cuda").to(dt)
    wf, af, bf, xf = (t.float() for t in (w, a, b, x))
    weff = torch.where(wf != 0, wf + 2.0 * (af @ bf), torch.zeros_like(wf))
    yd, _ = ops.lors_fwd(x, w, a, b, 2.0)
    ys, _ = ops.lors_fwd(x, w, a, b, 2.0, sparse24=True)
    bits = ops.pack_mask(w)
    yb, _ = ops.lors_fwd(x, w, a, b, 2.0, sparse24=True, mask_bits=bits)
    torch.cuda.synchronize()
    print(f"L={L} R={R} C={C} r={r}: sparse vs ref {rel(ys, xf @ weff.t()):.2e}  dense vs ref {rel(yd, xf @ weff.t()):.2e}"
          f"  sparse vs dense {rel(ys, yd):.2e}  bits==fromW {torch.equal(ys, yb)}", flush=True)
