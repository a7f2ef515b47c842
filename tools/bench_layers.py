"""North_star target check: LoRS fwd+bwd step over the seven projections of one
LLaMA-shaped transformer block (q/k/v/o/gate/up/down, 50% per-row sparse, bf16),
as the decoder runs them (q/k/v and gate/up grouped), against the bf16 roofline
(north_star: the slower of the FLOPs at 2.25 PF dense bf16 and the bytes at 8 TB/s).

    python tools/bench_layers.py [preset] [steps]

FLOPs per projection from the reference cost model (COST_MODELS["lors"], adapters.py:674-681);
inputs and upstream gradients are seeded N(0, 1) resident in HBM (larger than L2); CUDA events.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_08582_b200 import LoRSLinear, lors_group  # noqa: E402
from paper_2501_08582_b200 import decoder as D  # noqa: E402
from paper_2501_08582_b200.adapters import predict_cost  # noqa: E402
from paper_2501_08582_b200.prune import prune_rowwise, prune_two_four  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "llama2-7b"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = D.preset(name)
L = cfg.batch * cfg.seq
g = torch.Generator(device="cuda").manual_seed(0)
shapes = cfg.shapes()           # name -> (R, C)
layers = {}
for nm, (R, C) in shapes.items():
    w = torch.randn(R, C, device="cuda", generator=g) * 0.02
    w = prune_two_four(w) if cfg.sparsity == "two_four" else prune_rowwise(w, cfg.ratio)
    a = torch.randn(R, cfg.rank, device="cuda", generator=g) * 1e-3
    b = torch.randn(cfg.rank, C, device="cuda", generator=g) / cfg.rank ** 0.5
    layers[nm] = LoRSLinear(w.bfloat16(), a=a, b=b, alpha=cfg.alpha)
x_attn = torch.randn(L, cfg.dim, device="cuda", generator=g).bfloat16().requires_grad_(True)
x_o = torch.randn(L, shapes["o"][1], device="cuda", generator=g).bfloat16().requires_grad_(True)
x_down = torch.randn(L, shapes["down"][1], device="cuda", generator=g).bfloat16().requires_grad_(True)
x_mlp = torch.randn(L, cfg.dim, device="cuda", generator=g).bfloat16().requires_grad_(True)
dys = {nm: torch.randn(L, R, device="cuda", generator=g).bfloat16() for nm, (R, C) in shapes.items()}


def step():
    for m in layers.values():
        m.a.grad = m.b.grad = None
    q, k, v = lors_group([layers["q"], layers["k"], layers["v"]], x_attn)
    o = layers["o"](x_o)
    gt, up = lors_group([layers["gate"], layers["up"]], x_mlp)
    dn = layers["down"](x_down)
    torch.autograd.backward([q, k, v, o, gt, up, dn],
                            [dys["q"], dys["k"], dys["v"], dys["o"], dys["gate"], dys["up"], dys["down"]])


for _ in range(3):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    step()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
flops = sum(predict_cost("lors", R, C, L, cfg.rank).flops for (R, C) in shapes.values())
# minimum bytes: W twice, X twice, Y out, dY in, dX out, a / b / dA / dB (fp32) -- SURVEY 8 d3
byt = sum(2 * 2 * R * C + 2 * 2 * L * C + 2 * L * R + 2 * L * R + 2 * L * C + 4 * 4 * cfg.rank * (R + C)
          for (R, C) in shapes.values())
roof_s = max(flops / 2.25e15, byt / 8e12)
out = {"preset": name, "tokens": L, "rank": cfg.rank, "sparsity": cfg.sparsity, "ms_per_step": ms,
       "tokens_per_s": L / (ms * 1e-3), "algorithmic_tflops": flops / (ms * 1e-3) / 1e12,
       "frac_of_spec_roofline": roof_s / (ms * 1e-3),
       "note": "7 projections of one block, fwd + bwd (dX, dA, dB), q/k/v and gate/up grouped as in the decoder"}
print(json.dumps(out))
