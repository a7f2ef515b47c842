"""Per-kernel CUDA time of decoder fine-tuning steps (torch.profiler / CUPTI), top kernels.

    python tools/prof_decoder.py [preset] [steps]
"""
import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_08582_b200 import decoder as D
from paper_2501_08582_b200.trainer import Trainer, synthetic_tokens

name = sys.argv[1] if len(sys.argv) > 1 else "llama2-7b"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
sp = os.environ.get("SP24", "0") == "1"
cfg = D.preset(name)
model = D.LoRSDecoder(cfg, device="cuda", seed=0, linear_factory=D.lors_factory(cfg, seed=0, sparse24_forward=sp))
tr = Trainer(model, lr=2e-5)
toks = [synthetic_tokens(cfg.vocab, cfg.batch, cfg.seq, s, device="cuda") for s in range(steps + 2)]
for s in range(2):
    tr.step(toks[s])
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for s in range(steps):
        tr.step(toks[2 + s])
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0.0, 0])
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        k = e.name
        agg[k][0] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
        agg[k][1] += 1
tot = sum(v[0] for v in agg.values())
print(f"{name}: total kernel time per step {tot / steps / 1e3:.1f} ms over {steps} steps")
for k, (t, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:40]:
    print(f"{t / steps / 1e3:9.2f} ms/step {100 * t / tot:5.1f}%  n={n // steps:5d}  {k[:150]}")
