"""How much of a cfg3 step is host launch overhead: eager Trainer.step vs the same step captured in one
CUDA graph and replayed (probe only -- the captured optimizer's bias correction is frozen at capture)."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_08582_b200 import decoder as D  # noqa: E402
from paper_2501_08582_b200.trainer import Trainer, synthetic_tokens  # noqa: E402

cfg = D.preset(sys.argv[1] if len(sys.argv) > 1 else "llama2-7b")
model = D.LoRSDecoder(cfg, device="cuda", seed=0)
tr = Trainer(model, lr=2e-5)
toks = [synthetic_tokens(cfg.vocab, cfg.batch, cfg.seq, s, device="cuda") for s in range(8)]
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def timed(fn, n=6):
    fn()
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


for s in range(3):
    tr.step(toks[s])
eager = timed(lambda: tr.step(toks[3]))
print(f"eager ms/step {eager:.2f}  mem {torch.cuda.max_memory_allocated() / 1e9:.1f} GB", flush=True)
static = toks[4].clone()
torch.cuda.synchronize()
torch.cuda.empty_cache()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    loss = tr.step(static)
graphed = timed(g.replay)
print(f"graph ms/step {graphed:.2f}  loss {float(loss):.4f}  mem {torch.cuda.max_memory_allocated() / 1e9:.1f} GB")
