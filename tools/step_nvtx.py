"""One cfg3 (LLaMA-2-7B-shaped) fine-tuning step inside a process-wide NVTX start/end range "step" (the
backward runs on autograd's threads), after two warm-up steps:
    ncu --nvtx --nvtx-include "step" --metrics gpu__time_duration.sum --csv python tools/step_nvtx.py [preset] [graph]"""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_08582_b200 import decoder as D  # noqa: E402
from paper_2501_08582_b200.trainer import Trainer, synthetic_tokens  # noqa: E402

cfg = D.preset(sys.argv[1] if len(sys.argv) > 1 else "llama2-7b")
graph = len(sys.argv) > 2 and sys.argv[2] == "graph"     # the bench's path: the step replayed from a CUDA graph
model = D.LoRSDecoder(cfg, device="cuda", seed=0)
tr = Trainer(model, lr=2e-5, cuda_graph=graph)
toks = [synthetic_tokens(cfg.vocab, cfg.batch, cfg.seq, s, device="cuda") for s in range(3)]
for s in range(2):
    tr.step(toks[s])
torch.cuda.synchronize()
rid = torch.cuda.nvtx.range_start("step")
tr.step(toks[2])
torch.cuda.synchronize()
torch.cuda.nvtx.range_end(rid)
print("ok")
