import sys, numpy as np, torch
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
from paper_2501_08582_b200 import decoder as dec
from paper_2501_08582_b200.trainer import Trainer, synthetic_tokens
from ref_linear import oracle_factory
print("tf32 matmul", torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32)
for dtype in (torch.float32, torch.bfloat16):
  for lr in (1e-2, 1e-3):
    cfg = dec.preset("tiny", dtype=dtype, n_layers=2, seq=64)
    m = dec.LoRSDecoder(cfg, device="cuda"); ref = dec.LoRSDecoder(dec.replace(cfg, dtype=torch.float64), device="cpu", linear_factory=oracle_factory)
    ref.load_state_dict(m.state_dict())
    t1, t2 = Trainer(m, lr=lr), Trainer(ref, lr=lr)
    tok = synthetic_tokens(cfg.vocab, cfg.batch, cfg.seq, step=0, device="cpu")
    l1=[];l2=[]
    for s in range(30):
        l1.append(float(t1.step(tok.cuda()))); l2.append(float(t2.step(tok)))
    l1=np.array(l1); l2=np.array(l2); rel=np.abs(l1-l2)/l2
    print(dtype, lr, "loss", l2[0], l2[-1], "rel", np.array2string(rel[::3], precision=2))
