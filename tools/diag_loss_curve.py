"""Diagnostic: step-0 adapter gradients of the bf16 toy run vs a float64 simulation
with bf16 rounding at every layer boundary."""
import sys, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from test_loss_curve import _fixture
from oracle import lors_oracle as orc
import paper_2501_08582_b200 as P
d = _fixture(); D = 3; dev = "cuda"
def bf(a): return torch.from_numpy(np.asarray(a, dtype=np.float64)).to(torch.bfloat16).double().numpy()
idx = d["idx"][0]
# simulation
x = bf(d["x"][idx].T); t = d["t"][idx].T.astype(np.float64)
acts, pre = [x], []
for i in range(D):
    z = bf(orc.lors_forward(bf(d[f"base{i}"]), bf(d[f"a0_{i}"]), bf(d[f"b0_{i}"]), acts[-1]))
    pre.append(z)
    if i < D - 1: acts.append(np.maximum(z, 0))
dy = bf((pre[-1] - t) / 32)
sim = [None] * D
for i in range(D - 1, -1, -1):
    g = orc.lors_backward(bf(d[f"base{i}"]), bf(d[f"a0_{i}"]), bf(d[f"b0_{i}"]), acts[i], dy)
    sim[i] = g
    if i: dy = bf(bf(g.dx) * (pre[i - 1] > 0))
# GPU
layers = [P.LoRSLinear(torch.from_numpy(d[f"base{i}"]).to(dev, torch.bfloat16), a=torch.from_numpy(d[f"a0_{i}"]).float().to(dev),
                       b=torch.from_numpy(d[f"b0_{i}"]).float().to(dev)) for i in range(D)]
h = torch.from_numpy(d["x"][idx]).to(dev, torch.bfloat16)
for i, m in enumerate(layers):
    h = m(h)
    if i < D - 1: h = torch.relu(h)
loss = 0.5 * ((h.float() - torch.from_numpy(d["t"][idx]).to(dev)) ** 2).sum() / 32
loss.backward()
for i, m in enumerate(layers):
    ga = m.a.grad.double().cpu().numpy(); gb = m.b.grad.double().cpu().numpy()
    sa = sim[i].da; sb = sim[i].db
    print(f"layer {i}: da rel {orc.rel_l2(ga, sa):.2e} flips {int((np.sign(ga) != np.sign(sa)).sum())}/{sa.size} "
          f"|sa| min {np.abs(sa).min():.2e} med {np.median(np.abs(sa)):.2e}; db rel {orc.rel_l2(gb, sb):.2e} "
          f"flips {int((np.sign(gb) != np.sign(sb)).sum())} |sb| max {np.abs(sb).max():.2e} |gb| max {np.abs(gb).max():.2e}")
