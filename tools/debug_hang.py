"""Build a LORS_DEBUG_HANG variant of the library and report where pipelines stall."""
import ctypes as ct, os, sys, subprocess
sys.path.insert(0, ".")
from paper_2501_08582_b200 import build as B
import paper_2501_08582_b200._native as N
lib = B.build(force=True, extra_flags=["-DLORS_DEBUG_HANG"])
import torch
from paper_2501_08582_b200 import ops, prune
L, R, C, r = [int(v) for v in (sys.argv[1:5] or [256, 256, 128, 16])]
dx = len(sys.argv) > 5 and sys.argv[5] == "dx"
dt = torch.bfloat16
w = prune.prune_rowwise(torch.randn(R, C, device="cuda") * 0.02, 0.5).to(dt)
a = (torch.randn(R, r, device="cuda") * 0.05).to(dt)
b = (torch.randn(r, C, device="cuda") / r ** 0.5).to(dt)
x = torch.randn(L, C, device="cuda").to(dt)
dy = torch.randn(L, R, device="cuda").to(dt)
if dx:
    out = ops.lors_bwd(x, w, a, b, dy, 2.0)[0]
else:
    out = ops.lors_fwd(x, w, a, b, 2.0)[0]
torch.cuda.synchronize()
info = (ct.c_uint * 64)()
cdll = N.load()
cdll.lors_debug_hang_info(info)
n = info[0]
print("hang records:", n)
for i in range(min(n, 15)):
    blk, tid, addr, par = info[1 + 4 * i: 5 + 4 * i]
    print(f"  block=({blk & 0xffff},{blk >> 16}) thread={tid} warp={tid // 32} bar_smem=0x{addr:x} parity={par}")
wf = w.float(); weff = torch.where(wf != 0, wf + 2 * a.float() @ b.float(), torch.zeros_like(wf))
ref = dy.float() @ weff if dx else x.float() @ weff.t()
print("rel err", float((out.float() - ref).norm() / ref.norm()))
names = ["e_full", "p_early(relay)", "reempty", "a_full", "p_act(relay)", "wready"]
tot = info[46] * 256
print("MMA thread of cluster 0: total cycles", tot, "steps", info[47])
for i, n in enumerate(names):
    print(f"  wait {n:16s} {info[40+i]*256:>12d} cycles  ({info[40+i]*256/max(tot,1)*100:5.1f}%)")
