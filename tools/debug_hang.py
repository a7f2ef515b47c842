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
tot = info[46] * 16
print("cluster 0: main issuer total cycles", tot, "k-steps", info[47], "cycles/step", tot / max(info[47], 1))
names = {40: "main: accempty", 41: "main: mready", 42: "recompute: ffready", 43: "recompute: rready",
         48: "xform warp0: W landed (rready)", 49: "xform warp0: wempty", 50: "xform warp0: refull"}
for k, n in names.items():
    print(f"  wait {n:32s} {info[k]*16:>10d} cycles ({info[k]*16/max(tot,1)*100:5.1f}%)")
