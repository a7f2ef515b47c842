import sys, torch
sys.path.insert(0, ".")
from paper_2501_08582_b200 import ops, prune
L, R, C, r = 8192, 11008, 4096, 64
if len(sys.argv) > 1:
    L, R, C, r = map(int, sys.argv[1:5])
dt = torch.bfloat16
g = torch.Generator(device="cuda").manual_seed(0)
w = prune.prune_two_four(torch.randn(R, C, device="cuda", generator=g) * 0.02).to(dt)
a = (torch.randn(R, r, device="cuda", generator=g) * 1e-3).to(dt)
b = (torch.randn(r, C, device="cuda", generator=g) / r ** 0.5).to(dt)
x = torch.randn(L, C, device="cuda", generator=g).to(dt)
dy = torch.randn(L, R, device="cuda", generator=g).to(dt)
def t(fn, n=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
fw = t(lambda: ops.lors_fwd(x, w, a, b, 2.0))
bw = t(lambda: ops.lors_bwd(x, w, a, b, dy, 2.0))
bwx = t(lambda: ops.lors_bwd(x, w, a, b, dy, 2.0, need_dx=False))
mm = t(lambda: x @ w.t())
gflop_main = 2 * L * R * C / 1e9
print(f"fwd {fw:.0f} us ({gflop_main/fw*1e3:.0f} TF/s main), bwd {bw:.0f} us, bwd-noDX {bwx:.0f} us -> dX ~{bw-bwx:.0f} us; cuBLAS x@w^T {mm:.0f} us ({gflop_main/mm*1e3:.0f} TF/s)")
tot = fw + bw
flops = 2 * ((R*C*L + r*R*C + R*C) + (R*C*L + 2*r*R*L + 2*r*C*L + r*R*C + R*C))
print(f"step {tot:.0f} us, {L/tot*1e6/1e6:.2f} M tok/s, algorithmic {flops/tot/1e6:.0f} TF/s")
meta = ops.compress_24(w)[1]
fs = t(lambda: ops.lors_fwd(x, w, a, b, 2.0, sparse24=True, meta24=meta))
print(f"sparse-TC fwd {fs:.0f} us ({gflop_main/fs*1e3:.0f} TF/s dense-equivalent) vs dense-masked {fw:.0f} us")
bm = t(lambda: ops.lors_bwd(x, w, a, b, dy, 2.0, grad_mode="masked", need_dx=False), n=3)
print(f"masked-G fused grads (no dX) {bm:.0f} us ({2*R*C*L/bm/1e6:.0f} TF/s on the G GEMM)")
dxm, dam, dbm, _ = ops.lors_bwd(x, w, a, b, dy, 2.0, grad_mode="masked", need_dx=False)
wf, af, bf, xf, dyf = (tt.float() for tt in (w, a, b, x, dy))
G = (dyf.t() @ xf) * (wf != 0)
def rel(u, v): return float((u.float() - v).norm() / v.norm())
print(f"masked-G parity at cfg2: dA {rel(dam, 2 * G @ bf.t()):.2e}  dB {rel(dbm, 2 * af.t() @ G):.2e}")
