"""Prologue breakdown of the LoRS GEMMs (build with -DLORS_EXP_CLOCK -DLORS_EXP_CLOCK_PRO): CTA start ->
cluster sync done -> first recompute issued -> first transform done (warp 0) -> first main MMA issued."""
import ctypes as ct, os, sys, statistics, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_08582_b200 import _native, ops, prune
lib = _native.load()
L, R, C, r = 8192, 11008, 4096, 64
g = torch.Generator(device="cuda").manual_seed(0)
w = prune.prune_two_four(torch.randn(R, C, device="cuda", generator=g) * 0.02).bfloat16()
a = (torch.randn(R, r, device="cuda", generator=g) * 1e-3).bfloat16()
b = (torch.randn(r, C, device="cuda", generator=g) / r ** 0.5).bfloat16()
x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
dy = torch.randn(L, R, device="cuda", generator=g).bfloat16()
buf = (ct.c_ulonglong * (4096 * 8))()
n = ct.c_uint()
med = statistics.median
def run(name, fn):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    lib.lors_exp_clock_read(buf, ct.byref(n))
    fn(); torch.cuda.synchronize()
    lib.lors_exp_clock_read(buf, ct.byref(n))
    k = min(n.value, 4096)
    rec = [buf[8 * i: 8 * i + 8] for i in range(k) if buf[8 * i + 4]]
    d = lambda i, j: med([(e[j] - e[i]) / 1e3 for e in rec])
    print(f"{name}: start->sync {d(2, 4):.2f} us, sync->rec0 {d(4, 5):.2f}, rec0->xform0 done {d(5, 6):.2f}, "
          f"xform0->main0 {d(6, 7):.2f}; CTA {d(2, 3):.1f} us", flush=True)
run("fwd dense", lambda: ops.lors_fwd(x, w, a, b, 2.0))
run("dX", lambda: ops.lors_bwd(x, w, a, b, dy, 2.0))
