"""In-kernel SM clock of the LoRS GEMMs (build with -DLORS_EXP_CLOCK): MHz = dclock64 / dglobaltimer
per CTA, for the dense forward, the 2:4 forward and dX at cfg2."""
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
meta = ops.compress_24(w)[1]
buf = (ct.c_ulonglong * (4096 * 4))()
n = ct.c_uint()
def run(name, fn):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    lib.lors_exp_clock_read(buf, ct.byref(n))
    fn(); torch.cuda.synchronize()
    lib.lors_exp_clock_read(buf, ct.byref(n))
    k = min(n.value, 4096)
    mhz = [(buf[4*i+1]-buf[4*i]) / max(1, buf[4*i+3]-buf[4*i+2]) * 1e3 for i in range(k)]
    dur = [(buf[4*i+3]-buf[4*i+2]) / 1e3 for i in range(k)]
    t0 = min(buf[4*i+2] for i in range(k)); t1 = max(buf[4*i+3] for i in range(k))
    print(f"{name}: {k} CTAs, SM clock median {statistics.median(mhz):.0f} MHz (min {min(mhz):.0f}), "
          f"CTA duration median {statistics.median(dur):.1f} us, kernel span {(t1-t0)/1e3:.0f} us", flush=True)
run("fwd dense", lambda: ops.lors_fwd(x, w, a, b, 2.0))
run("fwd 2:4", lambda: ops.lors_fwd(x, w, a, b, 2.0, sparse24=True, meta24=meta))
run("dX", lambda: ops.lors_bwd(x, w, a, b, dy, 2.0, need_dx=True, grad_mode="ste") if False else ops.lors_fwd(dy[:, :4096].contiguous(), w[:4096].contiguous(), a[:4096].contiguous(), b, 2.0))
