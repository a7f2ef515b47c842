"""In-kernel timeline of the LoRS GEMMs (build with -DLORS_EXP_CLOCK): SM clock = dclock64 / dglobaltimer
per CTA, and per-CTA phases: start -> first main MMA issued (leader) -> accumulator complete -> staged ->
stored -> end."""
import ctypes as ct, os, sys, statistics, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_08582_b200 import _native, ops, prune
lib = _native.load()
L, R, C, r = 8192, 11008, 4096, 64
if len(sys.argv) > 1:
    L, R, C, r = map(int, sys.argv[1:5])
g = torch.Generator(device="cuda").manual_seed(0)
w = prune.prune_two_four(torch.randn(R, C, device="cuda", generator=g) * 0.02).bfloat16()
a = (torch.randn(R, r, device="cuda", generator=g) * 1e-3).bfloat16()
b = (torch.randn(r, C, device="cuda", generator=g) / r ** 0.5).bfloat16()
x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
dy = torch.randn(L, R, device="cuda", generator=g).bfloat16()
meta = ops.compress_24(w)[1]
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
    rec = [buf[8 * i: 8 * i + 8] for i in range(k)]
    mhz = [(e[1] - e[0]) / max(1, e[3] - e[2]) * 1e3 for e in rec]
    dur = [(e[3] - e[2]) / 1e3 for e in rec]
    t0 = min(e[2] for e in rec); t1 = max(e[3] for e in rec)
    lead = [e for e in rec if e[4]]
    pro = [(e[4] - e[2]) / 1e3 for e in lead]           # start -> first main MMA
    main = [(e[5] - e[4]) / 1e3 for e in lead]          # first main MMA -> accumulator complete
    stage = [(e[6] - e[5]) / 1e3 for e in rec]          # accumulator -> staged in smem
    store = [(e[7] - e[6]) / 1e3 for e in rec]          # TMA store issue -> read done
    tail = [(e[3] - e[7]) / 1e3 for e in rec]           # -> CTA end (cluster sync, dealloc)
    print(f"{name}: {k} CTAs, SM clock {med(mhz):.0f} MHz, CTA {med(dur):.1f} us = prologue {med(pro):.2f} + "
          f"mainloop {med(main):.2f} + stage {med(stage):.2f} + store {med(store):.2f} + tail {med(tail):.2f}; "
          f"kernel span {(t1 - t0) / 1e3:.0f} us", flush=True)
run("fwd dense", lambda: ops.lors_fwd(x, w, a, b, 2.0))
run("fwd 2:4", lambda: ops.lors_fwd(x, w, a, b, 2.0, sparse24=True, meta24=meta))
run("dX", lambda: ops.lors_bwd(x, w, a, b, dy, 2.0, grad_mode="ste"))
