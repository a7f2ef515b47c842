"""Timeline of the K1 pipeline (library built with -DLORS_TRACE, tools/build_variant.py trace):
globaltimer stamps per flat k-step of the first CTA pair, summarised as mean nanoseconds per k-step.
    LORS_B200_LIB=.../exp/trace/liblors_b200.so python tools/trace_k1.py [L R C r]"""
import ctypes as ct
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_08582_b200 import _native, ops, prune  # noqa: E402

L, R, C, r = (int(v) for v in sys.argv[1:5]) if len(sys.argv) > 4 else (4096, 11008, 4096, 16)
SP = len(sys.argv) > 5 and sys.argv[5] == "sp24"   # the 2:4 sparse-tensor-core forward (2:4 weight)
g = torch.Generator(device="cuda").manual_seed(0)
w = torch.randn(R, C, device="cuda", generator=g) * 0.02
w = (prune.prune_two_four(w) if SP else prune.prune_rowwise(w, 0.5)).bfloat16()
a = (torch.randn(R, r, device="cuda", generator=g) * 1e-3).bfloat16()
b = (torch.randn(r, C, device="cuda", generator=g) / r ** 0.5).bfloat16()
x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
meta = ops.compress_24(w)[1] if SP else None
for _ in range(3):
    ops.lors_fwd(x, w, a, b, 2.0, sparse24=SP, meta24=meta)
torch.cuda.synchronize()
buf = (ct.c_ulonglong * (2 * 24 * 512))()
lib = _native.load()
lib.lors_trace_read(buf)
t = np.frombuffer(buf, dtype=np.uint64).reshape(2, 24, 512).astype(np.int64)
names = {0: "iss: rec start", 1: "iss: sready ok", 2: "iss: refree ok", 3: "iss: main start", 4: "iss: afull ok",
         5: "iss: wready ok", 6: "iss: main issued", 7: "act: slot free", 8: "W: slot free", 9: "xf: start",
         10: "xf: refull ok", 11: "xf: W landed", 12: "xf: wempty ok", 13: "xf: arrived"}
lo, hi = 70, 300
print("(SM cycles, clock64)")
j = np.arange(lo, hi)
T = lambda cta, ev, idx: t[cta, ev, idx]  # noqa: E731
it = T(0, 0, j + 1) - T(0, 0, j)
print(f"issuer iteration (rec(j) + main(j-1)): mean {it.mean():.0f} median {np.median(it):.0f}")
d = T(0, 5, j - 1) - T(0, 0, j)
print(f"  fast path: 4 barriers (rec j, main j-1) mean {d.mean():.0f} median {np.median(d):.0f}")
d = T(0, 6, j - 1) - T(0, 5, j - 1)
print(f"  fast path: issue rec + main + commits   mean {d.mean():.0f} median {np.median(d):.0f}")
for cta in (0, 1):
    per = np.diff(t[cta, 13, lo:hi])
    d = t[cta, 9, lo + 1:hi] - t[cta, 13, lo:hi - 1]
    print(f"  xf arrive(j) -> start(j+1)     mean {d.mean():7.0f}  median {np.median(d):7.0f}")
    print(f"CTA {cta} transform period mean {per.mean():.0f}")
    for a_, b_, lbl in ((9, 10, "xf wait refull"), (10, 11, "xf tmem ld + W wait"), (11, 22, "xf W lds + tmem ld wait + release"),
                        (22, 12, "xf wait wempty"), (12, 23, "xf compute + stores"), (23, 13, "xf fences + arrive")):
        d = t[cta, b_, lo:hi] - t[cta, a_, lo:hi]
        print(f"  {lbl:28s} mean {d.mean():7.0f}  median {np.median(d):7.0f}")
d = T(0, 5, j) - T(0, 13, j)
print(f"issuer wready ok - CTA0 warp0 arrived: mean {d.mean():.0f}")
for ev, w in ((14, 3), (15, 5), (16, 7)):
    d = T(0, ev, j) - T(0, 13, j)
    print(f"  CTA0 warp {w} arrived - warp 0 arrived: mean {d.mean():.0f} median {np.median(d):.0f}")
last = np.max(np.stack([T(0, ev, j) for ev in (13, 14, 15, 16)]), axis=0)
for ev, lbl in ((1, "wready(jm)"), (2, "afull(jm)"), (4, "sready(jm+D)"), (5, "refree(jm+D)")):
    d = T(0, ev, j) - last
    print(f"  issuer passed {lbl:14s} - last CTA0 warp arrived: mean {d.mean():6.0f} median {np.median(d):6.0f}")
d = T(0, 5, j) - last
print(f"issuer wready ok - last of CTA0 warps 0/3/5/7 arrived: mean {d.mean():.0f} median {np.median(d):.0f}")
d = T(0, 10, j) - T(0, 2, j)
print(f"xf refull ok - rec issue (rec queue + exec + signal): mean {d.mean():.0f}")
# main(g) completion as seen by the activation producer (slot of step g + 3 freed by its commit)
done_ = T(0, 7, j + 3)
d = done_ - T(0, 6, j)
print(f"main issued -> main complete (seen by producer): mean {d.mean():.0f} median {np.median(d):.0f}")
d = np.diff(done_)
print(f"main completion period: mean {d.mean():.0f} median {np.median(d):.0f}")
d = T(0, 6, j) - done_[:0].sum() if False else T(0, 6, j + 1) - T(0, 7, j + 3)
print(f"main(j+1) issued - main(j) complete (negative: queued ahead): mean {d.mean():.0f} median {np.median(d):.0f}")
# tile boundaries (uniform tiles of nk k-steps): accumulator complete -> drained -> next tile's first main
nk = (C + 63) // 64
print(f"tile boundaries (nk = {nk} k-steps a tile), cycles:")
for n in range(1, 6):
    acc_done, acc_back = t[0, 18, n], t[0, 19, n]
    xf_end = t[0, 17, n]
    iss_wait0, iss_wait1 = t[0, 20, n + 1], t[0, 21, n + 1]
    first_main = t[0, 6, (n + 1) * nk] if (n + 1) * nk < 512 else 0
    last_main_issue = t[0, 6, (n + 1) * nk - 1] if (n + 1) * nk - 1 < 512 else 0
    print(f"  tile {n}: last main issued -> acc complete {acc_done - last_main_issue:6d}; xf loop end -> acc complete "
          f"{acc_done - xf_end:6d}; drain (acc complete -> handed back) {acc_back - acc_done:6d}; "
          f"handed back -> next first main issued {first_main - acc_back:6d}; issuer waited acc_empty {iss_wait1 - iss_wait0:6d}")
