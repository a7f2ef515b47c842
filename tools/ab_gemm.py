"""Per-shape LoRS GEMM times of one library build (LORS_B200_LIB selects a variant):
forward (K1), dX (K3) and, for 2:4 shapes, the sparse forward (K2).  Two numbers each:
`iso` = median of single launches after an L2 flush (burst clocks), `sus` = mean over
back-to-back launches for ~0.3 s (power-capped clocks, as inside a training step).

    LORS_B200_LIB=... python tools/ab_gemm.py [shape-filter]
"""
import os
import statistics
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_08582_b200 import ops, prune  # noqa: E402

SHAPES = [  # (name, L, R, C, r, pattern)
    ("cfg2", 8192, 11008, 4096, 64, "two_four"),
    ("cfg3 qkvo", 4096, 4096, 4096, 16, "rowwise"),
    ("cfg3 gate/up", 4096, 11008, 4096, 16, "rowwise"),
    ("cfg3 down", 4096, 4096, 11008, 16, "rowwise"),
    ("cfg4 gate/up", 4096, 14336, 4096, 64, "two_four"),
]


def iso(fn, n=15):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        fn()
    ts = []
    for _ in range(n):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


CLK = []


def _clock_thread(stop, out):
    try:
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(0)
        while not stop.is_set():
            out.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
            time.sleep(0.005)
    except Exception:  # noqa: BLE001
        pass


def sus(fn, seconds=0.3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    n = max(5, int(seconds / (e0.elapsed_time(e1) * 1e-3)))
    clk, stop = [], threading.Event()
    th = threading.Thread(target=_clock_thread, args=(stop, clk))
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    th.start()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    CLK.append(statistics.median(clk) if clk else 0)
    return e0.elapsed_time(e1) * 1e3 / n


filt = sys.argv[1] if len(sys.argv) > 1 else ""
lib = os.environ.get("LORS_B200_LIB", "default").split("/exp/")[-1].split("/")[0]
g = torch.Generator(device="cuda").manual_seed(0)
for name, L, R, C, r, pat in SHAPES:
    if filt not in name:
        continue
    w = torch.randn(R, C, device="cuda", generator=g) * 0.02
    w = (prune.prune_two_four(w) if pat == "two_four" else prune.prune_rowwise(w, 0.5)).bfloat16()
    a = (torch.randn(R, r, device="cuda", generator=g) * 0.02).bfloat16()
    b = (torch.randn(r, C, device="cuda", generator=g) / r ** 0.5).bfloat16()
    x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
    dy = torch.randn(L, R, device="cuda", generator=g).bfloat16()
    fwd = lambda: ops.lors_fwd(x, w, a, b, 2.0)  # noqa: E731
    dx = lambda: ops._lors_bwd_call(x, w, a, b, dy, 2.0, None, None, "ste", True, False, False, dx_only=True)  # noqa
    res = {"fwd": (iso(fwd), sus(fwd)), "dx": (iso(dx), sus(dx))}
    if os.environ.get("AB_CUBLAS"):
        mm = lambda: x @ w.t()  # noqa: E731
        res["cublas"] = (iso(mm), sus(mm))
    if pat == "two_four":
        meta = ops.compress_24(w)[1]
        sp = lambda: ops.lors_fwd(x, w, a, b, 2.0, sparse24=True, meta24=meta)  # noqa: E731
        res["sp24"] = (iso(sp), sus(sp))
    fl = 2 * L * R * C
    if os.environ.get("AB_CLOCKS"):
        print(f"[{lib}] {name:13s} clocks (MHz, median while the sus loops ran): " +
              " ".join(f"{k} {c:.0f}" for k, c in zip(res, CLK[-len(res):])), flush=True)
    print(f"[{lib}] {name:13s} " + "  ".join(f"{k} iso {v[0]:7.1f} sus {v[1]:7.1f} us ({fl / v[1] / 1e6:5.0f} TF/s)"
                                            for k, v in res.items()), flush=True)
