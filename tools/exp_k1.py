"""Time K1 (fwd), K3 (dX) and the 2:4 forward of whichever library LORS_B200_LIB points at (cfg2),
sampling SM clock and power with NVML while each op loops."""
import os, sys, threading, time, statistics, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml
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
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
def t(fn, n=int(os.environ.get('EXP_N', '20'))):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    samples, stop = [], threading.Event()
    def samp():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000))
            time.sleep(0.01)
    th = threading.Thread(target=samp); th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    stop.set(); th.join()
    s = samples[len(samples) // 4:] or samples
    return e0.elapsed_time(e1) / n * 1e3, statistics.median(c for c, _ in s), max(p for _, p in s)
def fmt(name, res):
    us, mhz, pw = res
    return f"{name} {us:.0f} us @{mhz:.0f} MHz {pw:.0f} W"
fw = t(lambda: ops.lors_fwd(x, w, a, b, 2.0))
dxo = t(lambda: ops.lors_bwd(x, w, a, b, dy, 2.0))
meta = ops.compress_24(w)[1]
fs = t(lambda: ops.lors_fwd(x, w, a, b, 2.0, sparse24=True, meta24=meta))
mm = t(lambda: x @ w.t())
name = os.path.basename(os.path.dirname(os.environ.get("LORS_B200_LIB", "default/x")))
print(f"[{name}] " + " | ".join([fmt("fwd", fw), fmt("bwd", dxo), fmt("fwd24", fs), fmt("cuBLAS", mm)]), flush=True)
