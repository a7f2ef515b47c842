"""Find the source of occasional multi-ms stalls in the e2e (module + host copies) loop."""
import os, sys, statistics, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_08582_b200 import prune
from paper_2501_08582_b200.module import LoRSLinear
L, R, C, r = 8192, 11008, 4096, 64
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
w = prune.prune_two_four(torch.randn(R, C, device=dev, generator=g) * 0.02).bfloat16()
layer = LoRSLinear(w, a=torch.randn(R, r, device=dev, generator=g) * 1e-3, b=torch.randn(r, C, device=dev, generator=g) / 8)
x = torch.randn(L, C, device=dev, generator=g).bfloat16()
dy = torch.randn(L, R, device=dev, generator=g).bfloat16()
hx = x.cpu().pin_memory(); hdy = dy.cpu().pin_memory()
hda = torch.empty(R, r).pin_memory(); hdb = torch.empty(r, C).pin_memory()
main = torch.cuda.current_stream()
mode = sys.argv[1]
use_copy_stream = "copystream" in mode
overlap = "overlap" in mode
os.environ["LORS_BWD_OVERLAP"] = "1" if overlap else "0"
d2h = "nod2h" not in mode
cs = torch.cuda.Stream()
slots = [(torch.empty_like(x), torch.empty_like(dy)) for _ in range(2)]
filled = [torch.cuda.Event() for _ in range(2)]; consumed = [torch.cuda.Event() for _ in range(2)]
for e in consumed: e.record(main)
def prefetch(k):
    xs, dys = slots[k % 2]
    s = cs if use_copy_stream else main
    with torch.cuda.stream(s):
        s.wait_event(consumed[k % 2]); xs.copy_(hx, non_blocking=True); dys.copy_(hdy, non_blocking=True)
        filled[k % 2].record(s)
def step(k):
    xs, dys = slots[k % 2]
    main.wait_event(filled[k % 2]); prefetch(k + 1)
    xd = xs.detach().requires_grad_(True); layer.a.grad = None; layer.b.grad = None
    layer(xd).backward(dys); consumed[k % 2].record(main)
    if d2h:
        hda.copy_(layer.a.grad, non_blocking=True); hdb.copy_(layer.b.grad, non_blocking=True)
prefetch(0)
N = 60
marks = [torch.cuda.Event(enable_timing=True) for _ in range(N + 1)]
for k in range(5): step(k)
marks[0].record(main)
for k in range(N):
    step(5 + k); marks[k + 1].record(main)
torch.cuda.synchronize()
t = [marks[i].elapsed_time(marks[i + 1]) for i in range(N)]
print(f"{mode}: median {statistics.median(t):.2f} ms, max {max(t):.2f} ms, >10ms: {sum(v > 10 for v in t)}")
