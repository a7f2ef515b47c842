"""Per-call GPU time of ops.lors_bwd (two-stream overlap) over many calls: spikes?"""
import os, sys, time, statistics, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_08582_b200 import ops, prune
L, R, C, r = map(int, sys.argv[1:5]) if len(sys.argv) > 4 else (4096, 4096, 4096, 64)
ov = os.environ.get("LORS_BWD_OVERLAP", "1")
g = torch.Generator(device="cuda").manual_seed(0)
w = prune.prune_rowwise(torch.randn(R, C, device="cuda", generator=g) * 0.02, 0.5).bfloat16()
a = (torch.randn(R, r, device="cuda", generator=g) * 1e-3).bfloat16()
b = (torch.randn(r, C, device="cuda", generator=g) / r ** 0.5).bfloat16()
x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
dy = torch.randn(L, R, device="cuda", generator=g).bfloat16()
if os.environ.get("PREWARM"):
    big = torch.empty(int(os.environ["PREWARM"]) << 20, dtype=torch.uint8, device="cuda"); del big
for _ in range(3): ops.lors_bwd(x, w, a, b, dy, 2.0)
torch.cuda.synchronize()
N = 40
ev = [torch.cuda.Event(enable_timing=True) for _ in range(N + 1)]
ev[0].record()
for i in range(N):
    ops.lors_bwd(x, w, a, b, dy, 2.0)
    ev[i + 1].record()
torch.cuda.synchronize()
t = [ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(N)]
print(f"prewarm={os.environ.get('PREWARM')} overlap={ov} {L}x{R}x{C} r={r}: median {statistics.median(t):.0f} us, min {min(t):.0f}, max {max(t):.0f};",
      " ".join(f"{v:.0f}" for v in t[:20]))
