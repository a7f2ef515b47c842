import torch, time, sys
n = 247 << 20
x = torch.empty(n, dtype=torch.uint8).pin_memory()
x.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(3): d.copy_(x, non_blocking=True)
torch.cuda.synchronize()
res = []
for rep in range(5):
    t = time.perf_counter()
    for _ in range(10): d.copy_(x, non_blocking=True)
    torch.cuda.synchronize()
    res.append(10 * n / (time.perf_counter() - t) / 1e9)
print("H2D GB/s", [round(v, 1) for v in res])
