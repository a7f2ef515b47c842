"""Experiment: kernel time of the fused Q/dA pass vs the R tiles per CTA (LORS_QDA_TR)."""
import os
import subprocess
import sys

if len(sys.argv) > 1:
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2501_08582_b200 import ops
    from torch.profiler import profile, ProfilerActivity
    L, R, C, r = (int(v) for v in sys.argv[1:5])
    g = torch.Generator(device="cuda").manual_seed(0)
    w = (torch.randn(R, C, device="cuda", generator=g) * 0.02).bfloat16()
    a = (torch.randn(R, r, device="cuda", generator=g) * 0.05).bfloat16()
    b = (torch.randn(r, C, device="cuda", generator=g) * 0.3).bfloat16()
    x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
    dy = torch.randn(L, R, device="cuda", generator=g).bfloat16()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        ops._lors_bwd_call(x, w, a, b, dy, 2.0, None, None, "ste", False, False, False)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(10):
            flush.zero_()
            ops._lors_bwd_call(x, w, a, b, dy, 2.0, None, None, "ste", False, False, False)
        torch.cuda.synchronize()
    tot = {}
    for e in prof.key_averages():
        if "q_da" in e.key or "skinny" in e.key:
            tot[e.key.split("(")[0][-40:]] = e.device_time_total / e.count
    print(os.environ.get("LORS_QDA_TR", "auto"), " ".join(f"{k}: {v:.1f}" for k, v in sorted(tot.items())), flush=True)
else:
    sweep = [("8192 11008 4096 64", (1, 2, 3, 4, 5, 6, 0)), ("4096 4096 4096 16", (2, 4, 8, 12, 16, 24, 0)),
             ("4096 11008 4096 16", (4, 8, 12, 16, 24, 0))]
    for shape, trs in sweep:
        print(shape, flush=True)
        for tr in trs:
            env = dict(os.environ)
            if tr:
                env["LORS_QDA_TR"] = str(tr)
            subprocess.run([sys.executable, __file__] + shape.split(), env=env)
