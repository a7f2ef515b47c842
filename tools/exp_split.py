"""Experiment: per-GEMM time of the persistent LoRS kernels with and without the
tail split (LORS_NO_TAIL_SPLIT), on the decoder's projection shapes."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_08582_b200 import ops  # noqa: E402

SHAPES = [  # (name, L, R, C, r)
    ("cfg3 qkvo", 4096, 4096, 4096, 16),
    ("cfg3 gate/up", 4096, 11008, 4096, 16),
    ("cfg3 down", 4096, 4096, 11008, 16),
    ("cfg4 q/o", 4096, 4096, 4096, 64),
    ("cfg4 kv", 4096, 1024, 4096, 64),
    ("cfg4 gate/up", 4096, 14336, 4096, 64),
    ("cfg4 down", 4096, 4096, 14336, 64),
    ("cfg5 qkvo", 4096, 5120, 5120, 64),
    ("cfg5 gate/up", 4096, 13824, 5120, 64),
    ("cfg5 down", 4096, 5120, 13824, 64),
    ("cfg2", 8192, 11008, 4096, 64),
]


REPS = int(os.environ.get("REPS", "5"))


def timeit(fn, n=20):
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
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2] * 1e3


def main():
    g = torch.Generator(device="cuda").manual_seed(0)
    for name, L, R, C, r in SHAPES:
        w = (torch.randn(R, C, device="cuda", generator=g) * 0.02).bfloat16()
        a = (torch.randn(R, r, device="cuda", generator=g) * 0.05).bfloat16()
        b = (torch.randn(r, C, device="cuda", generator=g) * 0.3).bfloat16()
        x = torch.randn(L, C, device="cuda", generator=g).bfloat16()
        dy = torch.randn(L, R, device="cuda", generator=g).bfloat16()
        res = {None: [[], []], "1": [[], []]}
        for rep in range(REPS):           # interleaved, so clock / power drift hits both arms
            for env in (None, "1"):
                if env:
                    os.environ["LORS_NO_TAIL_SPLIT"] = env
                else:
                    os.environ.pop("LORS_NO_TAIL_SPLIT", None)
                res[env][0].append(timeit(lambda: ops.lors_fwd(x, w, a, b, 2.0)))
                res[env][1].append(timeit(lambda: ops._lors_bwd_call(x, w, a, b, dy, 2.0, None, None, "ste", True,
                                                                     False, False, dx_only=True)))
        med = lambda v: sorted(v)[len(v) // 2]  # noqa: E731
        row = [name, med(res[None][0]), med(res[None][1]), med(res["1"][0]), med(res["1"][1])]
        fl = 2.0 * L * R * C
        print(f"{row[0]:14s} fwd split {row[1]:7.1f} us  nosplit {row[3]:7.1f} us ({row[3] / row[1]:.3f}x) | "
              f"dX split {row[2]:7.1f} us  nosplit {row[4]:7.1f} us ({row[4] / row[2]:.3f}x) | "
              f"fwd {fl / row[1] / 1e6:.0f} TF/s", flush=True)


if __name__ == "__main__":
    main()
