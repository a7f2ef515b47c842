"""Summarise tools/ab_gemm.py logs: median `sus` (and `iso`) microseconds per (variant, shape, kernel).
    python tools/ab_table.py gpurun_out/ab6.log"""
import re
import statistics
import sys
from collections import defaultdict

vals = defaultdict(list)
pat = re.compile(r"(\w+) iso\s+([\d.]+) sus\s+([\d.]+) us")
for ln in open(sys.argv[1]):
    m = re.match(r"\[(\S+)\]\s+(.+?)\s{2,}(fwd .*)", ln.strip())
    if not m:
        continue
    var, shape, rest = m.groups()
    for k, iso, sus in pat.findall(rest):
        vals[(shape, k, var)].append((float(iso), float(sus)))
variants = sorted({v for _, _, v in vals}, key=lambda v: (v != "default", v))
keys = sorted({(s, k) for s, k, _ in vals})
print(f"{'shape':14s} {'kernel':7s} " + " ".join(f"{v:>16s}" for v in variants) + "   (sus us, median; iso in parentheses)")
for s, k in keys:
    cells = []
    for v in variants:
        xs = vals.get((s, k, v))
        cells.append(f"{statistics.median(x[1] for x in xs):7.1f} ({statistics.median(x[0] for x in xs):6.1f})" if xs else " " * 16)
    print(f"{s:14s} {k:7s} " + " ".join(cells))
