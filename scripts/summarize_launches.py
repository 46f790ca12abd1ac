"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv`)
into a per-kernel markdown table: launches, total us, share.
Usage: summarize_launches.py launches.csv "title / command line" > summary.md"""
import csv
import io
import re
import sys

path = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else path
text = open(path).read()
start = text.find('"ID"')
rows = list(csv.reader(io.StringIO(text[start:])))
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = {}
for r in rows[1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki]
    m = re.match(r"(?:void )?(?:[\w:<>() ]*::)?(k_\w+)(<[^>]*>)?", name.replace("(anonymous namespace)::", ""))
    key = (m.group(1) + (m.group(2) or "")) if m else name[:60]
    v = float(r[vi].replace(",", ""))
    unit = r[ui]
    us = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
    a = agg.setdefault(key, [0, 0.0])
    a[0] += 1
    a[1] += us
tot = sum(a[1] for a in agg.values())
print(f"# {title}\n")
print("| kernel | launches | total us | share |\n|---|---|---|---|")
for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| `{k}` | {n} | {us:.1f} | {us / tot:.3f} |")
print(f"\n{sum(a[0] for a in agg.values())} launches, {tot / 1e3:.1f} ms of kernel time")
