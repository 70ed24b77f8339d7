"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel name:
count, total ms, share, mean us.  Usage: python tools/launch_summary.py launches.csv [out.json]"""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
agg = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    n = r[ki].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
    agg.setdefault(n, []).append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
tot = sum(sum(v) for v in agg.values())
out = {n: {"launches": len(v), "total_ms": sum(v), "share": sum(v) / tot, "mean_us": 1e3 * sum(v) / len(v)}
       for n, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))}
for n, d in out.items():
    print(f"{n:28s} {d['launches']:6d} {d['total_ms']:9.3f} ms {100 * d['share']:5.1f}% {d['mean_us']:9.2f} us")
print(f"total {tot:.3f} ms")
if len(sys.argv) > 2:
    json.dump({"total_ms": tot, "kernels": out}, open(sys.argv[2], "w"), indent=1)
