#!/usr/bin/env python
"""Mean / median gpu__time_duration per kernel name of an ncu --csv launch list (µs)."""
import collections, csv, statistics, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, im, iv, iu = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
t = collections.defaultdict(list)
for r in rows[1:]:
    if r[im] == "gpu__time_duration.sum":
        v = float(r[iv].replace(",", ""))
        t[r[ik].split("(")[0]].append(v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[iu], 1e-3))
tag = sys.argv[2] if len(sys.argv) > 2 else ""
for k, v in t.items():
    print(f"{tag} {k[:60]} n={len(v)} mean={statistics.mean(v):.1f}us median={statistics.median(v):.1f}us")
