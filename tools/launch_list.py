"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
iK, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
iU = h.index("Metric Unit") if "Metric Unit" in h else None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr + 1:]:
    if len(r) <= iV or r[iM] != "gpu__time_duration.sum":
        continue
    name = r[iK].split("(")[0].split("::")[-1]
    v = float(r[iV].replace(",", ""))
    unit = r[iU] if iU is not None else "ns"
    ns = v * {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
    agg[name][0] += 1
    agg[name][1] += ns
tot = sum(v[1] for v in agg.values())
n = sum(v[0] for v in agg.values())
print(f"{n} launches, {tot / 1e6:.3f} ms total")
for k, (c, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:28s} {c:6d} launches {ns / 1e3:10.1f} us {100 * ns / tot:5.1f}%  avg {ns / c / 1e3:7.2f} us")
