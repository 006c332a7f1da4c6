"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(r for r in rows if "Kernel Name" in r)
iname, ival, imet = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
agg = {}
for r in rows[rows.index(hdr) + 1:]:
    if len(r) <= ival or r[imet] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[iname]).replace("void ", "").replace("sem::", "")
    v = float(r[ival].replace(",", ""))
    u = r[hdr.index("Metric Unit")]
    unit = 1e-3 if u in ("ns", "nsecond") else (1e3 if u in ("ms", "msecond") else 1.0)
    n, t = agg.get(name, (0, 0.0))
    agg[name] = (n + 1, t + v * unit)
tot = sum(t for _, t in agg.values())
print("| kernel | launches | total us | share |\n|---|---|---|---|")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| {k} | {n} | {t:.0f} | {100 * t / tot:.1f}% |")
print(f"| **total** | {sum(n for n, _ in agg.values())} | {tot:.0f} | 100% |")
