"""Summary of an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel, the
number of launches and total / mean time, sorted by total.

  python tools/launch_summary.py LAUNCHES.csv [top]
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}
tot = collections.OrderedDict()
for r in rows[1:]:
    name = r[ki].replace("(anonymous namespace)::", "").replace("skx::<unnamed>::", "")
    name = name.split("(")[0][:70]
    ms = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    n, t = tot.get(name, (0, 0.0))
    tot[name] = (n + 1, t + ms)
allt = sum(t for _, t in tot.values())
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print(f"{len(rows) - 1} launches, {allt:.2f} ms of kernel time\n")
print("| kernel | launches | total ms | mean ms | share |")
print("|---|---|---|---|---|")
for name, (n, t) in sorted(tot.items(), key=lambda x: -x[1][1])[:top]:
    print(f"| {name} | {n} | {t:.3f} | {t / n:.4f} | {100 * t / allt:.1f}% |")
