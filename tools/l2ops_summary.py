"""Summarise an ncu --metrics CSV of L2 sector operations per kernel
(lts__t_sectors_op_read/write/red/atom, lts__throughput, DRAM bytes):
python tools/l2ops_summary.py gpurun_out/l2ops.csv [min_us]."""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if r and not r[0].startswith("==")]
min_us = float(sys.argv[2]) if len(sys.argv) > 2 else 40.0
h = rows[0]
ix = {n: i for i, n in enumerate(h)}
k = OrderedDict()
for r in rows[1:]:
    key = (r[ix["ID"]], r[ix["Kernel Name"]])
    k.setdefault(key, {})[r[ix["Metric Name"]]] = r[ix["Metric Value"]]


def g(m, x):
    v = m.get(x, "nan").replace(",", "")
    try:
        return float(v)
    except ValueError:
        return float("nan")


print("| kernel | ms | L2 sectors M (read / write / red / atom) | L2 sector ops G/s | lts__throughput % |"
      " L2 hit % | DRAM rd / wr GB | DRAM % | issue % |")
print("|---|---|---|---|---|---|---|---|---|")
for (i, name), m in k.items():
    t = g(m, "gpu__time_duration.sum")
    if t < min_us * 1e3:
        continue
    sect = g(m, "lts__t_sectors.sum")
    nm = name.split("(")[0].replace("void ", "").replace("skx::<unnamed>::", "")[:44]
    print(f"| {nm} | {t / 1e6:.3f} | {sect / 1e6:.0f} ({g(m, 'lts__t_sectors_op_read.sum') / 1e6:.0f} / "
          f"{g(m, 'lts__t_sectors_op_write.sum') / 1e6:.0f} / {g(m, 'lts__t_sectors_op_red.sum') / 1e6:.0f} / "
          f"{g(m, 'lts__t_sectors_op_atom.sum') / 1e6:.0f}) | {sect / t:.0f} | "
          f"{g(m, 'lts__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
          f"{g(m, 'lts__t_sector_hit_rate.pct'):.1f} | {g(m, 'dram__bytes_read.sum') / 1e9:.2f} / "
          f"{g(m, 'dram__bytes_write.sum') / 1e9:.2f} | "
          f"{g(m, 'dram__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
          f"{g(m, 'smsp__issue_active.avg.pct_of_peak_sustained_elapsed'):.1f} |")
