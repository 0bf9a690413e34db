"""Markdown summary of `ncu -i REPORT --page raw --csv` output (one row per
kernel launch), for reports too large to bring back from the GPU box.

  python tools/ncu_csv_summary.py RAW.csv [--min-ms 0.02]
"""
import argparse
import csv

p = argparse.ArgumentParser()
p.add_argument("csv")
p.add_argument("--min-ms", type=float, default=0.02)
a = p.parse_args()
rows = list(csv.reader(open(a.csv)))
hdr, units = rows[0], dict(zip(rows[0], rows[1]))
SCALE = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
         "sector": 1e-6, "Ksector": 1e-3, "Msector": 1.0, "Gsector": 1e3}
COLS = [("time ms", "gpu__time_duration.sum"), ("DRAM rd GB", "dram__bytes_read.sum"),
        ("DRAM wr GB", "dram__bytes_write.sum"),
        ("DRAM % peak", "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("L2 % peak", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("L2 hit %", "lts__t_sector_hit_rate.pct"),
        ("L2 rd Msect", "lts__t_sectors_op_read.sum"), ("L2 red Msect", "lts__t_sectors_op_red.sum"),
        ("L2 wr Msect", "lts__t_sectors_op_write.sum"),
        ("tex miss Msect", "lts__t_sectors_srcunit_tex_lookup_miss.sum"),
        ("issue %", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        ("warps %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
        ("regs", "launch__registers_per_thread"), ("grid", "launch__grid_size")]


def val(d, k):
    v = d.get(k, "")
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    return x * SCALE.get(units.get(k, ""), 1.0)


print("| kernel | " + " | ".join(c for c, _ in COLS) + " |")
print("|---" * (len(COLS) + 1) + "|")
for r in rows[2:]:
    d = dict(zip(hdr, r))
    t = val(d, "gpu__time_duration.sum")
    if isinstance(t, float) and t < a.min_ms:
        continue
    name = d.get("Kernel Name", "?").replace("(anonymous namespace)::", "").replace("skx::", "")
    name = name.split("(")[0][:48]
    cells = []
    for _, k in COLS:
        v = val(d, k)
        cells.append(f"{v:.3g}" if isinstance(v, float) else str(v))
    print(f"| {name} | " + " | ".join(cells) + " |")
