"""Markdown summary of an ncu --set full report: one row per kernel launch.
usage: python tools/ncu_summary.py REPORT.ncu-rep [alg_bytes_json]"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
alg = json.load(open(sys.argv[2])) if len(sys.argv) > 2 else {}
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], dict(zip(rows[0], rows[1]))
SCALE = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
K = {"t": "gpu__time_duration.sum", "rd": "dram__bytes_read.sum", "wr": "dram__bytes_write.sum",
     "l2": "lts__t_sector_hit_rate.pct", "l1": "l1tex__t_sector_hit_rate.pct",
     "warps": "sm__warps_active.avg.pct_of_peak_sustained_active",
     "issue": "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "regs": "launch__registers_per_thread", "grid": "launch__grid_size",
     "block": "launch__block_size", "sec": "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
     "req": "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"}
print("| # | kernel | grid x block | regs | time ms | DRAM rd GB | DRAM wr GB | DRAM GB/s | L2 hit % "
      "| L1 hit % | ld sectors/req | warps active % | issue active % | top stall |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for i, r in enumerate(rows[2:]):
    d = dict(zip(hdr, r))

    def f(k, nd=2):
        v = d.get(K[k], "")
        try:
            return round(float(v.replace(",", "")) * SCALE.get(units.get(K[k], ""), 1.0), nd)
        except ValueError:
            return ""
    st = {k.split("stalled_")[1]: float(v.replace(",", "") or 0) for k, v in d.items()
          if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued") and v}
    tot = sum(st.values()) or 1
    top = max(st, key=st.get) if st else ""
    name = d["Kernel Name"].split("(")[0].replace("void ", "").split("::")[-1]
    t, rd, wr = f("t", 6), f("rd", 6), f("wr", 6)
    bw = round((rd + wr) / (t * 1e-3), 0) if t and rd != "" and wr != "" else ""
    sec, req = f("sec", 0), f("req", 0)
    spr = round(sec / req, 2) if sec and req else ""
    print(f"| {i} | {name} | {d.get(K['grid'])} x {d.get(K['block'])} | {d.get(K['regs'])} | "
          f"{f('t', 3)} | {f('rd')} | {f('wr')} | {bw} | {f('l2', 1)} | {f('l1', 1)} | {spr} | "
          f"{f('warps', 1)} | {f('issue', 1)} | {top} {round(100 * st.get(top, 0) / tot)}% |")
