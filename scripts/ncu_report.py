"""Development aid: one-screen summary of an ncu --set full report (per kernel: duration,
throughputs, occupancy, DRAM bytes, stall reasons) for profiles/."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(det)))
h = rows[0]
ki, ii, mi, vi, ui = (h.index(c) for c in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
want = ("Duration", "Memory Throughput", "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Compute (SM) Throughput", "Issued Ipc Active", "Executed Instructions", "Registers Per Thread",
        "Achieved Occupancy", "Warp Cycles Per Issued Instruction")
for r in rows[1:]:
    if r[mi] in want:
        print(f"{r[ii]:>3} {r[ki].split('(')[0][:34]:34s} {r[mi]:36s} {r[vi]:>14s} {r[ui]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hh = rr[0]
cols = {c: hh.index(c) for c in hh}
stall = [c for c in hh if c.startswith("smsp__average_warp_latency_issue_stalled_") and c.endswith(".ratio")
         or c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("_per_issue_active.ratio")]
units = rr[1]
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
for r in rr[2:]:
    name = r[cols["Kernel Name"]].split("(")[0][:34]
    def f(c):
        try:
            return float(r[cols[c]].replace(",", "")) * scale.get(units[cols[c]], 1.0)
        except (KeyError, ValueError):
            return 0.0
    rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
    st = sorted(((c.split("stalled_")[1].replace("_per_issue_active.ratio", ""), f(c)) for c in stall),
                key=lambda kv: -kv[1])
    tot = sum(v for _, v in st) or 1.0
    print(f"{r[cols['ID']]:>3} {name:34s} dram read {rd/1e9:.3f} GB write {wr/1e9:.3f} GB; stalls: " +
          ", ".join(f"{k} {100*v/tot:.0f}%" for k, v in st[:6]))
