"""Development aid: summarise an ncu report (key metrics + hottest SASS lines)."""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
want = ("Duration", "Executed Instructions", "Issued Ipc Active", "DRAM Throughput", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Achieved Occupancy", "Registers Per Thread", "Avg. Active Threads Per Warp",
        "Warp Cycles Per Issued Instruction", "Memory Throughput", "Eligible Warps Per Scheduler",
        "Compute (SM) Throughput", "L2 Cache Throughput", "Grid Size")
rows = list(csv.reader(io.StringIO(det)))
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
for r in rows[1:]:
    if r[mi] in want:
        print(f"{r[ki][:40]:40s} {r[mi]:40s} {r[vi]:>16s} {r[ui]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) > 2:
    hh = rr[0]
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
                "smsp__inst_executed.sum", "gpu__time_duration.sum"):
        if key in hh:
            i = hh.index(key)
            for r in rr[2:]:
                print(f"raw {key:45s} {r[i]:>20s} {rr[1][i]}")
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
h = rows[1]
ai, si, ie = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
ws, at = h.index("Warp Stall Sampling (All Samples)"), h.index("Avg. Threads Executed")
data = []
for r in rows[2:]:
    try:
        data.append((r[ai], r[si], int(r[ie].replace(",", "") or 0), int(r[ws].replace(",", "") or 0), r[at]))
    except (ValueError, IndexError):
        pass
tot = sum(d[2] for d in data) or 1
tots = sum(d[3] for d in data) or 1
print(f"SASS total executed {tot:.4e}  stall samples {tots}")
for d in sorted(data, key=lambda d: -d[3])[:top]:
    print(f"{d[0][-5:]:>6} exec {d[2]:>11} ({100*d[2]/tot:4.1f}%) stall {100*d[3]/tots:4.1f}% thr {d[4]:>5}  {d[1][:70]}")
