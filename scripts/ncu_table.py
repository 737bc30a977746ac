"""Development aid: one line per captured kernel of an ncu --set full report: duration, DRAM /
L1TEX / L2 throughput %, IPC, occupancy, DRAM bytes, and the top warp-stall reasons."""
import csv, io, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
col = {k: i for i, k in enumerate(h)}
SCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1.0, "ms": 1e3,
         "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}          # -> GB


def g(r, k):
    try:
        return float(r[col[k]].replace(",", "")) * SCALE.get(units[col[k]], 1.0)
    except (KeyError, ValueError):
        return float("nan")


stall_keys = [k for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")]
seen = set()
for r in rows[2:]:
    name = r[col["Kernel Name"]].split("(")[0].replace("void ", "")
    if name in seen:
        continue
    seen.add(name)
    st = sorted(((g(r, k), k[len("smsp__pcsamp_warps_issue_stalled_"):]) for k in stall_keys), reverse=True)
    tot = sum(v for v, _ in st if v == v) or 1.0
    top = ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in st[:4])
    print(f"{name[:44]:44s} {g(r, 'gpu__time_duration.sum'):8.1f} us  DRAM {g(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):5.1f}%  "
          f"L1TEX {g(r, 'l1tex__throughput.avg.pct_of_peak_sustained_active'):5.1f}%  L2 {g(r, 'lts__throughput.avg.pct_of_peak_sustained_elapsed'):5.1f}%  "
          f"IPC {g(r, 'sm__inst_executed.avg.per_cycle_active'):4.2f}  occ {g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):5.1f}%  "
          f"dram {g(r, 'dram__bytes_read.sum') + g(r, 'dram__bytes_write.sum'):6.3f} GB | {top}")
