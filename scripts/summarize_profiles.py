"""Turn gpurun_out ncu artefacts into the tracked summaries under profiles/ (per round)."""
import csv, io, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]                        # e.g. r01
launches = sys.argv[2]                   # ncu --metrics gpu__time_duration.sum csv
full = sys.argv[3] if len(sys.argv) > 3 else None   # ncu --set full report of the top kernels
workload = sys.argv[4] if len(sys.argv) > 4 else "rmat-s21-ef16"

rows = list(csv.reader(open(launches)))
for i, r in enumerate(rows):
    if r and r[0] == "ID":
        hdr, start = r, i + 1
        break
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
per = []
for r in rows[start:]:
    v = float(r[vi].replace(",", ""))
    v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
          "second": 1e3, "s": 1e3}[r[ui]]
    per.append((r[ki].split("(")[0].replace("void ", ""), v))
agg = {}
for k, v in per:
    a = agg.setdefault(k, [0.0, 0])
    a[0] += v
    a[1] += 1
tot = sum(v for _, v in per)
out = [f"# {tag}: ncu launch list ({launches}), gpu__time_duration.sum, --clock-control none",
       "# cold-cache serialised launches: compare SHARES of the step, not absolutes",
       f"# {len(per)} launches, total {tot:.3f} ms", "",
       f"{'ms total':>10} {'share':>6} {'launches':>8} {'ms/launch':>10}  kernel"]
for k, (v, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    out.append(f"{v:10.3f} {100*v/tot:5.1f}% {c:8d} {v/c:10.4f}  {k}")
open(os.path.join(ROOT, "profiles", f"{tag}_launches.txt"), "w").write("\n".join(out) + "\n")
print("\n".join(out[:20]))

if full:
    det = subprocess.run(["ncu", "-i", full, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", full, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    keep = ("Duration", "DRAM Throughput", "L2 Hit Rate", "L1/TEX Hit Rate", "Executed Instructions",
            "Issued Ipc Active", "Achieved Occupancy", "Registers Per Thread", "Memory Throughput",
            "Compute (SM) Throughput", "L2 Cache Throughput", "Avg. Active Threads Per Warp",
            "Warp Cycles Per Issued Instruction", "Grid Size", "Block Size", "Static Shared Memory Per Block")
    lines = [f"# {tag}: ncu --set full summary of {os.path.basename(full)}"]
    drows = list(csv.reader(io.StringIO(det)))
    h = drows[0]
    K, M, V, U = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    top = {}   # the dominant (bitmap) kernel's L2 hit rate and DRAM throughput
    for r in drows[1:]:
        if r[M] in keep:
            lines.append(f"{r[K].split('(')[0][:28]:28s} {r[M]:36s} {r[V]:>18s} {r[U]}")
        if "k_hash_cta<0, 1>" in r[K] and r[M] in ("L2 Hit Rate", "DRAM Throughput") and r[M] not in top:
            top[r[M]] = float(r[V].replace(",", ""))
    rr = list(csv.reader(io.StringIO(raw)))
    h = rr[0]
    traffic = 0.0
    stall_keys = [k for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
    for r in rr[2:]:
        name = r[h.index("Kernel Name")].split("(")[0]
        rd = float(r[h.index("dram__bytes_read.sum")].replace(",", ""))
        wr = float(r[h.index("dram__bytes_write.sum")].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale[rr[1][h.index("dram__bytes_read.sum")]]
        wr *= scale[rr[1][h.index("dram__bytes_write.sum")]]
        traffic += rd + wr
        lines.append(f"{name[:28]:28s} dram read {rd/1e9:.3f} GB  write {wr/1e9:.3f} GB")
        st = sorted(((float(r[h.index(k)].replace(',', '') or 0), k) for k in stall_keys), reverse=True)
        tots = sum(v for v, _ in st) or 1
        lines.append("   stalls: " + ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} "
                                              f"{100*v/tots:.0f}%" for v, k in st[:6]))
    open(os.path.join(ROOT, "profiles", f"{tag}_intersect_full.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    d = json.load(open(tf)) if os.path.exists(tf) else {}
    d[workload] = {"dram_bytes_per_launch": traffic, "source": f"profiles/{tag}_intersect_full.txt "
                   "(sum of dram__bytes_read+write over the intersection kernels of one step)",
                   "bitmap_kernel_l2_hit_pct": top.get("L2 Hit Rate"),
                   "bitmap_kernel_dram_throughput_pct": top.get("DRAM Throughput")}
    json.dump(d, open(tf, "w"), indent=1)
