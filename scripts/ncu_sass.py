"""Development aid: per-SASS-line stall samples of the FIRST kernel in an ncu report."""
import csv, io, subprocess, sys
rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.006
kfilter = sys.argv[3] if len(sys.argv) > 3 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if kfilter:
    cmd += ["-k", f"regex:{kfilter}"]
rows = list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))
blocks, cur = [], None
for r in rows:
    if r and r[0].startswith("Kernel Name"):
        cur = []
        blocks.append(cur)
        continue
    if cur is not None:
        cur.append(r)
b = blocks[0]
h = b[0]
ai, si, ie = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
ws, at = h.index("Warp Stall Sampling (All Samples)"), h.index("Avg. Threads Executed")
data = []
for r in b[1:]:
    try:
        data.append((r[ai][-4:], r[si], int(r[ie] or 0), int(r[ws] or 0), r[at]))
    except (ValueError, IndexError):
        pass
tot = sum(d[3] for d in data) or 1
te = sum(d[2] for d in data) or 1
print(f"samples {tot} executed {te}")
for d in data:
    if d[3] > tot * thr or d[2] > te * 0.01:
        print(f"{d[0]} exec {d[2]:>10} st {100*d[3]/tot:5.1f}% thr {d[4]:>3} {d[1][:80]}")
