"""Development aid: per-CUDA-source-line stall samples of an ncu report (needs -lineinfo)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 3:
    args += ["-k", sys.argv[3]]
out = subprocess.run(args, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res, fname, hdr, func = {}, None, None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Function Name":
        func = r[1][:40]; continue
    if r[0] == "Line No":
        hdr = r; ws = hdr.index("Warp Stall Sampling (All Samples)"); ie = hdr.index("Instructions Executed"); continue
    if hdr and r[0] not in ("",) and len(r) > ws:
        try:
            s = int(r[ws].replace(",", "") or 0) if r[ws] != "-" else 0
            e = int(r[ie].replace(",", "") or 0) if r[ie] != "-" else 0
        except ValueError:
            continue
        k = (func, fname, r[0])
        a = res.setdefault(k, [0, 0, r[1].strip()[:80]])
        a[0] += s; a[1] += e
tot = sum(v[0] for v in res.values()) or 1
for (func, f, ln), (s, e, src) in sorted(res.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100*s/tot:5.1f}% exec {e:>10d} {f}:{ln} {src}")
