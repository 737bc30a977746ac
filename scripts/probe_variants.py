"""Development aid: phase timings of each variants/<name>/libtc_b200.so on one graph config."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
graph = sys.argv[1] if len(sys.argv) > 1 else "s21"
names = sys.argv[2].split(",") if len(sys.argv) > 2 else sorted(os.listdir(os.path.join(ROOT, "variants")))
code = r'''
import sys, os, numpy as np, torch
sys.path.insert(0, @ROOT@)
import paper_1804_06926_b200 as tc
tc._LIB_PATH = @LIB@
import graphgen as G
g = @GRAPH@
rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda(); cl = torch.from_numpy(g.col.view(np.int32)).cuda()
best = None
for it in range(6):
    T, st = tc.count_ex(rp, cl, with_stats=True)
    if it >= 1 and (best is None or st["ms_total"] < best["ms_total"]): best = st
print(f"@NAME@ T={T} total={best['ms_total']:.2f} clean={best['ms_clean']:.2f} orient={best['ms_orient']:.2f} bin={best['ms_bin']:.2f} ix={best['ms_intersect']:.2f}", flush=True)
'''
gexpr = {"s21": "G.rmat(21, 16)", "s22": "G.rmat(22, 16)", "s23": "G.rmat(23, 16)", "s24": "G.rmat(24, 16)",
         "cl": "G.chung_lu()", "road": "G.road_mesh()", "clique": "G.clique_union()"}[graph]
for nm in names:
    lib = os.path.join(ROOT, "paper_1804_06926_b200", "libtc_b200.so") if nm == "base" else \
        os.path.join(ROOT, "variants", nm, "libtc_b200.so")
    c = code.replace("@ROOT@", repr(ROOT)).replace("@LIB@", repr(lib)).replace("@GRAPH@", gexpr).replace("@NAME@", nm)
    subprocess.run([sys.executable, "-c", c])
