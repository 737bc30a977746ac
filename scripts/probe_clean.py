"""Development aid: clean-input (TC_CLEAN | TC_SORTED) phase times on R-MAT sN for library
variants: TC_LIBS=a:path,b:path (default: the in-tree build)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import graphgen as G
import paper_1804_06926_b200 as tc
import bench
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 21
g = G.rmat(scale, 16)
rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda(); cl = torch.from_numpy(g.col.view(np.int32)).cuda()
crp, ccl = bench.clean_csr_of(tc, torch, rp, cl)
libs = [x.split(":", 1) for x in os.environ.get("TC_LIBS", "").split(",") if x] or [("tree", tc._LIB_PATH)]
for rep in range(2):
    for name, path in libs:
        tc._lib = None
        tc._LIB_PATH = path
        for it in range(3):
            T, st = tc.count_ex(crp, ccl, clean=True, sorted_rows=True, with_stats=True)
        T2, st2 = tc.count_ex(rp, cl, with_stats=True)
        print(f"{name}: clean-input total={st['ms_total']:.2f} orient={st['ms_orient']:.2f} bin={st['ms_bin']:.2f} "
              f"ix={st['ms_intersect']:.2f} | raw total={st2['ms_total']:.2f} clean={st2['ms_clean']:.2f} "
              f"orient={st2['ms_orient']:.2f} T={T}", flush=True)
