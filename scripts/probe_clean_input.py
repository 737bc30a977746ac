"""Development aid: SURVEY 8(d)'s clean-input call (TC_CLEAN | TC_SORTED) on R-MAT s21 and the
road mesh's clean CSR through the pipeline: median of 7 CUDA-event timed calls + phases."""
import sys, os, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import graphgen as G
import paper_1804_06926_b200 as tc
if os.environ.get("TC_LIB"):
    tc._LIB_PATH = os.environ["TC_LIB"]
from bench import clean_csr_of
for name, g in (("s21", G.rmat(21)), ("chung_lu", G.chung_lu())):
    rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda(); cl = torch.from_numpy(g.col.view(np.int32)).cuda()
    crp, ccl = clean_csr_of(tc, torch, rp, cl)
    ts = []
    for it in range(9):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        T = tc.count_ex(crp, ccl, clean=True, sorted_rows=True)
        b.record(); torch.cuda.synchronize()
        if it >= 2: ts.append(a.elapsed_time(b))
    _, st = tc.count_ex(crp, ccl, clean=True, sorted_rows=True, with_stats=True)
    print(f"{os.environ.get('TC_LIB','').split('/')[-2:-1]} {name} clean-input T={T} {statistics.median(ts):.3f} ms orient {st['ms_orient']:.3f} bin {st['ms_bin']:.3f} ix {st['ms_intersect']:.3f}", flush=True)
    del rp, cl, crp, ccl; torch.cuda.empty_cache()
