"""Development aid: per-call latency (synchronous, median of 30) of tc_count_ex on small and mid
R-MAT graphs through the pipeline (tiny_max_n = 0), with kernel launch counts."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import graphgen as G
import paper_1804_06926_b200 as tc
kw = {}
if len(sys.argv) > 1:
    import json
    kw = json.loads(sys.argv[1])
for sc in (8, 10, 12, 14, 16, 18):
    g = G.rmat(sc, 16)
    rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda(); cl = torch.from_numpy(g.col.view(np.int32)).cuda()
    for _ in range(5):
        tc.count_ex(rp, cl, tiny_max_n=0, lowdeg_max=0, **kw)
    ts = []
    l0 = tc.launches_issued()
    for _ in range(30):
        torch.cuda.synchronize()
        t = time.perf_counter()
        T = tc.count_ex(rp, cl, tiny_max_n=0, lowdeg_max=0, **kw)
        ts.append(time.perf_counter() - t)
    print(f"s{sc}: {1e6 * sorted(ts)[15]:8.1f} us/call  launches/call {(tc.launches_issued() - l0) / 30:.0f}  T={T}", flush=True)
