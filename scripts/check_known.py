"""Large-config parity of the CURRENT code against oracle totals computed earlier on the same
seeded inputs by scripts/check_s24.py (which calls only oracle/): profiles/r02_s26_parity.json
(R-MAT s26) and profiles/r01_s24_parity.json (R-MAT s24).  Runs tc_count_ex under both a1
methods and the sharded multi-GPU pipeline emulated at worlds 2 / 8 (shard.emulate).  Writes
one JSON line."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import graphgen as G
import paper_1804_06926_b200 as tc
from paper_1804_06926_b200 import shard

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
src = {26: "r02_s26_parity.json", 24: "r01_s24_parity.json"}[scale]
rec = json.loads(open(os.path.join(ROOT, "profiles", src)).read().strip().splitlines()[-1])
T_or = rec["T_oracle"]
g = G.rmat(scale, 16)
rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda()
cl = torch.from_numpy(g.col.view(np.int32)).cuda()
out = {"workload": g.name, "raw_arcs": g.arcs, "T_oracle": T_or, "oracle_source": "profiles/" + src}
for method in (0, 1):
    T, st = tc.count_ex(rp, cl, with_stats=True, clean_method=method)
    T, st = tc.count_ex(rp, cl, with_stats=True, clean_method=method)
    out[f"clean_method{method}"] = {"T": T, "ms_total": st["ms_total"], "ms_clean": st["ms_clean"],
                                    "bit_exact": T == T_or}
    tc.trim_workspace() if hasattr(tc, "trim_workspace") else None
for world in (2, 8):
    t0 = time.time()
    T, _, _ = shard.emulate(rp, cl, world)
    out[f"sharded_world{world}"] = {"T": T, "bit_exact": T == T_or, "s": time.time() - t0}
    torch.cuda.empty_cache()
out["bit_exact"] = all(v["bit_exact"] for k, v in out.items() if isinstance(v, dict))
print(json.dumps(out))
