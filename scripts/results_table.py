"""Development aid: BASELINE.md results rows (GPU median of 5 + oracle on host cores)."""
import sys, os, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import graphgen as G, oracle as O
import paper_1804_06926_b200 as tc
cfgs = [("C0 karate", G.karate, True), ("C0 K20", lambda: G.complete(20), True),
        ("C1 R-MAT s21 ef16", lambda: G.rmat(21), True),
        ("C1' R-MAT s21 ef48", lambda: G.rmat(21, 48, seed=4821), False),
        ("C2 Chung-Lu LJ-like", G.chung_lu, True), ("C3 road mesh", G.road_mesh, True),
        ("C4 R-MAT s22", lambda: G.rmat(22), False), ("C4 R-MAT s23", lambda: G.rmat(23), False),
        ("C4 R-MAT s24", lambda: G.rmat(24), False), ("C5 clique-union", G.clique_union, True)]
want = sys.argv[1:]
print("| Config | n | m | T | GPU ms (median of 5, 1 B200) | edges/s | intersect ms | B_hash/t of HBM | oracle s (16 thr) | parity |")
print("|---|---|---|---|---|---|---|---|---|---|")
for name, mk, run_oracle in cfgs:
    if want and not any(w in name for w in want):
        continue
    g = mk()
    rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda(); cl = torch.from_numpy(g.col.view(np.int32)).cuda()
    tc.count_ex(rp, cl)
    ms, ix, st = [], [], None
    for _ in range(5):
        T, st = tc.count_ex(rp, cl, with_stats=True)
        ms.append(st["ms_total"]); ix.append(st["ms_intersect"])
    med, mix = statistics.median(ms), statistics.median(ix)
    frac = st["bytes_hash"] / (mix * 1e-3) / 6545.6e9 if mix > 0 else 0
    osec, par = "-", "closed form" if name.startswith("C0") else "-"
    if run_oracle:
        t0 = time.perf_counter(); To = O.count(g.n, g.rowptr, g.col); osec = f"{time.perf_counter() - t0:.2f}"
        par = "bit-exact" if To == T else f"MISMATCH {To}"
    print(f"| {name} | {g.n:,} | {st['m_undirected']:,} | {T:,} | {med:.3f} | {st['m_undirected'] / med * 1e3:.3e} | "
          f"{mix:.3f} | {frac:.2f} | {osec} | {par} |", flush=True)
    del rp, cl
    torch.cuda.empty_cache()
