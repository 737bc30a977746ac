"""Development aid: oracle wall time (threads from OMP_NUM_THREADS) on the named configs."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen as G, oracle as O
cfgs = {"C1": lambda: G.rmat(21), "C3": G.road_mesh, "C5": G.clique_union, "K20": lambda: G.complete(20),
        "karate": G.karate}
for name in sys.argv[1:]:
    g = cfgs[name]()
    O.count(g.n, g.rowptr, g.col)
    t0 = time.perf_counter(); T = O.count(g.n, g.rowptr, g.col); s = time.perf_counter() - t0
    print(f"{name} threads={O.num_threads()} T={T} oracle_s={s:.4f}", flush=True)
