"""Development aid: for the CTA HASH owners (d+ >= 64, rank span beyond the 2^17-bit
bitmap), how much of N+(owner) lies in the top bitmap window [n - 2^17 + 32, n)?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import graphgen as G
import paper_1804_06926_b200 as tc
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
g = G.rmat(scale, 16)
rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda(); cl = torch.from_numpy(g.col.view(np.int32)).cuda()
off, col = tc.orient(rp, cl)
off = off.cpu().numpy().astype(np.int64); col = col.cpu().numpy().view(np.uint32).astype(np.int64)
n = g.n
dplus = np.diff(off)
dminus = np.bincount(col, minlength=n)
deg = dplus + dminus
order = np.lexsort((np.arange(n), deg))          # rank order (d, id)
newid = np.empty(n, np.int64); newid[order] = np.arange(n)
W0 = n - (1 << 17) + 32
src = np.repeat(np.arange(n), dplus)
hash_owner = (dplus >= 64) & (newid < W0)
sel = hash_owner[src]
in_window = newid[col[sel]] >= W0
# weight each owner element by the owner's in-degree (probe lists ~ in-entries)
w = dminus[src[sel]].astype(np.float64)
print(f"s{scale}: n={n} hash owners={int(hash_owner.sum())} their elements={int(sel.sum())} "
      f"in top window: {in_window.mean():.3f} (in-degree weighted {np.average(in_window, weights=w):.3f})")
for k in (18, 19, 20):
    W = n - (1 << k) + 32
    print(f"  window 2^{k}: fraction {(newid[col[sel]] >= W).mean():.3f}")
