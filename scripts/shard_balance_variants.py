"""Development aid: shard_balance (max/mean of per-rank a6 time) for variants/<name>/ builds."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
scale = sys.argv[1]
for nm in sys.argv[2].split(","):
    lib = os.path.join(ROOT, "paper_1804_06926_b200", "libtc_b200.so") if nm == "base" else \
        os.path.join(ROOT, "variants", nm, "libtc_b200.so")
    code = f"""
import sys, json; sys.path.insert(0, {ROOT!r}); sys.argv = ['x', '{scale}']; __file__ = {os.path.join(ROOT, 'scripts', 'shard_balance.py')!r}
import paper_1804_06926_b200 as tc; tc._LIB_PATH = {lib!r}
exec(open({os.path.join(ROOT, 'scripts', 'shard_balance.py')!r}).read())
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    import json
    for line in r.stdout.splitlines():
        d = json.loads(line)
        for g, res in d.items():
            print(nm, g, {w: (round(res[w]["ix_max_over_mean"], 3), round(max(res[w]["ix_ms"]), 2))
                          for w in ("world2", "world4", "world8")}, flush=True)
    if r.returncode:
        print(r.stderr[-2000:])
