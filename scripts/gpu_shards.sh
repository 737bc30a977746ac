# One gpurun lease: shard balance (scripts/shard_balance.py) of the default build and of
# variants/<name> builds.   bash scripts/gpu_shards.sh "<scales>" "<names>"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in $2; do
  if [ "$v" = base ]; then lib=""; else lib=variants/$v/libtc_b200.so; fi
  echo "== $v"; TC_LIB=$lib python scripts/shard_balance.py $1 | python -c "
import json,sys
for line in sys.stdin:
    d=json.loads(line); k=list(d)[0]; d=d[k]
    print(k, 'world1 total', round(d['total_ms_world1'],2), 'ix', round(d['ix_ms_world1'],2))
    for w in ('world2','world4','world8'): print(' ', w, 'ix', [round(x,2) for x in d[w]['ix_ms']], 'max/mean', round(d[w]['ix_max_over_mean'],3), 'sum/w1', round(d[w]['ix_sum_over_world1'],3), 'step', round(d[w]['projected_step_ms'],2))
"
done
