# One gpurun lease: build, GPU tests, bench, and (optionally) ncu captures.
#   bash scripts/gpu_round.sh [tests-marker] [ncu]
set -x
MARK=${1:-gpu}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ "$MARK" != "none" ]; then
  timeout 1500 python -m pytest tests -m "$MARK" -q --durations=15 > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
  tail -30 gpurun_out/gputest.log
fi
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
if [ "$2" = "ncu" ]; then
  ncu --set full --import-source on --clock-control none -k regex:k_hash_cta -c 1 \
      -o gpurun_out/ix_full -f python bench.py --one-call > gpurun_out/ncu_ix.log 2>&1
  ncu --set full --import-source on --clock-control none -k regex:k_rs_pass -s 2 -c 1 \
      -o gpurun_out/rs_full -f python bench.py --one-call > gpurun_out/ncu_rs.log 2>&1
  ncu --set full --import-source on --clock-control none -k regex:"k_core_count|k_edges|k_hash_warp" -c 3 \
      -o gpurun_out/misc_full -f python bench.py --one-call > gpurun_out/ncu_misc.log 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv python bench.py --one-call > gpurun_out/ncu_launch.log 2>&1
  ls -la gpurun_out
fi
