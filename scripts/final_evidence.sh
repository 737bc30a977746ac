# One gpurun lease: everything the round's evidence needs (smoke, the whole -m gpu suite, the bench
# line, the s21 launch list, ncu --set full captures of the step's main kernels).
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -4 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -14 gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --one-call > gpurun_out/launches.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_hash_cta|k_rs_pass|k_unique_scatter|k_edges|k_orient_pairs|k_hash_warp|k_core_count" \
    -c 12 -o gpurun_out/full -f python bench.py --one-call > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
