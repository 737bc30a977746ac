# One gpurun call: bench line, launch list of the bench command, full captures.
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-next > gpurun_out/launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_hash_cta|k_hash_warp" -c 3 \
    -o gpurun_out/ix_full python scripts/one_call.py 21 > gpurun_out/ix_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_rs_pass|k_edges" -s 1 -c 3 \
    -o gpurun_out/pre_full python scripts/one_call.py 21 > gpurun_out/pre_full.log 2>&1
ls -la gpurun_out
