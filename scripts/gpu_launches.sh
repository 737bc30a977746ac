# One gpurun lease: ncu launch list (per-kernel device times) of one bench-workload call.
#   bash scripts/gpu_launches.sh [scale] [extra bench.py args]
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
S=${1:-21}; shift
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_s$S$1.csv \
    python bench.py --one-call --scale $S "$@" > gpurun_out/ncu_launch.log 2>&1
python scripts/launch_table.py gpurun_out/launches_s$S$1.csv
