# One gpurun lease: phase timings of variants/<name> builds (scripts/probe_variants.py).
#   bash scripts/gpu_variants.sh "<graphs>" "<names>" [pytest-args...]
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
G=$1; N=$2; shift 2
if [ $# -gt 0 ]; then timeout 900 python -m pytest -q "$@" > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/gputest.log; fi
for g in $G; do timeout 600 python scripts/probe_variants.py $g $N; done
