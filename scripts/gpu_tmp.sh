python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_graph.py -x -q 2>&1 | tail -15
python scripts/probe_latency.py '{"graph_cache":1}'
