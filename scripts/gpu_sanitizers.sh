# One gpurun lease: compute-sanitizer memcheck / racecheck / synccheck over every entry point
# (scripts/sanitize.py, library-pool workspace so every block is tracked).
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
export TC_ALLOCATOR=library
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 1500 compute-sanitizer --tool $tool python scripts/sanitize.py 2>&1 | grep -E "ok|SUMMARY|rror|hazard" | tail -12
done
