python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
mkdir -p gpurun_out/sanitizer2
timeout 300 python tools/sanitize_paths.py 2>&1 | tail -2
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_paths.py > gpurun_out/sanitizer2/$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitizer2/$tool.log
done
