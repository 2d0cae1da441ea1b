O=gpurun_out/san2; mkdir -p $O
for T in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $T --target-processes all python tools/sanitize_paths.py > $O/sanitizer_${T}_all_paths.log 2>&1
  echo "$T rc=$?"; tail -3 $O/sanitizer_${T}_all_paths.log
done
