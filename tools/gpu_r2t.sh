# Round-2 pass T: full GPU suite + smoke + sanitizers after the sharding fixes.
T=${1:-r2t}
O=gpurun_out/$T
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -3 $O/tests.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; tail -1 $O/smoke.log
for S in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $S --target-processes all python tools/sanitize_paths.py > $O/sanitizer_$S.log 2>&1; echo "$S rc=$?"; tail -1 $O/sanitizer_$S.log
done
