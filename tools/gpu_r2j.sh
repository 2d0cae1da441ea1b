# Round-2 pass J: full GPU suite + smoke, every config with the oracle leg, launch list + ncu of
# router / permute / combine / GEMMs, sanitizers on every engine path (incl. sharded shared).
T=${1:-r2j}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/$T
python __graft_entry__.py > gpurun_out/$T/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/$T/tests.log 2>&1; echo "rc=$?" >> gpurun_out/$T/tests.log
tail -3 gpurun_out/$T/tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/$T/smoke.log 2>&1; tail -1 gpurun_out/$T/smoke.log
bash tools/gpu_allcfg.sh gpurun_out/$T/allcfg
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$T/launches_c1.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"router|permute|combine" -c 3 -o gpurun_out/$T/prof_route_c1 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"router|permute|combine" -c 3 -o gpurun_out/$T/prof_route_c4 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --config dsv2_lite > /dev/null 2>&1
for S in memcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $S --target-processes all python tools/sanitize_paths.py > gpurun_out/$T/sanitizer_$S.log 2>&1; echo "$S rc=$?"; tail -2 gpurun_out/$T/sanitizer_$S.log
done
ls gpurun_out/$T
