# Round-2 pass E (re-entry): router sweep, all GPU tests, smoke, C1/C4 bench, launch list, router ncu.
T=${1:-r2e}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/$T build
python __graft_entry__.py > gpurun_out/$T/build.log 2>&1
bash tools/gpu_router_sweep.sh gpurun_out/$T
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/$T/tests.log 2>&1; echo "rc=$?" >> gpurun_out/$T/tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/$T/smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/$T/c1.json 2> gpurun_out/$T/c1.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --config dsv2_lite > gpurun_out/$T/c4.json 2> gpurun_out/$T/c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$T/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"router" -c 2 -o gpurun_out/$T/prof_router python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
tail -3 gpurun_out/$T/tests.log; tail -1 gpurun_out/$T/smoke.log
