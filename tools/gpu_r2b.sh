# Round-2 pass B: all GPU tests, then C1 / C4 benches and Task B with one and two partitions.
T=${1:-r2b}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/$T
timeout 2000 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/$T/tests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/$T/tests.log
B="timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu"
$B > gpurun_out/$T/c1.json 2> gpurun_out/$T/c1.err
$B --config dsv2_lite > gpurun_out/$T/c4.json 2> gpurun_out/$T/c4.err
$B --taskb > gpurun_out/$T/tb1.json 2> gpurun_out/$T/tb1.err
$B --taskb --partitions 2 > gpurun_out/$T/tb2.json 2> gpurun_out/$T/tb2.err
$B --taskb --partitions 2 --mover > gpurun_out/$T/tb2m.json 2> gpurun_out/$T/tb2m.err
tail -3 gpurun_out/$T/tests.log
