# Full evidence pass: GPU tests, smoke, bench, ncu launch list + full capture of the top kernel.
# usage: bash tools/gpu_round.sh <tag>
T=${1:-r01}
set -x
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; tail -c 4000 gpurun_out/bench_$T.json; tail -3 gpurun_out/bench_$T.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref_$T.json 2>&1; tail -c 1500 gpurun_out/bench_ref_$T.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:expert_gemm -s 2 -c 2 -o gpurun_out/prof_gemm_$T python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"router|permute|combine" -c 3 -o gpurun_out/prof_route_$T python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
ls gpurun_out
