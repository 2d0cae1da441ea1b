set -x
python tools/h2d_probe.py 2>&1 | tail -20
timeout 1500 python -m pytest tests -m gpu -x -q -k "full_size" -s 2>&1 | grep -E "max token|passed|failed|Error|error" | tail -20
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch_bench.log 2>&1; tail -2 gpurun_out/ncu_launch_bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:expert_gemm -s 2 -c 2 -o gpurun_out/prof_gemm_r01 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full_gemm.log 2>&1; tail -3 gpurun_out/ncu_full_gemm.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"router|permute|combine|scan" -c 4 -o gpurun_out/prof_route_r01 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_full_route.log 2>&1; tail -3 gpurun_out/ncu_full_route.log
ls -la gpurun_out
