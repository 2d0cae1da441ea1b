set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 900 python -m paper_2504_09345_b200.profiler --config mixtral_8x7b --tokens 4096,16384,65536,131072 > gpurun_out/profiler_c1.json 2>gpurun_out/profiler_c1.err; tail -c 3000 gpurun_out/profiler_c1.json; tail -5 gpurun_out/profiler_c1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01b.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
python tools/ncu_summary.py --launches gpurun_out/launches_r01b.csv --out gpurun_out/sum_b 2>&1 | head -40
