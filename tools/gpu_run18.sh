# Task B (NEXT-2): new tests first (verbose), then the whole GPU suite, then the Task B bench.
mkdir -p gpurun_out/taskb
python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_taskb.py -x -q -s 2>&1 | tail -30 | tee gpurun_out/taskb/pytest_taskb.log
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 | tee gpurun_out/taskb/pytest_all.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/taskb/bench_moe.json 2>gpurun_out/taskb/bench_moe.err
timeout 600 python bench.py --steps 10 --warmup 3 --taskb > gpurun_out/taskb/bench_taskb.json 2>gpurun_out/taskb/bench_taskb.err
tail -c 600 gpurun_out/taskb/bench_moe.json; echo; tail -c 1500 gpurun_out/taskb/bench_taskb.json
