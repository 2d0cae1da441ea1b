mkdir -p gpurun_out/taskb2
python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_taskb.py tests/test_gpu_parity.py -q -k "host or taskb" 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 --taskb > gpurun_out/taskb2/bench_taskb.json 2> gpurun_out/taskb2/bench_taskb.err
python -c "
import json;d=json.load(open('gpurun_out/taskb2/bench_taskb.json'));print(round(d['value']), d['roofline_step']['frac'], d['e2e'])"
