# full GPU suite after the W13 repacking + swap-AB kernel (opt-in), then C1 bench (default path)
mkdir -p gpurun_out/r25
python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4 | tee gpurun_out/r25/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r25/bench.json 2> gpurun_out/r25/bench.err
python -c "
import json;d=json.load(open('gpurun_out/r25/bench.json'));k=d['per_kernel_ms_per_step_rank0']
print(round(d['value']), d['e2e']['value'], 'g1 %.3f g2 %.3f'%(k['gemm1_ms'],k['gemm2_ms']), 'frac %.3f'%d['roofline']['frac'], d['roofline_step']['frac'])"
