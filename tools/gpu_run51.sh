python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3
mkdir -p gpurun_out/allcfg2
for C in mixtral_8x7b mixtral_8x22b dbrx dsv2_lite; do
  timeout 900 python bench.py --config $C --steps 20 --warmup 3 --no-cpu > gpurun_out/allcfg2/bench_$C.json 2> gpurun_out/allcfg2/bench_$C.err
  python -c "
import json;d=json.load(open('gpurun_out/allcfg2/bench_$C.json'));k=d['per_kernel_ms_per_step_rank0']
print('$C', round(d['value']), 'e2e', round(d['e2e']['value']), 'step %.2f'%d['ms_per_step'], 'roof %.4f'%d['roofline_step']['frac'], 'g1frac %.3f'%d['roofline']['frac'], 'slots', d['config']['staging_slots'], 'launches', d['gpu_launches_per_step'])"
done
timeout 900 python bench.py --config mixtral_8x7b --steps 20 --warmup 3 --taskb > gpurun_out/allcfg2/bench_taskb.json 2> gpurun_out/allcfg2/bench_taskb.err
python -c "
import json;d=json.load(open('gpurun_out/allcfg2/bench_taskb.json'));print('taskb', round(d['value']), 'e2e', round(d['e2e']['value']), 'roof %.4f'%d['roofline_step']['frac'])"
