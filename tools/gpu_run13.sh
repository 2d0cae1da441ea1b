set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "not full_size" 2>&1 | tail -3
for C in dsv2_lite mixtral_8x7b; do timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_${C}_coal.json 2>&1; python -c "
import json;d=json.load(open('gpurun_out/bench_${C}_coal.json')); r=d['roofline_step']
print('$C', round(d['value']), 'slots', d['config']['staging_slots'], 'frac', round(r['frac'],4), 'h2d_gbs', round(r['h2d_achieved_gbs_in_copies_rank0'],2), 'e2e', round(d['e2e']['value']), d['per_kernel_ms_per_step_rank0'])"; done
