python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for C in dsv2_lite mixtral_8x7b; do
  timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-cpu --no-e2e > /tmp/b_$C.json 2>/dev/null
  python -c "
import json;d=json.load(open('/tmp/b_$C.json'));k=d['per_kernel_ms_per_step_rank0']
print('$C', round(d['value']), 'step %.2f'%d['ms_per_step'], 'roof %.4f'%d['roofline_step']['frac'], 'g1 %.3f g2 %.3f'%(k['gemm1_ms'],k['gemm2_ms']), 'g1frac %.3f'%d['roofline']['frac'], 'launches/step', d['gpu_launches_per_step'])"
done
