python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
for G in 4 6 8; do
  MOE_COPY_GROUP=$G timeout 900 python bench.py --config dsv2_lite --steps 20 --warmup 3 --no-cpu --no-e2e > /tmp/b.json 2>/dev/null
  python -c "
import json;d=json.load(open('/tmp/b.json'));k=d['per_kernel_ms_per_step_rank0'];r=d['roofline_step']
print('group $G', round(d['value']), 'step %.3f'%d['ms_per_step'], 'roof %.4f'%r['frac'], 'h2d_gbs %.2f'%r['h2d_achieved_gbs_in_copies_rank0'], 'g1 %.3f'%k['gemm1_ms'], 'launches', d['gpu_launches_per_step'])"
done
