python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
for SG in "16 8" "24 12" "32 16" "32 8"; do set -- $SG
  MOE_COPY_GROUP=$2 timeout 900 python bench.py --config dsv2_lite --slots $1 --steps 20 --warmup 3 --no-cpu --no-e2e > /tmp/b.json 2>/tmp/b.err
  python -c "
import json;d=json.load(open('/tmp/b.json'));k=d['per_kernel_ms_per_step_rank0'];r=d['roofline_step']
print('slots $1 group $2', round(d['value']), 'step %.3f'%d['ms_per_step'], 'roof %.4f'%r['frac'], 'h2d_gbs %.2f'%r['h2d_achieved_gbs_in_copies_rank0'], 'g1 %.3f'%k['gemm1_ms'], 'launches', d['gpu_launches_per_step'])" || tail -3 /tmp/b.err
done
