python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for C in mixtral_8x7b dsv2_lite mixtral_8x22b dbrx; do for TS in 0 1; do
  MOE_GEMM_TAILSPLIT=$TS timeout 900 python bench.py --config $C --steps 8 --warmup 3 --no-cpu --no-e2e > /tmp/b_$C.json 2>/dev/null
  python -c "
import json;d=json.load(open('/tmp/b_$C.json'));k=d['per_kernel_ms_per_step_rank0']
print('$C split=$TS', round(d['value']), 'step %.2f'%d['ms_per_step'], 'g1 %.3f g2 %.3f'%(k['gemm1_ms'],k['gemm2_ms']), 'g1frac %.3f'%d['roofline']['frac'])"
done; done
MOE_GEMM_TAILSPLIT=1 timeout 900 python -m paper_2504_09345_b200.profiler --tokens 65536,131072 --steps 2 2>/dev/null | tail -c 400
