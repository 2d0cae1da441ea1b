python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for C in dsv2_lite mixtral_8x7b; do
  timeout 900 python bench.py --config $C --steps 20 --warmup 3 --no-cpu --no-e2e > /tmp/b_$C.json 2>/dev/null
  python -c "
import json;d=json.load(open('/tmp/b_$C.json'));k=d['per_kernel_ms_per_step_rank0']
print('$C', round(d['value']), 'step %.2f'%d['ms_per_step'], 'roof %.4f'%d['roofline_step']['frac'], 'g1 %.3f g2 %.3f'%(k['gemm1_ms'],k['gemm2_ms']))"
done
timeout 1200 python -m paper_2504_09345_b200.profiler --config dsv2_lite --tokens 32768,65536,131072,196608 --steps 3 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); print('dsv2 n_real', round(d['n_real']), [(p['tokens'], round(p['step_ms'],2), round(p['gpu_ms'],2)) for p in d['points']])"
