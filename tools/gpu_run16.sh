timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for P in auto 0; do
 MOE_GEMM_PAIR=$P timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/c1_pair_$P.json 2>&1
 python -c "
import json;d=json.load(open('gpurun_out/c1_pair_$P.json')); r=d['roofline']
print('pair=$P', round(d['value']), 'gemm1 TF', round(r['achieved']), 'frac', round(r['frac'],3), d['per_kernel_ms_per_step_rank0'])"
done
MOE_GEMM_PAIR=auto timeout 900 python -m paper_2504_09345_b200.profiler --config mixtral_8x7b --tokens 4096,16384,65536,131072 > gpurun_out/profiler_auto.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/profiler_auto.json')); print('auto', [(p['tokens'], round(p['gemm_ms'],2)) for p in d['points']], 'n_real', round(d['n_real']))"
