mkdir -p gpurun_out/swap
python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "swap or tiny or ragged or tile_variants" 2>&1 | tail -2
for C in mixtral_8x7b dsv2_lite; do
  SW=1; MOE_GEMM_SWAP=$SW timeout 600 python bench.py --config $C --steps 8 --warmup 3 --no-cpu --no-e2e > gpurun_out/swap/bench_${C}_rr4.json 2>&1
  python -c "
import json;d=json.load(open('gpurun_out/swap/bench_${C}_rr4.json'));k=d['per_kernel_ms_per_step_rank0']
print('$C swap-rr', round(d['value']), 'g1 %.3f g2 %.3f'%(k['gemm1_ms'],k['gemm2_ms']), 'frac %.3f'%d['roofline']['frac'], 'step %.2f'%d['ms_per_step'])"
done
MOE_GEMM_SWAP=1 timeout 900 python -m paper_2504_09345_b200.profiler --tokens 65536,131072 --steps 2 > gpurun_out/swap/profiler_rr4.json 2>&1; tail -c 700 gpurun_out/swap/profiler_rr4.json; echo
MOE_GEMM_SWAP=1 timeout 600 ncu --set full --clock-control none -k regex:swap -c 2 -f -o gpurun_out/swap/ncu_swaprr4_c1 python tools/layer_once.py mixtral_8x7b 0 1 > /dev/null 2>&1
