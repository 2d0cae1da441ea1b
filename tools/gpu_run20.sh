# swap-AB vs regular: C1..C4 bench (per-kernel ms), profiler sweep at large T
mkdir -p gpurun_out/swap
python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
for C in mixtral_8x7b mixtral_8x22b dbrx dsv2_lite; do
  for SW in 0 1; do
    MOE_GEMM_SWAP=$SW timeout 600 python bench.py --config $C --steps 8 --warmup 3 --no-cpu --no-e2e > gpurun_out/swap/bench_${C}_swap$SW.json 2>gpurun_out/swap/bench_${C}_swap$SW.err
    python -c "
import json;d=json.load(open('gpurun_out/swap/bench_${C}_swap$SW.json'));k=d['per_kernel_ms_per_step_rank0']
print('$C swap=$SW', round(d['value']), 'g1 %.3f g2 %.3f'%(k['gemm1_ms'],k['gemm2_ms']), 'frac %.3f'%d['roofline']['frac'], 'step %.2f'%d['ms_per_step'])"
  done
done
for SW in 0 1; do
  MOE_GEMM_SWAP=$SW timeout 900 python -m paper_2504_09345_b200.profiler --tokens 16384,65536,131072 --steps 2 > gpurun_out/swap/profiler_swap$SW.json 2>&1
  tail -c 1500 gpurun_out/swap/profiler_swap$SW.json; echo
done
