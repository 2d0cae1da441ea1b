mkdir -p gpurun_out/swap
python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
run() {  # label, env...
  env "$@" MOE_GEMM_SWAP=1 timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e > /tmp/b.json 2>/dev/null
  g1=$(python -c "import json;d=json.load(open('/tmp/b.json'));k=d['per_kernel_ms_per_step_rank0'];print('g1 %.3f g2 %.3f'%(k['gemm1_ms'],k['gemm2_ms']))")
  env "$@" MOE_GEMM_SWAP=1 timeout 600 python -m paper_2504_09345_b200.profiler --tokens 65536 --steps 2 > /tmp/p.json 2>/dev/null
  g65=$(python -c "import json;d=json.load(open('/tmp/p.json'));print('65k gemm %.2f'%d['points'][0]['gemm_ms'])")
  echo "$* : C1 $g1 | $g65"
}
run MOE_SWAP_DBG=0
run MOE_SWAP_DBG=1
run MOE_SWAP_DBG=2
run MOE_GEMM_GROUPM=8
run MOE_GEMM_GROUPM=32
run MOE_GEMM_GROUPM=4
