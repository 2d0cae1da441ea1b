set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm_tile_variants" 2>&1 | tail -3
for P in 1; do MOE_GEMM_PAIR=$P timeout 900 python -m paper_2504_09345_b200.profiler --config mixtral_8x7b --tokens 4096,16384,65536,131072 > gpurun_out/profiler_pair$P.json 2>gpurun_out/profiler_pair$P.err; cat gpurun_out/profiler_pair$P.json; tail -3 gpurun_out/profiler_pair$P.err; done
MOE_GEMM_PAIR=1 timeout 600 ncu --set full --clock-control none -k regex:expert_gemm -s 2 -c 2 -o gpurun_out/prof_pair2 python tools/layer_once.py mixtral_8x7b 16384 1 > gpurun_out/ncu_pair2.log 2>&1; tail -1 gpurun_out/ncu_pair2.log
