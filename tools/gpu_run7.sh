set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm_tile_variants" 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for P in 0 1; do MOE_GEMM_PAIR=$P timeout 900 python -m paper_2504_09345_b200.profiler --config mixtral_8x7b --tokens 4096,16384,65536,131072 > gpurun_out/profiler_pair$P.json 2>gpurun_out/profiler_pair$P.err; cat gpurun_out/profiler_pair$P.json; tail -3 gpurun_out/profiler_pair$P.err; done
