set -x
MOE_GEMM_PAIR=1 timeout 600 ncu --set full --clock-control none -k regex:expert_gemm -s 2 -c 2 -o gpurun_out/prof_pair python tools/layer_once.py mixtral_8x7b 16384 1 > gpurun_out/ncu_pair.log 2>&1; tail -2 gpurun_out/ncu_pair.log
MOE_GEMM_PAIR=0 timeout 600 ncu --set full --clock-control none -k regex:expert_gemm -s 2 -c 2 -o gpurun_out/prof_single python tools/layer_once.py mixtral_8x7b 16384 1 > gpurun_out/ncu_single.log 2>&1; tail -2 gpurun_out/ncu_single.log
