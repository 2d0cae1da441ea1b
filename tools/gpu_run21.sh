mkdir -p gpurun_out/swap
python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
MOE_GEMM_SWAP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:swap -c 2 -f -o gpurun_out/swap/ncu_swap_c1 python tools/layer_once.py mixtral_8x7b 0 1 > gpurun_out/swap/ncu_swap_c1.log 2>&1
MOE_GEMM_SWAP=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:pair -c 1 -f -o gpurun_out/swap/ncu_pair_c1 python tools/layer_once.py mixtral_8x7b 0 1 > gpurun_out/swap/ncu_pair_c1.log 2>&1
tail -3 gpurun_out/swap/ncu_swap_c1.log gpurun_out/swap/ncu_pair_c1.log
