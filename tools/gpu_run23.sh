mkdir -p gpurun_out/swap
python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
MOE_GEMM_SWAP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:swap_kernel -c 1 -f -o gpurun_out/swap/ncu_swap_65k python tools/layer_once.py mixtral_8x7b 65536 1 > /dev/null 2>&1
MOE_GEMM_SWAP=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -c 1 -f -o gpurun_out/swap/ncu_pair_65k python tools/layer_once.py mixtral_8x7b 65536 1 > /dev/null 2>&1
ls -la gpurun_out/swap/*65k*
