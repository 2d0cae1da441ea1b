# swap-AB GEMM bring-up: new packing (all GEMM tests) + swap tests, then C1 bench both ways
mkdir -p gpurun_out/swap
python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "tiny or ragged" 2>&1 | tail -3
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -s -k "swap" 2>&1 | tail -15 | tee gpurun_out/swap/pytest_swap.log
