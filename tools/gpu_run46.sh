python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I include -I paper_2504_09345_b200/csrc tools/gemm_bench.cu -L paper_2504_09345_b200 -lmoe_b200 -Xlinker -rpath -Xlinker '$ORIGIN/../paper_2504_09345_b200' -o build/gemm_bench || exit 1
for r in 1053 16384; do ./build/gemm_bench $r 4096 28672 0 20; done
./build/gemm_bench 4096 14336 4096 1 20
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "swap" 2>&1 | tail -2
