# router v7: warp-per-token top-k for N_e > 16 (v6 vs v7 per shape, with the block-0 probe) + router parity tests
O=gpurun_out/router7m
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p $O build
python -c "from paper_2504_09345_b200 import build; build.build()" > $O/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include -I paper_2504_09345_b200/csrc tools/router_bench.cu -L paper_2504_09345_b200 -lmoe_b200 -o build/router_bench
export LD_LIBRARY_PATH=paper_2504_09345_b200:$LD_LIBRARY_PATH
for shape in "4096 4096 8 2" "512 4096 8 2" "8192 6144 8 2" "16384 6144 16 4" "32768 2048 64 6" "131072 4096 8 2" "1000 512 40 3" "64 128 8 2"; do
  MOE_ROUTER=6 ./build/router_bench $shape; MOE_ROUTER=7 ./build/router_bench $shape
  for t in 1 2; do MOE_ROUTER=7 MOE_ROUTER_TPT=$t ./build/router_bench $shape; done
done > $O/sweep.txt 2>&1
cat $O/sweep.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "router_experts_per_warp or full_size" > $O/tests.log 2>&1; tail -3 $O/tests.log
