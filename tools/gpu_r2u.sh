T=${1:-r2u}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/$T build
python __graft_entry__.py > gpurun_out/$T/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include -I paper_2504_09345_b200/csrc tools/router_bench.cu -L paper_2504_09345_b200 -lmoe_b200 -o build/router_bench
export LD_LIBRARY_PATH=paper_2504_09345_b200:$LD_LIBRARY_PATH
for shape in "4096 4096 8 2" "512 4096 8 2" "8192 6144 8 2" "1000 512 8 2"; do
  ./build/router_bench $shape; MOE_ROUTER_REG=1 ./build/router_bench $shape; MOE_ROUTER_REG=1 MOE_ROUTER_EPT=1 ./build/router_bench $shape
done 2>&1 | cut -c1-170
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "router_experts_per_warp and v6-0-tpt1" 2>&1 | tail -2
MOE_ROUTER_REG=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "router_experts_per_warp and (v6-0-tpt1 or v6-1-tpt1)" 2>&1 | tail -2
