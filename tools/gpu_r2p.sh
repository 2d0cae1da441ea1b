T=${1:-r2p}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/$T build
python __graft_entry__.py > gpurun_out/$T/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include -I paper_2504_09345_b200/csrc tools/router_bench.cu -L paper_2504_09345_b200 -lmoe_b200 -o build/router_bench
export LD_LIBRARY_PATH=paper_2504_09345_b200:$LD_LIBRARY_PATH
for shape in "4096 4096 8 2" "8192 6144 8 2" "16384 6144 16 4" "32768 2048 64 6" "131072 4096 8 2"; do
  ./build/router_bench $shape
  for ks in 1 2 4; do for t in 1 2; do MOE_ROUTER_EPT=8 MOE_ROUTER_KS=$ks MOE_ROUTER_TPT=$t ./build/router_bench $shape; done; done
done > gpurun_out/$T/sweep.txt 2>&1
cat gpurun_out/$T/sweep.txt | cut -c1-175
