# Router kernel sweep (v3 = round 1; v6 = the default: fp64-widened staging, cp.async ring, register prefetch) on the
# BASELINE shapes + the 131k-token C1 regime + the 128-expert envelope.
# usage: bash tools/gpu_router_sweep.sh <outdir>
O=${1:-gpurun_out/router}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p $O build
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include -I paper_2504_09345_b200/csrc tools/router_bench.cu -L paper_2504_09345_b200 -lmoe_b200 -o build/router_bench
export LD_LIBRARY_PATH=paper_2504_09345_b200:$LD_LIBRARY_PATH
for shape in "4096 4096 8 2" "512 4096 8 2" "8192 6144 8 2" "16384 6144 16 4" "32768 2048 64 6" "4096 2048 64 6" "131072 4096 8 2" "4000 2048 128 1" "1000 512 40 3"; do
  MOE_ROUTER=3 ./build/router_bench $shape
  ./build/router_bench $shape
  for t in 1 2 4; do MOE_ROUTER_TPT=$t ./build/router_bench $shape; done
  MOE_ROUTER_EPT=1 MOE_ROUTER_TPT=1 ./build/router_bench $shape; MOE_ROUTER_EPT=1 MOE_ROUTER_TPT=2 ./build/router_bench $shape
done > $O/sweep.txt 2>&1
cat $O/sweep.txt
