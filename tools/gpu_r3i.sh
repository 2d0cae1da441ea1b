# router v7 probe: where block 0's cycles go (loop, last warp, top-k) at C1 / C4 / DBRX
O=gpurun_out/router7l
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p $O build
python -c "from paper_2504_09345_b200 import build; build.build()" > $O/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include -I paper_2504_09345_b200/csrc tools/router_bench.cu -L paper_2504_09345_b200 -lmoe_b200 -o build/router_bench
export LD_LIBRARY_PATH=paper_2504_09345_b200:$LD_LIBRARY_PATH
for shape in "4096 4096 8 2" "16384 6144 16 4" "32768 2048 64 6" "1000 512 40 3"; do
  MOE_ROUTER=7 ./build/router_bench $shape; MOE_ROUTER=7 MOE_ROUTER_TPT=1 ./build/router_bench $shape
done > $O/sweep.txt 2>&1
cat $O/sweep.txt
