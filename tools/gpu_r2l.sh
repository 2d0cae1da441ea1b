T=${1:-r2l}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/$T build
python __graft_entry__.py > gpurun_out/$T/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include -I paper_2504_09345_b200/csrc tools/router_bench.cu -L paper_2504_09345_b200 -lmoe_b200 -o build/router_bench
export LD_LIBRARY_PATH=paper_2504_09345_b200:$LD_LIBRARY_PATH
for shape in "4096 4096 8 2" "512 4096 8 2" "8192 6144 8 2" "16384 6144 16 4" "32768 2048 64 6" "131072 4096 8 2" "4096 2048 64 6"; do ./build/router_bench $shape; done > gpurun_out/$T/router.txt 2>&1
cat gpurun_out/$T/router.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"router" -c 1 -o gpurun_out/$T/prof_router_c1 ./build/router_bench 4096 4096 8 2 3 > /dev/null 2>&1
