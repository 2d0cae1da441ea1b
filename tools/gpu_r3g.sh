# router v7 ncu --set full (source level) at C1 and C4 + probe lines
O=gpurun_out/router7j
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p $O build
python -c "from paper_2504_09345_b200 import build; build.build()" > $O/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -lineinfo -I include -I paper_2504_09345_b200/csrc tools/router_bench.cu -L paper_2504_09345_b200 -lmoe_b200 -o build/router_bench
export LD_LIBRARY_PATH=paper_2504_09345_b200:$LD_LIBRARY_PATH
for shape in "4096 4096 8 2" "32768 2048 64 6"; do MOE_ROUTER=7 ./build/router_bench $shape; done > $O/sweep.txt 2>&1
cat $O/sweep.txt
MOE_ROUTER=7 timeout 600 ncu --set full --import-source on --clock-control none -k regex:router_v7 -c 1 -o $O/v7_c1 ./build/router_bench 4096 4096 8 2 3 > $O/ncu_c1.log 2>&1
MOE_ROUTER=7 timeout 600 ncu --set full --import-source on --clock-control none -k regex:router_v7 -c 1 -o $O/v7_c4 ./build/router_bench 32768 2048 64 6 3 > $O/ncu_c4.log 2>&1
ls $O
