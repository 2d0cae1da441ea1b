# conv_probe (F2F / LDS / router-step latencies) + the v7 router probe with widening 4 channels ahead
O=gpurun_out/router7e
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p $O build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/conv_probe.cu -o build/conv_probe && ./build/conv_probe > $O/conv_probe.txt 2>&1
cat $O/conv_probe.txt
python -c "from paper_2504_09345_b200 import build; build.build()" > $O/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include -I paper_2504_09345_b200/csrc tools/router_bench.cu -L paper_2504_09345_b200 -lmoe_b200 -o build/router_bench
export LD_LIBRARY_PATH=paper_2504_09345_b200:$LD_LIBRARY_PATH
for shape in "4096 4096 8 2" "32768 2048 64 6"; do
  for e in auto 1 8; do
    if [ $e = auto ]; then unset MOE_ROUTER_EPT; else export MOE_ROUTER_EPT=$e; fi
    MOE_ROUTER=7 timeout 60 ./build/router_bench $shape
  done
  unset MOE_ROUTER_EPT
done > $O/sweep.txt 2>&1
cat $O/sweep.txt
