# router v7 with the 4-threads-per-token top-k above 16 experts: sweep + routing parity tests
O=gpurun_out/router7n
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p $O build
python __graft_entry__.py > $O/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include -I paper_2504_09345_b200/csrc tools/router_bench.cu -L paper_2504_09345_b200 -lmoe_b200 -o build/router_bench
export LD_LIBRARY_PATH=paper_2504_09345_b200:$LD_LIBRARY_PATH
for shape in "4096 4096 8 2" "16384 6144 16 4" "32768 2048 64 6" "4096 2048 64 6" "1000 512 40 3" "2000 1024 33 8"; do
  ./build/router_bench $shape; MOE_ROUTER_TPT=1 ./build/router_bench $shape
done > $O/sweep.txt 2>&1
cat $O/sweep.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "router or full_size or tie or special" > $O/tests.log 2>&1; tail -3 $O/tests.log
