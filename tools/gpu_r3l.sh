# router v7 over the 65..128-expert envelope vs v6 (MOE_ROUTER_V7_MAX was a knob of that build only; v6 and the knob were removed after this run): sweep + parity
O=gpurun_out/router7o
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p $O build
python __graft_entry__.py > $O/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include -I paper_2504_09345_b200/csrc tools/router_bench.cu -L paper_2504_09345_b200 -lmoe_b200 -o build/router_bench
export LD_LIBRARY_PATH=paper_2504_09345_b200:$LD_LIBRARY_PATH
for shape in "4000 2048 128 1" "8192 2048 128 8" "1000 512 100 4" "32768 2048 128 6" "4096 4096 96 2"; do
  MOE_ROUTER=6 ./build/router_bench $shape
  for t in auto 1 2; do
    if [ $t = auto ]; then unset MOE_ROUTER_TPT; else export MOE_ROUTER_TPT=$t; fi
    MOE_ROUTER_V7_MAX=128 ./build/router_bench $shape
  done
  unset MOE_ROUTER_TPT
done > $O/sweep.txt 2>&1
cat $O/sweep.txt
MOE_ROUTER_V7_MAX=128 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "router_experts_per_warp and 128" > $O/tests.log 2>&1; tail -3 $O/tests.log
