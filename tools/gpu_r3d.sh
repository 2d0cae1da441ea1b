# router v7 with one 2-D TMA box per chunk: probe sweep + router-variant parity tests
O=gpurun_out/router7i
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p $O build
python -c "from paper_2504_09345_b200 import build; build.build()" > $O/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include -I paper_2504_09345_b200/csrc tools/router_bench.cu -L paper_2504_09345_b200 -lmoe_b200 -o build/router_bench
export LD_LIBRARY_PATH=paper_2504_09345_b200:$LD_LIBRARY_PATH
for shape in "4096 4096 8 2" "512 4096 8 2" "8192 6144 8 2" "16384 6144 16 4" "32768 2048 64 6" "131072 4096 8 2" "4000 2048 128 1" "1000 512 40 3" "64 128 8 2"; do
  timeout 60 ./build/router_bench $shape
  for t in auto 1 2; do
    for e in auto 4 8; do
      if [ $t = auto ]; then unset MOE_ROUTER_TPT; else export MOE_ROUTER_TPT=$t; fi
      if [ $e = auto ]; then unset MOE_ROUTER_EPT; else export MOE_ROUTER_EPT=$e; fi
      MOE_ROUTER=7 timeout 60 ./build/router_bench $shape
    done
  done
  unset MOE_ROUTER_TPT MOE_ROUTER_EPT
done > $O/sweep.txt 2>&1
cat $O/sweep.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "router_experts_per_warp" > $O/tests.log 2>&1; tail -3 $O/tests.log
