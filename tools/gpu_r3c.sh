# router v7 in-kernel clock probe (cycles per channel, SM MHz) on C1 / C4 shapes
O=gpurun_out/router7d
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p $O build
python -c "from paper_2504_09345_b200 import build; build.build()" > $O/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include -I paper_2504_09345_b200/csrc tools/router_bench.cu -L paper_2504_09345_b200 -lmoe_b200 -o build/router_bench
export LD_LIBRARY_PATH=paper_2504_09345_b200:$LD_LIBRARY_PATH
for shape in "4096 4096 8 2" "512 4096 8 2" "4096 1024 8 2" "32768 2048 64 6" "131072 4096 8 2"; do
  for e in auto 1 4 8; do
    if [ $e = auto ]; then unset MOE_ROUTER_EPT; else export MOE_ROUTER_EPT=$e; fi
    MOE_ROUTER=7 timeout 60 ./build/router_bench $shape
  done
  unset MOE_ROUTER_EPT
done > $O/sweep.txt 2>&1
cat $O/sweep.txt
nvidia-smi -q -d CLOCK | head -30 > $O/clocks.txt
