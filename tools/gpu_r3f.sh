# router v7 default: router sweep (v6 vs v7), full GPU suite + smoke, default bench line and C4 line
O=gpurun_out/r3f
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p $O build
python __graft_entry__.py > $O/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include -I paper_2504_09345_b200/csrc tools/router_bench.cu -L paper_2504_09345_b200 -lmoe_b200 -o build/router_bench
export LD_LIBRARY_PATH=paper_2504_09345_b200:$LD_LIBRARY_PATH
for shape in "4096 4096 8 2" "8192 6144 8 2" "16384 6144 16 4" "32768 2048 64 6" "131072 4096 8 2" "64 128 8 2" "4000 2048 128 1"; do
  MOE_ROUTER=6 ./build/router_bench $shape; ./build/router_bench $shape
done > $O/router_sweep.txt 2>&1
cat $O/router_sweep.txt
timeout 2400 python -m pytest tests -m gpu -q -x --durations=5 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -3 $O/tests.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; tail -c 400 $O/bench_default.json; echo
timeout 900 python bench.py --config dsv2_lite --no-cpu > $O/bench_dsv2.json 2> $O/bench_dsv2.err; tail -c 200 $O/bench_dsv2.json; echo
