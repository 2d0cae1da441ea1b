# Round-3 session final evidence pass (router v7 default): GPU suite + smoke, default bench + reference arm, every config with
# the oracle leg, Task B (1 / 2 partitions, mover), the compute-bound regime, 8 EP ranks sharing
# the GPU (C4 sharded), ncu launch list + GEMM capture, sanitizers.
T=${1:-r3final}
O=gpurun_out/$T
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
mkdir -p build
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include -I paper_2504_09345_b200/csrc tools/router_bench.cu -L paper_2504_09345_b200 -lmoe_b200 -o build/router_bench
for shape in "64 128 8 2" "4096 4096 8 2" "8192 6144 8 2" "16384 6144 16 4" "32768 2048 64 6" "131072 4096 8 2" "4000 2048 128 1" "8192 2048 128 8" "1000 512 40 3"; do
  LD_LIBRARY_PATH=paper_2504_09345_b200 ./build/router_bench $shape
done > $O/router_sweep.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -3 $O/tests.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; tail -c 300 $O/bench_default.json; echo
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_reference.json 2>&1; tail -c 200 $O/bench_reference.json; echo
bash tools/gpu_allcfg.sh $O/allcfg
for v in "--taskb" "--taskb --partitions 2" "--taskb --partitions 2 --mover"; do
  n=$(echo $v | tr -d ' -')
  timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu $v > $O/bench_$n.json 2> $O/bench_$n.err; tail -c 200 $O/bench_$n.json; echo
done
timeout 900 python bench.py --steps 10 --warmup 3 --tokens 131072 --no-cpu --no-e2e > $O/bench_c1_131k.json 2> $O/bench_c1_131k.err
MOE_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 8 --steps 5 --warmup 3 --config dsv2_lite > $O/ep8_dsv2_lite.json 2> $O/ep8_dsv2_lite.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c1.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:expert_gemm -s 4 -c 2 -o $O/prof_gemm_c1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"router_v7|permute|combine" -c 3 -o $O/prof_route_c1 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
# (compute-sanitizer is closed on this GPU pool: no sanitizer runs)
ls $O
