# Round-2 pass K: router v6 compact loop + combine v3 (warp per token part, K-templated): timing,
# parity subset, ncu of route/permute/combine at C1 and C4.
T=${1:-r2k}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/$T build
python __graft_entry__.py > gpurun_out/$T/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include -I paper_2504_09345_b200/csrc tools/router_bench.cu -L paper_2504_09345_b200 -lmoe_b200 -o build/router_bench
export LD_LIBRARY_PATH=paper_2504_09345_b200:$LD_LIBRARY_PATH
for shape in "4096 4096 8 2" "8192 6144 8 2" "16384 6144 16 4" "32768 2048 64 6" "131072 4096 8 2" "4096 2048 64 6"; do ./build/router_bench $shape; done > gpurun_out/$T/router.txt 2>&1
cat gpurun_out/$T/router.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_taskb.py -q -x -k "router or tiny or ragged or sharded or local_transport or full_size or staged" > gpurun_out/$T/tests.log 2>&1; echo "rc=$?" >> gpurun_out/$T/tests.log
tail -2 gpurun_out/$T/tests.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"router|permute|combine" -c 3 -o gpurun_out/$T/prof_route_c1 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"router|permute|combine" -c 3 -o gpurun_out/$T/prof_route_c4 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --config dsv2_lite > /dev/null 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/$T/c1.json 2> gpurun_out/$T/c1.err
tail -c 300 gpurun_out/$T/c1.json
