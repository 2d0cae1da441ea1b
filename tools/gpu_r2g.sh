# Round-2 pass G: router v6 sweep (bitwise vs v3) + router parity tests, ncu --set full of the
# router (C1, C4) and of the expert GEMMs at C1 (traffic per launch of the current binary).
T=${1:-r2g}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/$T
python __graft_entry__.py > gpurun_out/$T/build.log 2>&1
timeout 600 bash tools/gpu_router_sweep.sh gpurun_out/$T > /dev/null 2>&1
grep -c "0 of" gpurun_out/$T/sweep.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "router or full_size or tiny or ragged or sharded" > gpurun_out/$T/tests.log 2>&1; echo "rc=$?" >> gpurun_out/$T/tests.log
tail -2 gpurun_out/$T/tests.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"router" -c 1 -o gpurun_out/$T/prof_router_c1 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"router" -c 1 -o gpurun_out/$T/prof_router_c4 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --config dsv2_lite > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:expert_gemm -s 4 -c 4 -o gpurun_out/$T/prof_gemm_c1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$T/launches_c1.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
ls gpurun_out/$T
