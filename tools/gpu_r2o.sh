# Round-2 pass O: the verified router (R6b): sweep + the routing / parity tests that exercise it.
T=${1:-r2o}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/$T
python __graft_entry__.py > gpurun_out/$T/build.log 2>&1
timeout 900 bash tools/gpu_router_sweep.sh gpurun_out/$T > /dev/null 2>&1
grep -v "KS=[124] TPT=[124]" gpurun_out/$T/sweep.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_taskb.py -q -x -k "router or tiny or ragged or tie or full_size or every_top_k or staged or determinism or sharded or local" > gpurun_out/$T/tests.log 2>&1; echo "rc=$?" >> gpurun_out/$T/tests.log
tail -3 gpurun_out/$T/tests.log
