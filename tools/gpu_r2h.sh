T=${1:-r2h}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/$T
python __graft_entry__.py > gpurun_out/$T/build.log 2>&1
timeout 600 bash tools/gpu_router_sweep.sh gpurun_out/$T > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "router or tiny or ragged or sharded or local_transport" > gpurun_out/$T/tests.log 2>&1; echo "rc=$?" >> gpurun_out/$T/tests.log
tail -2 gpurun_out/$T/tests.log
grep "MOE_ROUTER=6" gpurun_out/$T/sweep.txt
