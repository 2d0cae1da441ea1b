T=${1:-r2n}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/$T
python __graft_entry__.py > gpurun_out/$T/build.log 2>&1
timeout 600 bash tools/gpu_router_sweep.sh gpurun_out/$T > /dev/null 2>&1
grep -E "TPT=auto LANES=auto|LANES=expert" gpurun_out/$T/sweep.txt | grep -v "ROUTER=3"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "router or tiny or full_size" > gpurun_out/$T/tests.log 2>&1; echo "rc=$?" >> gpurun_out/$T/tests.log
tail -2 gpurun_out/$T/tests.log
