# Round-2 pass C: fp64 probe, EP full-size IPC tests, alpha/beta A/B, C4 e2e diagnostics.
T=${1:-r2c}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/$T
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_probe.cu -o build/fp64_probe && ./build/fp64_probe > gpurun_out/$T/fp64_probe.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_ep_ipc.py -q -s --durations=10 > gpurun_out/$T/ep_tests.log 2>&1; echo "rc=$?" >> gpurun_out/$T/ep_tests.log
timeout 900 python tools/ab_partitions.py --steps 8 --rounds 3 > gpurun_out/$T/ab.json 2> gpurun_out/$T/ab.err
timeout 600 python bench.py --config dsv2_lite --steps 20 --warmup 3 --no-cpu > gpurun_out/$T/c4.json 2> gpurun_out/$T/c4.err
tail -3 gpurun_out/$T/ep_tests.log
