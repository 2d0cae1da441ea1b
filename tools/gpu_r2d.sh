# Round-2 pass D: router sweep + router parity tests + full-size parity + default bench.
T=${1:-r2d}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/$T
bash tools/gpu_router_sweep.sh gpurun_out/$T
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "router or full_size or tiny or ragged" > gpurun_out/$T/tests.log 2>&1; echo "rc=$?" >> gpurun_out/$T/tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/$T/c1.json 2> gpurun_out/$T/c1.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --config dsv2_lite > gpurun_out/$T/c4.json 2> gpurun_out/$T/c4.err
tail -2 gpurun_out/$T/tests.log
