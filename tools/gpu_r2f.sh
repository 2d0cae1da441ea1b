# Round-2 pass F: sharded shared experts (MOE_FLAG_SHARD_SHARED) tests, EP bench path checks at
# the BASELINE shapes (8 ranks sharing this GPU), the C1 compute-bound regime (2 x n_real).
T=${1:-r2f}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/$T
python __graft_entry__.py > gpurun_out/$T/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sharded or local_transport" > gpurun_out/$T/tests_local.log 2>&1; echo "rc=$?" >> gpurun_out/$T/tests_local.log
tail -3 gpurun_out/$T/tests_local.log
timeout 900 python -m pytest tests/test_gpu_ep_ipc.py -q -x -s -k "sharded" > gpurun_out/$T/tests_ipc.log 2>&1; echo "rc=$?" >> gpurun_out/$T/tests_ipc.log
tail -3 gpurun_out/$T/tests_ipc.log
for c in dsv2_lite mixtral_8x7b mixtral_8x22b; do
  MOE_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 8 --steps 5 --warmup 3 --config $c --no-e2e > gpurun_out/$T/ep8_$c.json 2> gpurun_out/$T/ep8_$c.err
  tail -c 300 gpurun_out/$T/ep8_$c.json; echo
done
MOE_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 8 --steps 5 --warmup 3 --config dsv2_lite --no-e2e --shared replicated > gpurun_out/$T/ep8_dsv2_lite_repl.json 2> gpurun_out/$T/ep8_dsv2_lite_repl.err
timeout 900 python bench.py --steps 10 --warmup 3 --tokens 131072 --no-cpu --no-e2e > gpurun_out/$T/c1_131k.json 2> gpurun_out/$T/c1_131k.err
tail -c 400 gpurun_out/$T/c1_131k.json
