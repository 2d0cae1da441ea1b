# Round-2 pass Q: sharded shared experts with slice widths that divide no slot (per-slot W2
# views), bench P2P setup that keeps collectives aligned when a rank fails, EP4 C4 with e2e.
T=${1:-r2q}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/$T
python __graft_entry__.py > gpurun_out/$T/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_taskb.py tests/test_gpu_ep_ipc.py -q -x -k "sharded or local_expert" > gpurun_out/$T/tests.log 2>&1; echo "rc=$?" >> gpurun_out/$T/tests.log
tail -2 gpurun_out/$T/tests.log
for W in 4 8; do
  MOE_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 2958$W bench.py --gpus $W --steps 3 --warmup 3 --config dsv2_lite > gpurun_out/$T/ep${W}_c4.json 2> gpurun_out/$T/ep${W}_c4.err
  echo "W=$W rc=$?"; tail -c 250 gpurun_out/$T/ep${W}_c4.json; echo
done
