# Round-2 pass S: bench modes under EP (2 / 4 ranks sharing the GPU): Task B, alpha/beta
# partitions, the mover, replicated shared experts, the NCCL transport request.
T=${1:-r2s}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/$T
python __graft_entry__.py > gpurun_out/$T/build.log 2>&1
p=29700
for W in 2 4; do for v in "--taskb" "--taskb --partitions 2" "--mover" "--config dsv2_lite --shared replicated" "--config dsv2_lite --mover"; do
  p=$((p+1)); n=$(echo "$W $v" | tr -d ' -')
  MOE_BENCH_SHARE_GPU=1 timeout 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port $p bench.py --gpus $W --steps 2 --warmup 3 $v > gpurun_out/$T/$n.json 2> gpurun_out/$T/$n.err
  rc=$?
  python -c "
import json
try:
    d=json.loads(open('gpurun_out/$T/$n.json').read().strip().splitlines()[-1])
    print('W=$W $v rc=$rc', round(d['value']), 'e2e', round(d['e2e']['value']), d['e2e']['matches_device_path'], d['config']['ep_transport'], d['config'].get('shared_experts'))
except Exception as e:
    print('W=$W $v rc=$rc FAILED', e)
"
  tail -2 gpurun_out/$T/$n.err | grep -i "error\|exit" | head -2
done; done
