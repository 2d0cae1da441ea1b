# Round-2 pass R: bench.py under torchrun with W = 2 / 4 / 8 ranks sharing the GPU, every
# BASELINE workload, e2e on -- a path check of every EP shape the bench can run (timings meaningless).
T=${1:-r2r}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/$T
python __graft_entry__.py > gpurun_out/$T/build.log 2>&1
p=29600
for c in mixtral_8x7b mixtral_8x22b dbrx dsv2_lite; do for W in 2 4 8; do
  p=$((p+1))
  MOE_BENCH_SHARE_GPU=1 timeout 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port $p bench.py --gpus $W --steps 2 --warmup 3 --config $c > gpurun_out/$T/ep${W}_$c.json 2> gpurun_out/$T/ep${W}_$c.err
  rc=$?
  python -c "
import json,sys
try:
    d=json.loads(open('gpurun_out/$T/ep${W}_$c.json').read().strip().splitlines()[-1])
    print('$c W=$W rc=$rc', round(d['value']), 'e2e', round(d['e2e']['value']), d['e2e']['matches_device_path'], d['config']['ep_transport'], d['config'].get('shared_experts'))
except Exception as e:
    print('$c W=$W rc=$rc FAILED', e)
"
done; done
