python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_ep_ipc.py -q 2>&1 | tail -3
MOE_BENCH_SHARE_GPU=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 --steps 3 --warmup 1 --no-cpu --config tiny > /tmp/b2.json 2>/tmp/b2.err; echo rc=$?
python -c "
import json;d=json.load(open('/tmp/b2.json'));print(round(d['value']), d['config']['ep_transport'])"; grep -i "unavailable\|error" /tmp/b2.err | head -3
