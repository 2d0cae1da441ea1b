python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
timeout 600 python bench.py --steps 10 --warmup 3 > /tmp/b1.json 2>/tmp/b1.err; tail -3 /tmp/b1.err
python -c "
import json;d=json.load(open('/tmp/b1.json'));print(round(d['value']), d['ms_per_step_dist_rank0'], d['single_call_latency_ms'], d['host_affinity'], d['cpu_baseline']['cores'], d['e2e']['value'])"
MOE_BENCH_SHARE_GPU=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus 2 --steps 3 --warmup 1 --no-cpu --config tiny > /tmp/b2.json 2>/tmp/b2.err; echo rc=$?
python -c "
import json;d=json.load(open('/tmp/b2.json'));print(round(d['value']), d['config']['ep_transport'], d['host_affinity'], d['single_call_latency_ms'])"; grep -i "error\|Trace" /tmp/b2.err | head -5
