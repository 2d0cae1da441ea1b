python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
nvidia-smi topo -m 2>&1 | head -8; lscpu | grep -i "numa\|socket\|model name" | head -6
for A in 1 0; do
  MOE_BENCH_NO_AFFINITY=$A timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu > /tmp/b.json 2>/dev/null
  python -c "
import json;d=json.load(open('/tmp/b.json'));r=d['roofline_step']
print('no_affinity=$A', round(d['value']), 'e2e', round(d['e2e']['value']), 'probe %.2f'%r['host_link_probe_gbs_rank0'], 'achieved %.2f'%r['h2d_achieved_gbs_in_copies_rank0'], d['host_affinity'])"
done
