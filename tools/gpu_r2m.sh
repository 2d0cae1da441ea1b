T=${1:-r2m}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/$T
python __graft_entry__.py > gpurun_out/$T/build.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --config dsv2_lite > gpurun_out/$T/c4.json 2> gpurun_out/$T/c4.err
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/$T/c1.json 2> gpurun_out/$T/c1.err
python -c "
import json
for c in ['c1','c4']:
    d=json.loads(open('gpurun_out/$T/'+c+'.json').read().strip().splitlines()[-1])
    print(c, d['value'], d['e2e']['value'], json.dumps(d['e2e'].get('link_roofline')), d['roofline_step']['frac'])
"
