timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_taskb.py -x -q -k "full_size or ragged or tie or router or random or maxima or tiny or staged" 2>&1 | tail -2
for C in dsv2_lite dbrx mixtral_8x7b; do
  timeout 300 python bench.py --config $C --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_$C.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/r2_$C.json'));k=d['per_kernel_ms_per_step_rank0'];print('$C route_ms', round(k['route_ms'],4), 'value', round(d['value']), 'step', round(d['roofline_step']['frac'],4))"
done
