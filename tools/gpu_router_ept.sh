# Router experts-per-warp (MOE_ROUTER_EPT) sweep: route_ms per step for EPT 1/2/4/8 on C1, DBRX,
# DSV2-Lite (invalid combinations fall back to the default), then the routing parity tests.
mkdir -p gpurun_out/ept
for C in mixtral_8x7b dbrx dsv2_lite; do
 for E in 1 2 4 8; do
  MOE_ROUTER_EPT=$E timeout 300 python bench.py --config $C --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ept/b_${C}_$E.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/ept/b_${C}_$E.json'));k=d['per_kernel_ms_per_step_rank0'];print('$C ept=$E route_ms', round(k['route_ms'],4), 'value', round(d['value']))" 2>/dev/null
 done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -k "full_size or ragged or tie or router or random" 2>&1 | tail -2
