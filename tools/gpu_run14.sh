for S in 8 12 16; do for G in 2 4; do
MOE_COPY_GROUP=$G timeout 600 python bench.py --config dsv2_lite --steps 10 --warmup 3 --no-cpu --no-e2e --slots $S > gpurun_out/c4_s${S}_g${G}.json 2>&1
python -c "
import json;d=json.load(open('gpurun_out/c4_s${S}_g${G}.json')); r=d['roofline_step']
print('slots $S group $G', round(d['value']), 'frac', round(r['frac'],4), 'h2d_gbs', round(r['h2d_achieved_gbs_in_copies_rank0'],2), 'h2d_ms', round(d['per_kernel_ms_per_step_rank0']['h2d_ms'],3), 'ms', round(d['ms_per_step'],3))"
done; done
