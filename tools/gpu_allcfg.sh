set -x
for C in mixtral_8x22b dbrx dsv2_lite tiny; do
  timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_$C.json 2> gpurun_out/bench_$C.err; tail -c 600 gpurun_out/bench_$C.json | head -c 600; echo; tail -2 gpurun_out/bench_$C.err
done
for C in dbrx dsv2_lite; do MOE_GEMM_PAIR=1 timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_${C}_pair.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/bench_${C}_pair.json'));print('$C pair', d['value'], d['per_kernel_ms_per_step_rank0'])"; done
