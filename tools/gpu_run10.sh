set -x
for H in 0 1; do for P in 0 1; do
MOE_GEMM_L2HINT=$H MOE_GEMM_PAIR=$P timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active -k regex:expert_gemm -s 2 -c 2 --csv python tools/layer_once.py mixtral_8x7b 65536 1 2>&1 | grep -E "expert_gemm" | awk -F'","' '{print $5" | "$(NF-2)" = "$NF}' | cut -c1-40,150-260
echo "---- H=$H P=$P"
done; done
for H in 0 1; do MOE_GEMM_L2HINT=$H timeout 900 python -m paper_2504_09345_b200.profiler --config mixtral_8x7b --tokens 4096,16384,65536,131072 > gpurun_out/profiler_h$H.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/profiler_h$H.json')); print('H=$H', [(p['tokens'], round(p['gemm_ms'],2)) for p in d['points']], 'n_real', round(d['n_real']))"; done
